// Floor of a software-pipelined level loop: slots of the NEXT level's row are loaded
// before the current chain (registers), so after the barrier a thread only issues its
// K ring gathers, the K value loads, the DMUL/DADD chain, one STS, and the barrier.
// usage: ./level_pipe   (prints cycles/level for K entries and R active rows)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NT = 480;
template <int K>
__global__ void lk(int levels, int nrows, long long* out, double* sink, double* gout, int mode) {
  extern __shared__ __align__(128) uint8_t smem[];
  double* ring = (double*)smem;                    // 4096 doubles
  uint16_t* slot = (uint16_t*)(smem + 32768);      // [8 levels][8][512] u16
  double* val = (double*)(smem + 32768 + 65536);   // [8][512]
  const int t = threadIdx.x;
  for (int i = t; i < 4096; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
  for (int i = t; i < 8 * 8 * 512; i += blockDim.x) slot[i] = (uint16_t)((i * 2654435761u) & 4095);
  for (int i = t; i < 8 * 512; i += blockDim.x) val[i] = 1e-3 * (i & 7);
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  uint16_t sl[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) sl[k] = slot[k * 512 + t];
  const bool act = t < nrows;
  for (int l = 0; l < levels; ++l) {
    if (act) {
      double zz[K], v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) zz[k] = ring[sl[k]];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = val[k * 512 + t];
      // next level's slots (independent of the ring)
      const uint16_t* ns = slot + ((l + 1) & 7) * 8 * 512 + t;
#pragma unroll
      for (int k = 0; k < 8; ++k) sl[k] = ns[k * 512];
      double a = 1.0 + l;
#pragma unroll
      for (int k = 0; k < K; ++k) a = a - v[k] * zz[k];
      ring[(l * 512 + t) & 4095] = a;
      if (mode == 1) gout[(l * 512 + t) & ((1 << 20) - 1)] = a;          // coalesced STG per level
      if (mode == 2) gout[((l * 512 + t) * 97) & ((1 << 20) - 1)] = a;   // scattered STG per level
      acc += a;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  }
  long long t1 = clock64();
  if (t == 0) out[0] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}
template <int K>
void run(long long* out, double* sink, double* gout, int mode) {
  int smem = 32768 + 65536 + 32768;
  cudaFuncSetAttribute(lk<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nrows : {1, 32, 160, 480}) {
    lk<K><<<1, NT, smem>>>(10000, nrows, out, sink, gout, mode);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("mode %d K %d rows %3d : %6.1f cycles/level (%s)\n", mode, K, nrows, c / 10000.0, cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
  double* gout; cudaMalloc(&gout, 8 << 20);
  for (int mode = 0; mode < 3; ++mode) { run<1>(out, sink, gout, mode); run<3>(out, sink, gout, mode); run<7>(out, sink, gout, mode); }
}
