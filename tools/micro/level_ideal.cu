// Floor of a level-synchronous sparse triangular solve step on one SM:
// per level each active thread gathers K ring values written by the previous level,
// folds them (sequential chain or tree), stores its value to the ring, then syncs.
// mode 0: 480 consumer threads + bar.sync; mode 1: one warp, rows strided over lanes, __syncwarp.
// sum 0: chain a - v*z ... ; sum 1: pairwise tree.
// Operands (slots, values) come from shared memory, loaded before the sync (next level).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NT = 480;
constexpr int RING = 4096;
template <int K, int SUM>
__device__ __forceinline__ double fold(double a, const double* v, const double* z) {
  if (SUM == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) a = a - v[k] * z[k];
    return a;
  } else {
    double p[K];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = v[k] * z[k];
#pragma unroll
    for (int s = 1; s < K; s *= 2)
#pragma unroll
      for (int k = 0; k + s < K; k += 2 * s) p[k] = p[k] + p[k + s];
    return a - p[0];
  }
}
template <int K, int SUM, int MODE>
__global__ void lv(int levels, int nrows, long long* out, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  double* ring = (double*)smem;
  uint16_t* slot = (uint16_t*)(smem + RING * 8);            // [level%2][K][512]
  double* val = (double*)(smem + RING * 8 + 2 * K * 512 * 2);  // [K][512]
  const int t = threadIdx.x;
  for (int i = t; i < RING; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
  for (int i = t; i < 2 * K * 512; i += blockDim.x) slot[i] = 0;
  for (int i = t; i < K * 512; i += blockDim.x) val[i] = 1e-3 * (i & 7);
  uint16_t* gofs = slot;  // [K][512] gather offsets within the previous level
  for (int i = t; i < K * 512; i += blockDim.x) gofs[i] = (uint16_t)(((i % 512) * 7 + (i / 512) * 13) % (nrows > 0 ? nrows : 1));
  __syncthreads();
  // slot pattern: row r of level l reads rows (r*7+k*13) % nrows of level l-1
  long long t0 = clock64();
  double acc = 0;
  if (MODE == 0) {
    for (int l = 0; l < levels; ++l) {
      if (t < nrows) {
        const int base_prev = ((l - 1) * 512) & (RING - 1);
        double v[K], z[K];
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = val[k * 512 + t];
#pragma unroll
        for (int k = 0; k < K; ++k) z[k] = ring[(base_prev + gofs[k * 512 + t]) & (RING - 1)];
        double a = fold<K, SUM>(1.0, v, z);
        ring[((l * 512) + t) & (RING - 1)] = a;
        acc += a;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    }
  } else {
    if (t < 32) {
      for (int l = 0; l < levels; ++l) {
        const int base_prev = ((l - 1) * 512) & (RING - 1);
        for (int r = t; r < nrows; r += 32) {
          double v[K], z[K];
#pragma unroll
          for (int k = 0; k < K; ++k) v[k] = val[k * 512 + r];
#pragma unroll
          for (int k = 0; k < K; ++k) z[k] = ring[(base_prev + gofs[k * 512 + r]) & (RING - 1)];
          double a = fold<K, SUM>(1.0, v, z);
          ring[((l * 512) + r) & (RING - 1)] = a;
          acc += a;
        }
        __syncwarp();
      }
    }
  }
  long long t1 = clock64();
  if (t == 0) out[0] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}
template <int K, int SUM, int MODE>
void run(int nrows, long long* out, double* sink) {
  int smem = RING * 8 + 2 * K * 512 * 2 + K * 512 * 8;
  cudaFuncSetAttribute(lv<K, SUM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int levels = 4000;
  lv<K, SUM, MODE><<<1, MODE == 0 ? NT : 32, smem>>>(levels, nrows, out, sink);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
  printf("K %d %-5s %-8s rows %3d : %7.1f cycles/level (%s)\n", K, SUM ? "tree" : "chain", MODE ? "warp" : "bar480",
         nrows, (double)c / levels, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* out;
  double* sink;
  cudaMalloc(&out, 8);
  cudaMalloc(&sink, 8);
  for (int nr : {1, 32, 64, 96, 128, 256}) {
    run<8, 0, 0>(nr, out, sink);
    run<8, 1, 0>(nr, out, sink);
    run<4, 0, 0>(nr, out, sink);
    if (nr <= 128) {
      run<8, 0, 1>(nr, out, sink);
      run<8, 1, 1>(nr, out, sink);
      run<4, 0, 1>(nr, out, sink);
    }
  }
}
