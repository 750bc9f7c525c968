#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// variant bits: 1 = skip barrier, 2 = skip fold (ring load/store only), 4 = skip STS
__global__ void lk(int levels, int K, int variant, long long* out, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  double* ring = (double*)smem;
  int* slot = (int*)(smem + 65536);
  double* val = (double*)(smem + 65536 + 16384);
  const int t = threadIdx.x;
  for (int i = t; i < 8192; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
  for (int i = t; i < 8 * 512; i += blockDim.x) { slot[i] = (i * 2654435761u) & 8191; val[i] = 1e-3 * (i & 7); }
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int l = 0; l < levels; ++l) {
    double a = ring[(l * 37 + t) & 8191];
    if (!(variant & 2)) {
      int sl[8]; double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) if (k < K) { sl[k] = slot[k * 512 + t]; v[k] = val[k * 512 + t]; }
      double zz[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) if (k < K) zz[k] = ring[sl[k]];
#pragma unroll
      for (int k = 0; k < 8; ++k) if (k < K) a = a - v[k] * zz[k];
    }
    if (!(variant & 4)) ring[(l * 512 + t) & 8191] = a;
    acc += a;
    if (!(variant & 1)) asm volatile("bar.sync 1, 512;" ::: "memory");
  }
  long long t1 = clock64();
  if (t == 0) out[0] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
  int smem = 65536 + 16384 + 32768 + 128;
  cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int v : {0, 1, 2, 3, 4, 6, 7})
    for (int K : {1, 8}) {
      lk<<<1, 512, smem>>>(10000, K, v, out, sink);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("variant %d (nobar=%d nofold=%d nosts=%d) K %d : %6.1f cycles/level\n", v, v & 1, (v >> 1) & 1, (v >> 2) & 1, K, c / 10000.0);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
