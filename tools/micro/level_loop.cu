// Microbenchmark: cost of one dependency level in the streamed-solve structure:
// 16 consumer warps, each thread folds K entries gathered from shared memory (slot ->
// ring), writes the ring, then a named barrier; optional spinning producer warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NT = 512;
__global__ void level_kernel(int levels, int K, int producer_mode, int nrows, long long* out, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  double* ring = (double*)smem;           // 8192 doubles
  int* slot = (int*)(smem + 65536);       // 8 * 512 ints
  double* val = (double*)(smem + 65536 + 16384);  // 8 * 512 doubles
  const int t = threadIdx.x;
  for (int i = t; i < 8192; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
  for (int i = t; i < 8 * 512; i += blockDim.x) { slot[i] = (i * 2654435761u) & 8191; val[i] = 1e-3 * (i & 7); }
  __syncthreads();
  if (t >= NT) {
    if (producer_mode == 1 && t == NT) {
      volatile int* flag = (int*)(smem + 65536 + 16384 + 32768);
      while (*flag == 0) __nanosleep(32);
    }
    return;
  }
  long long t0 = clock64();
  double acc = 0;
  for (int l = 0; l < levels; ++l) {
    if (t < nrows) {
      double a = ring[(l * 37 + t) & 8191];
      int sl[8]; double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) if (k < K) { sl[k] = slot[k * 512 + t]; v[k] = val[k * 512 + t]; }
      double zz[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) if (k < K) zz[k] = ring[sl[k]];
#pragma unroll
      for (int k = 0; k < 8; ++k) if (k < K) a = a - v[k] * zz[k];
      ring[(l * 512 + t) & 8191] = a;
      acc += a;
    }
    asm volatile("bar.sync 1, 512;" ::: "memory");
  }
  long long t1 = clock64();
  if (t == 0) { out[0] = t1 - t0; volatile int* flag = (int*)(smem + 65536 + 16384 + 32768); *flag = 1; }
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
  int smem = 65536 + 16384 + 32768 + 128;
  cudaFuncSetAttribute(level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int pm = 0; pm < 2; ++pm)
    for (int K : {1, 4, 8})
      for (int nrows : {32, 512}) {
        int threads = pm ? NT + 32 : NT;
        cudaMemset(sink, 0, 8);
        // reset flag region via a clean launch each time (smem is per launch)
        level_kernel<<<1, threads, smem>>>(10000, K, pm, nrows, out, sink);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
        printf("producer %d K %d rows %3d : %6.1f cycles/level  (%s)\n", pm, K, nrows, c / 10000.0,
               cudaGetErrorString(cudaGetLastError()));
      }
}
