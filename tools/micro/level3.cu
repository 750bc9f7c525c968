#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// loop: a = ring[(l*37+t)&mask]; acc += a   (double), various warps / smem sizes
__global__ void lk(int levels, int mask, long long* out, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  double* ring = (double*)smem;
  const int t = threadIdx.x;
  for (int i = t; i <= mask; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int l = 0; l < levels; ++l) acc += ring[(l * 37 + t) & mask];
  long long t1 = clock64();
  if (t == 0) out[0] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}
__global__ void lkf(int levels, int mask, long long* out, float* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* ring = (float*)smem;
  const int t = threadIdx.x;
  for (int i = t; i <= mask; i += blockDim.x) ring[i] = 1.0f + i * 1e-6f;
  __syncthreads();
  long long t0 = clock64();
  float acc = 0;
  for (int l = 0; l < levels; ++l) acc += ring[(l * 37 + t) & mask];
  long long t1 = clock64();
  if (t == 0) out[0] = t1 - t0;
  if (acc == 12345.0f) sink[0] = acc;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(lkf, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int th : {32, 128, 512})
    for (int sm : {16384, 131072}) {
      int mask = sm / 8 - 1;
      cudaEventRecord(e0);
      lk<<<1, th, sm>>>(100000, mask, out, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("double threads %3d smem %6d: %6.1f cyc/iter, %6.2f ns/iter (wall)\n", th, sm, c / 1e5, ms * 1e6 / 1e5);
      lkf<<<1, th, sm>>>(100000, sm / 4 - 1, out, (float*)sink);
      cudaDeviceSynchronize();
      cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("float  threads %3d smem %6d: %6.1f cyc/iter\n", th, sm, c / 1e5);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
