// Latency microbenchmarks on B200: named barrier (16 warps), dependent LDS chain,
// dependent DADD chain, DMUL+DADD chain.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_bar(int n, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 512;" ::: "memory");
  if (threadIdx.x == 0) out[0] = clock64() - t0;
}
__global__ void k_lds(int n, long long* out, int* sink) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = s[p];
  if (threadIdx.x == 0) out[0] = clock64() - t0;
  if (p == -1) sink[0] = p;
}
__global__ void k_dadd(int n, long long* out, double* sink) {
  double a = threadIdx.x * 1e-3, b = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a - b;
  if (threadIdx.x == 0) out[0] = clock64() - t0;
  if (a == 12345.0) sink[0] = a;
}
__global__ void k_dmuladd(int n, long long* out, double* sink) {
  double a = threadIdx.x * 1e-3, b = 1e-9, c = 0.999;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a - b * a;
  if (threadIdx.x == 0) out[0] = clock64() - t0;
  if (a == 12345.0) sink[0] = a;
}
__global__ void k_sts_bar(int n, long long* out) {
  __shared__ double s[1024];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { s[(i * 512 + threadIdx.x) & 1023] = i; asm volatile("bar.sync 1, 512;" ::: "memory"); }
  if (threadIdx.x == 0) out[0] = clock64() - t0;
}
int main() {
  long long* out; double* ds; int* is; cudaMalloc(&out, 8); cudaMalloc(&ds, 8); cudaMalloc(&is, 8);
  long long c; int n = 10000;
  k_bar<<<1, 512>>>(n, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("bar.sync 512 thr: %.1f cyc\n", c / (double)n);
  cudaDeviceSynchronize();
  k_sts_bar<<<1, 512>>>(n, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("STS+bar.sync: %.1f cyc\n", c / (double)n);
  k_lds<<<1, 32>>>(n, out, is); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("dep LDS chain (1 warp): %.1f cyc\n", c / (double)n);
  k_lds<<<1, 512>>>(n, out, is); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("dep LDS chain (16 warps): %.1f cyc\n", c / (double)n);
  k_dadd<<<1, 32>>>(n, out, ds); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("dep DADD chain (1 warp): %.1f cyc\n", c / (double)n);
  k_dadd<<<1, 512>>>(n, out, ds); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("dep DADD chain (16 warps): %.1f cyc\n", c / (double)n);
  k_dmuladd<<<1, 32>>>(n, out, ds); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("dep DMUL+DADD chain (1 warp): %.1f cyc\n", c / (double)n);
  k_dmuladd<<<1, 512>>>(n, out, ds); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("dep DMUL+DADD chain (16 warps): %.1f cyc\n", c / (double)n);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
