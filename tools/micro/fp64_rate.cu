// FP64 vs FP32 issue throughput per SM: 512 threads x 8 independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int OP>
__global__ void k(int iters, T seed, long long* out, T* sink) {
  T a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + (T)(threadIdx.x + j);
  const T m = (T)1.0000001, c = (T)1e-7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = a[j] + c;
      if (OP == 1) a[j] = a[j] * m;
      if (OP == 2) a[j] = fma(a[j], m, c);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == (T)12345) sink[0] = s;
}
template <typename T, int OP>
void run(const char* name, int threads) {
  long long* out; T* sink;
  cudaMalloc(&out, 8 * 1024); cudaMalloc(&sink, 64);
  const int iters = 4096;
  k<T, OP><<<1, threads>>>(iters, (T)1, out, sink);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
  double ops = (double)iters * 8 * threads;
  printf("%-10s threads %4d: %7.2f ops/clk/SM  (%.2f cycles per warp-instr per SMSP)\n", name, threads, ops / c,
         (double)c / ((double)iters * 8 * threads / 32 / 4));
  cudaFree(out); cudaFree(sink);
}
int main() {
  for (int th : {32, 128, 512}) {
    run<double, 0>("DADD", th);
    run<double, 1>("DMUL", th);
    run<double, 2>("DFMA", th);
    run<float, 0>("FADD", th);
    run<float, 2>("FFMA", th);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
