// Isolate the cost of the fold step in a 512-thread level loop (one CTA).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void lk(int levels, int variant, long long* out, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  double* ring = (double*)smem;
  int* slot = (int*)(smem + 65536);
  double* val = (double*)(smem + 65536 + 16384);
  const int t = threadIdx.x;
  for (int i = t; i < 8192; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
  for (int i = t; i < 8 * 512; i += blockDim.x) {
    slot[i] = (variant & 16) ? ((i & 511) + 1024) : (int)((i * 2654435761u) & 8191);
    val[i] = 1e-3 * (i & 7);
  }
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int l = 0; l < levels; ++l) {
    double a = ring[(l * 37 + t) & 8191];
    const int sl = (variant & 1) ? t : ((variant & 2) ? ((t * 37 + l) & 8191) : slot[t]);
    const double v = val[t];
    const double zz = ring[sl];
    if (variant & 4) a = a + zz;          // no multiply
    else if (variant & 8) a = zz;         // no FP at all
    else a = a - v * zz;
    ring[(l * 512 + t + 4096) & 8191] = a;
    acc += a;
    asm volatile("bar.sync 1;" ::: "memory");
  }
  long long t1 = clock64();
  if (t == 0) out[0] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 8); cudaMalloc(&sink, 8);
  int smem = 65536 + 16384 + 32768 + 128;
  cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm[] = {"full", "sl=t", "sl=arith", "", "no-mul", "", "", "", "no-fp"};
  for (int v : {0, 1, 2, 4, 8, 16, 16 + 8})
    for (int th : {32, 512}) {
      lk<<<1, th, smem>>>(10000, v, out, sink);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("variant %2d %-9s threads %3d: %6.1f cycles/level\n", v, (v & 16) ? "seq-slots" : nm[v], th, c / 10000.0);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
