// Microbenchmark: per-SM streaming bandwidth of cp.async.bulk (TMA 1D) with a
// multi-stage smem ring, one CTA per SM, like the PSLR streamed triangular solve.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void stream_kernel(const uint8_t* src, size_t per_cta, int nst, int sb, double* sink, int mis) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem;
  uint8_t* st = smem + 128;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  int nchunk = (int)(per_cta / sb);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int u) {
    int s = u % nst;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(sb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(st + (size_t)s * sb)), "l"(base + (size_t)u * sb + mis), "r"(sb), "r"(sa(&full[s])) : "memory");
  };
  if (threadIdx.x == 0) for (int u = 0; u < nst && u < nchunk; ++u) issue(u);
  double acc = 0;
  for (int u = 0; u < nchunk; ++u) {
    int s = u % nst;
    uint32_t par = (u / nst) & 1;
    asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(sa(&full[s])), "r"(par) : "memory");
    acc += ((const double*)(st + (size_t)s * sb))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && u + nst < nchunk) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(u + nst); }
  }
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  size_t total = (size_t)2 << 30;  // 2 GiB buffer
  uint8_t* buf; double* sink;
  cudaMalloc(&buf, total); cudaMemset(buf, 1, total); cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int ctas_list[] = {32};
  int sbs[] = {32768};
  int nsts[] = {4};
  for (int mis : {0, 16, 64, 112})
  for (int ctas : ctas_list)
    for (int sb : sbs)
      for (int nst : nsts) {
        int smem = 128 + nst * sb;
        if (smem > 227 * 1024) continue;
        size_t per = (size_t)(total / ctas) / sb * sb;
        if (per > (size_t)64 << 20) per = (size_t)64 << 20;
        stream_kernel<<<ctas, 512, smem>>>(buf, per - 4096, nst, sb, sink, mis);
        cudaEventRecord(a);
        stream_kernel<<<ctas, 512, smem>>>(buf, per - 4096, nst, sb, sink, mis);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double gbs = (double)per * ctas / (ms * 1e-3) / 1e9;
        printf("mis %3d ctas %3d sb %6d nst %d : %8.1f GB/s total, %6.1f GB/s per CTA\n", mis, ctas, sb, nst, gbs, gbs / ctas);
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
