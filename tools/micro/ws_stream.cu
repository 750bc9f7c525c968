// Warp-specialised TMA pipeline microbenchmark (the structure of subdomain_step_kernel):
// 16 consumer warps + 1 producer warp, full/empty mbarriers, optional second (rhs) bulk copy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool test(uint64_t* b, uint32_t par) {
  uint32_t ok; asm volatile("{\n .reg .pred P1;\n mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0,1,0,P1;\n}\n" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory"); return ok; }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(sa(b)), "r"(par) : "memory"); }
__device__ __forceinline__ void exptx(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory"); }
__global__ void k(const uint8_t* src, const double* rsrc, size_t per_cta, int nst, int sb, int rb, int mode, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem; uint64_t* empty = full + 8;
  uint8_t* st = smem + 256; uint8_t* rst = st + (size_t)nst * sb;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const double* rbase = rsrc + (size_t)blockIdx.x * (per_cta / 4);
  int nchunk = (int)(per_cta / sb);
  int arrivals = (mode & 1) ? 2 : 1;
  if (threadIdx.x == 0) { for (int s = 0; s < nst; ++s) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[s])), "r"(arrivals)); asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(sa(&empty[s]))); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x >= 512) {
    if ((threadIdx.x & 31) == 0) {
      for (int u = 0; u < nchunk; ++u) {
        int s = u % nst, use = u / nst;
        if (use) while (!test(&empty[s], (use - 1) & 1)) { if (mode & 2) __nanosleep(32); }
        exptx(&full[s], sb); bulk(st + (size_t)s * sb, base + (size_t)u * sb, sb, &full[s]);
        if (mode & 1) { exptx(&full[s], rb); bulk(rst + (size_t)s * rb, rbase + (size_t)u * (rb / 8), rb, &full[s]); }
      }
    }
    return;
  }
  double acc = 0;
  for (int u = 0; u < nchunk; ++u) {
    int s = u % nst;
    wait(&full[s], (u / nst) & 1);
    acc += ((const double*)(st + (size_t)s * sb))[threadIdx.x];
    if (mode & 4) asm volatile("bar.sync 1, 512;" ::: "memory");
    __syncwarp();
    if ((threadIdx.x & 31) == 0) arrive(&empty[s]);
  }
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  size_t total = (size_t)1 << 30; uint8_t* buf; double* rbuf; double* sink;
  cudaMalloc(&buf, total); cudaMemset(buf, 1, total); cudaMalloc(&rbuf, total / 4 + 4096); cudaMemset(rbuf, 0, total / 4); cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode : {0, 1, 2, 3, 4, 5, 7})
    for (int nst : {4, 5}) {
      int sb = 32768, rb = 8192;
      int smem = 256 + nst * (sb + rb);
      size_t per = (size_t)16 << 20;
      k<<<32, 544, smem>>>(buf, rbuf, per, nst, sb, rb, mode, sink);
      cudaEventRecord(a);
      k<<<32, 544, smem>>>(buf, rbuf, per, nst, sb, rb, mode, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("mode %d (rhs=%d sleep=%d levelbar=%d) nst %d: %7.1f GB/s per CTA, %.3f us/chunk\n", mode, mode & 1, (mode >> 1) & 1, (mode >> 2) & 1, nst,
             per / (ms * 1e-3) / 1e9, ms * 1e3 / (per / sb));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
