// Per-SM TMA stream with the step kernel's protocol: 15 consumer warps wait on full[s]
// and each arrives on empty[s]; one producer thread polls empty[] (test_wait +
// nanosleep) or blocks on it (try_wait), or the last consumer warp issues the refill.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ bool test(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n .reg .pred P1;\n mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  return ok;
}
constexpr int NC = 15;  // consumer warps
__global__ void k(const uint8_t* src, size_t per_cta, int nst, int sb, int mode, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 8;
  int* cnt = (int*)(empty + 8);
  uint8_t* st = smem + 1024;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const int nchunk = (int)(per_cta / sb);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(NC));
      cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int u) {
    int s = u % nst;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(sb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(st + (size_t)s * sb)), "l"(base + (size_t)u * sb), "r"(sb), "r"(sa(&full[s])) : "memory");
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == NC) {  // producer warp
    if (lane != 0 || mode == 2) return;
    for (int u = 0; u < nchunk; ++u) {
      const int s = u % nst;
      if (u >= nst) {
        const uint32_t par = ((u / nst) - 1) & 1;
        if (mode == 0) { while (!test(&empty[s], par)) __nanosleep(20); }
        else wait(&empty[s], par);
      }
      issue(u);
    }
    return;
  }
  if (mode == 2 && threadIdx.x == 0) for (int u = 0; u < nst && u < nchunk; ++u) issue(u);
  double acc = 0;
  for (int u = 0; u < nchunk; ++u) {
    const int s = u % nst;
    wait(&full[s], (u / nst) & 1);
    acc += ((const double*)(st + (size_t)s * sb))[threadIdx.x];
    __syncwarp();
    if (lane == 0) {
      if (mode == 2) {
        if (atomicAdd(&cnt[s], 1) == NC - 1) {
          cnt[s] = 0;
          if (u + nst < nchunk) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(u + nst); }
        }
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
      }
    }
  }
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  size_t total = (size_t)1 << 30;
  uint8_t* buf; double* sink;
  cudaMalloc(&buf, total); cudaMemset(buf, 1, total); cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int ctas = 32;
  for (int pad : {0, 1})
  for (int mode = 0; mode < 2; ++mode)
    for (int sb : {25600, 32768}) for (int nst : {4}) {
      int smem = pad ? 227 * 1024 : 1024 + nst * sb;
      if (smem > 227 * 1024) continue;
      size_t per = (size_t)16 << 20;
      k<<<ctas, 512, smem>>>(buf, per, nst, sb, mode, sink);
      cudaEventRecord(a);
      k<<<ctas, 512, smem>>>(buf, per, nst, sb, mode, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("pad %d mode %d (%s) sb %6d nst %d : %6.1f GB/s per CTA\n", pad, mode, mode == 0 ? "poll" : mode == 1 ? "block" : "last-warp", sb, nst, (double)per / (ms * 1e-3) / 1e9);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
