// Cost of the producer's per-chunk issue sequence on one thread (no consumers):
// mode bits: 1 = second (rhs) bulk copy per chunk, 2 = cp.async descriptor fetch + wait_group 11,
// 4 = placement record store before the arrive, 8 = 128-B misaligned rhs source.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint8_t* src, int nchunk, int sb, int rb, int mode, long long* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem;        // 16
  uint4* dq = (uint4*)(smem + 256);        // 16
  int2* pos = (int2*)(smem + 512);         // 16
  uint8_t* ring = smem + 1024;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 16; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(sa(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const uint4* descs = (const uint4*)src;
  long long t0 = clock64();
  for (int u = 0; u < nchunk; ++u) {
    const int s = u & 15;
    if (u >= 16) {  // slot reuse: wait for the copy 16 chunks ago
      const uint32_t par = ((u >> 4) - 1) & 1;
      asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(sa(&full[s])), "r"(par) : "memory");
    }
    if (mode & 2) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa(&dq[(u + 12) & 15])), "l"(descs + u + 12) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 11;" ::: "memory");
    }
    const uint32_t at = (uint32_t)(s & 3) * (sb + 8192);
    if (mode & 4) pos[s] = make_int2((int)at, (int)(at + sb));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(sb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(ring + at)), "l"(src + 4096 + (size_t)(u % 64) * sb), "r"(sb), "r"(sa(&full[s])) : "memory");
    if (mode & 1) {
      const size_t roff = (mode & 8) ? 16 : 0;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(rb) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(ring + at + sb)), "l"(src + (64 << 20) + roff + (size_t)(u % 64) * rb), "r"(rb), "r"(sa(&full[s])) : "memory");
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&full[s])) : "memory");
    }
  }
  long long t1 = clock64();
  out[0] = t1 - t0;
}
int main() {
  uint8_t* src;
  long long* out;
  cudaMalloc(&src, 128 << 20);
  cudaMemset(src, 0, 128 << 20);
  cudaMalloc(&out, 8);
  const int sb = 24576, rb = 4096, n = 2000;
  const int smem = 1024 + 4 * (sb + 8192);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode : {0, 1, 2, 4, 3, 7, 15}) {
    k<<<1, 32, smem>>>(src, n, sb, rb, mode, out);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("mode %2d: %7.1f cycles per chunk (%.1f GB/s at 1.965 GHz) %s\n", mode, (double)c / n,
           (double)(sb + ((mode & 1) ? rb : 0)) * n / (c / 1.965e9) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
