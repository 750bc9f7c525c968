// Per-SM streaming bandwidth: TMA bulk ring vs plain LDG with many loads in flight,
// 1, 32, 148 and 296 CTAs (296: two per SM), 8 MB per CTA from HBM (buffer >> L2 in total).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void tma_kernel(const uint8_t* src, size_t per_cta, int nst, int sb, double* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 16;
  uint8_t* st = smem + 256;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const int nchunk = (int)(per_cta / sb);
  const int nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(nw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x >= nw * 32) {
    if (threadIdx.x != nw * 32) return;
    for (int u = 0; u < nchunk; ++u) {
      const int s = u % nst;
      if (u >= nst) {
        const uint32_t par = ((u / nst) - 1) & 1;
        asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(sa(&empty[s])), "r"(par) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(sb) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(st + (size_t)s * sb)), "l"(base + (size_t)u * sb), "r"(sb), "r"(sa(&full[s])) : "memory");
    }
    return;
  }
  double acc = 0;
  for (int u = 0; u < nchunk; ++u) {
    const int s = u % nst;
    const uint32_t par = (u / nst) & 1;
    asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(sa(&full[s])), "r"(par) : "memory");
    acc += ((const double*)(st + (size_t)s * sb))[threadIdx.x];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
  }
  if (acc == 1234.5) sink[0] = acc;
}
template <int D>
__global__ void ldg_kernel(const uint8_t* src, size_t per_cta, double* sink) {
  const double2* p = (const double2*)(src + (size_t)blockIdx.x * per_cta);
  const size_t n = per_cta / 16;
  double acc = 0;
  for (size_t i0 = threadIdx.x; i0 < n; i0 += (size_t)D * blockDim.x) {
    double2 v[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const size_t i = i0 + (size_t)d * blockDim.x;
      v[d] = i < n ? __ldcs(p + i) : make_double2(0, 0);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) acc += v[d].x + v[d].y;
  }
  if (acc == 1234.5) sink[0] = acc;
}
int main() {
  const size_t per = 8u << 20;
  uint8_t* src;
  double* sink;
  cudaMalloc(&src, per * 296);
  cudaMemset(src, 0, per * 296);
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch, int ctas) {
    launch(ctas);
    cudaEventRecord(e0);
    launch(ctas);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return (double)per / (ms * 1e-3) / 1e9;
  };
  for (int ctas : {1, 32, 148, 296}) {
    for (int sb : {16384, 24576, 32768, 49152}) {
      for (int nst : {4, 6}) {
        int smem = 256 + sb * nst;
        if (smem > 227 * 1024 || (ctas == 296 && smem > 113 * 1024)) continue;
        cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        double g = timeit([&](int c) { tma_kernel<<<c, 512, smem>>>(src, per, nst, sb, sink); }, ctas);
        printf("ctas %3d TMA sb %6d nst %d (%3d KB in flight): %6.1f GB/s per CTA, %7.0f GB/s total\n", ctas, sb, nst, sb * nst / 1024, g, g * ctas);
      }
    }
    double g;
    g = timeit([&](int c) { ldg_kernel<8><<<c, 512>>>(src, per, sink); }, ctas);
    printf("ctas %3d LDG 512x8x16B (64 KB in flight): %6.1f GB/s per CTA, %7.0f GB/s total\n", ctas, g, g * ctas);
    g = timeit([&](int c) { ldg_kernel<16><<<c, 512>>>(src, per, sink); }, ctas);
    printf("ctas %3d LDG 512x16x16B (128 KB in flight): %6.1f GB/s per CTA, %7.0f GB/s total\n", ctas, g, g * ctas);
    g = timeit([&](int c) { ldg_kernel<16><<<c, 1024>>>(src, per, sink); }, ctas);
    printf("ctas %3d LDG 1024x16x16B (256 KB in flight): %6.1f GB/s per CTA, %7.0f GB/s total\n", ctas, g, g * ctas);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
