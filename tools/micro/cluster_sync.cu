// Per-iteration cost of CTA-pair synchronisation (cluster of 2) vs a CTA barrier:
//  mode 0: bar.sync (512 threads) per iteration
//  mode 1: remote DSMEM store + barrier.cluster.arrive.release / wait.acquire
//  mode 2: remote DSMEM store + mbarrier handshake: each warp's lane 0 arrives (release.cluster)
//          on the partner's mbarrier and on its own; threads wait on the local one
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(2, 1, 1) k(int iters, int mode, long long* out, double* sink) {
  __shared__ double ring[4096];
  __shared__ __align__(8) uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank(), peer = me ^ 1;
  const int t = threadIdx.x;
  for (int i = t; i < 4096; i += blockDim.x) ring[i] = i;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(2 * (blockDim.x / 32)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  double* rring = cl.map_shared_rank(ring, peer);
  uint64_t* rbar = cl.map_shared_rank(&bar, peer);
  double acc = 0;
  uint32_t par = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const double v = ring[(it * 37 + t) & 4095];
    acc += v;
    if (mode == 0) {
      ring[(it * 512 + t + 2048) & 4095] = acc;
      asm volatile("bar.sync 0;" ::: "memory");
    } else if (mode == 1) {
      ring[(it * 512 + t + 2048) & 4095] = acc;
      rring[(it * 512 + t + 2048) & 4095] = acc;
      asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      ring[(it * 512 + t + 2048) & 4095] = acc;
      rring[(it * 512 + t + 2048) & 4095] = acc;
      __syncwarp();
      if ((t & 31) == 0) {
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(sa(&bar)), "r"(peer));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
      }
      asm volatile(
          "{\n .reg .pred P;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}\n" ::"r"(sa(&bar)),
          "r"(par)
          : "memory");
      par ^= 1;
    }
  }
  long long t1 = clock64();
  if (t == 0 && me == 0) out[mode] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
  (void)rbar;
  cl.sync();
}

int main() {
  long long* out; double* sink;
  cudaMalloc(&out, 64); cudaMalloc(&sink, 8);
  for (int mode = 0; mode < 3; ++mode) {
    k<<<2, 512>>>(20000, mode, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, out + mode, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %7.1f cycles/iteration (%s)\n", mode, c / 20000.0, cudaGetErrorString(e));
  }
  return 0;
}
