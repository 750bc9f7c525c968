// step_kernel.cu — the fused per-subdomain PSLR step kernel (sm_100a).
//
// One CTA per subdomain runs the whole per-subdomain chain of one launch:
//   interior phase:  xb = B_b^{-1} (b1 (-) b2)         (E folded into the right-hand side)
//   interface phase: w = i1 (+|-) i2 ; y = [C0_b^{-1}] w [+ cadd] ; [partials = V_b^T y]
// Only Cg couples subdomains and it reads a vector produced by a previous launch, so
// one launch per Horner step is the only grid-wide synchronisation.
//
// Warp-specialised: 16 consumer warps walk the dependency levels (thread t owns row t
// of each packed segment; named barrier 1 separates levels), one producer warp streams
// the packed factors (pack.cpp) through an nst-stage shared-memory pipeline with TMA
// bulk copies (cp.async.bulk + full/empty mbarriers) and runs bulk L2 prefetches
// further ahead.  Each chunk also brings its rows' right-hand sides (a contiguous
// slice of the position-ordered rhs array) with a second bulk copy on the same
// mbarrier, issued once the consumers signal that the phase's rhs is final.
// Solution values live in a shared-memory ring indexed by level-order position.
//
// Arithmetic contract (bit-exact with scipy, library built with -fmad=false):
//   L: z_i = b_i - L_ij z_j ... (ascending j);  U: z_i = b_i/sd_i - U'_ij z_j ..., x_i = z_i*invd_i.
#include <cuda_runtime.h>

#include "pslr_internal.h"

namespace pslr {

constexpr int kConsumerWarps = kStepThreads / 32;
constexpr int kBlockThreads = kStepThreads + 32;  // + one producer warp
constexpr int kL2Ahead = 8 * 32 * 1024;           // bytes prefetched into L2 beyond the smem stages
constexpr int kBatch = 8;                          // entries gathered per batch in the row loop

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      " selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// barrier among the consumer warps only (the producer warp never joins)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kStepThreads) : "memory");
}

__device__ __forceinline__ int A4(int x) { return (x + 3) & ~3; }
__device__ __forceinline__ int A2(int x) { return (x + 1) & ~1; }

// SpMV row over read-only inputs (the matrix and a vector produced by an earlier launch)
__device__ __forceinline__ double spmv_row_ro(const DevCsr& M, int row, const double* __restrict__ x) {
  double s = 0.0;
  const int e0 = __ldg(M.ptr + row), e1 = __ldg(M.ptr + row + 1);
  for (int e = e0; e < e1; ++e) s = s + __ldg(M.val + e) * __ldg(x + __ldg(M.col + e));
  return s;
}
// SpMV row over a vector written earlier in this launch (no read-only cache path)
__device__ __forceinline__ double spmv_row_rw(const DevCsr& M, int row, const double* x) {
  double s = 0.0;
  const int e0 = __ldg(M.ptr + row), e1 = __ldg(M.ptr + row + 1);
  for (int e = e0; e < e1; ++e) s = s + __ldg(M.val + e) * x[__ldg(M.col + e)];
  return s;
}

// Optional timeline of one CTA (PSLR_TRACE=1): (code<<32|arg, %globaltimer ns) pairs.
// Thread 0 of CTA 0 reserves a window with one atomic per launch, then stores plainly.
__shared__ long long* g_trace_ptr;
__shared__ int g_trace_n;
constexpr int kTraceWindow = 1 << 15;

__device__ __forceinline__ void trace_begin(const StepConst& K) {
  if (K.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long i =
        atomicAdd(reinterpret_cast<unsigned long long*>(K.trace), (unsigned long long)kTraceWindow);
    g_trace_ptr = (i + kTraceWindow <= (unsigned long long)K.trace_cap) ? K.trace + 2 + 2 * i : nullptr;
    g_trace_n = 0;
  }
}
__device__ __forceinline__ void trace_ev(const StepConst& K, int code, int arg) {
  if (K.trace && blockIdx.x == 0 && threadIdx.x == 0 && g_trace_ptr && g_trace_n < kTraceWindow) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    g_trace_ptr[2 * g_trace_n] = ((long long)code << 32) | (unsigned)arg;
    g_trace_ptr[2 * g_trace_n + 1] = (long long)ns;
    ++g_trace_n;
  }
}

// Shared-memory control block
struct Ctl {
  uint64_t full[8];       // data + rhs landed (2 arrivals + tx bytes)
  uint64_t empty[8];      // all consumer warps done with the stage (kConsumerWarps arrivals)
  uint64_t rhs_ready[4];  // phase k's rhs array is final (1 arrival)
};

// The chunks of up to four factor streams of this CTA's block form one sequence.
struct Streams {
  int nphase;
  int begin[5];
  const uint8_t* data[4];
  const ChunkDesc* chunks[4];  // this block's first chunk of the phase
  const double* rhs[4];        // position-ordered right-hand-side array of each phase

  __device__ __forceinline__ int phase_of(int u) const {
    int k = 0;
    while (k + 1 < nphase && u >= begin[k + 1]) ++k;
    return k;
  }
  __device__ __forceinline__ ChunkDesc desc(int u) const {
    const int k = phase_of(u);
    return chunks[k][u - begin[k]];
  }
};

// Producer: lane 0 of the producer warp.
// Descriptors of 32 consecutive chunks held one per lane of the producer warp, so the
// producer pays one global-load latency per 32 chunks instead of one per chunk.
struct DescCache {
  int base = -(1 << 30);
  ChunkDesc mine{};
  __device__ __forceinline__ ChunkDesc get(const Streams& S, int u, int total) {
    const int lane = threadIdx.x & 31;
    if (u < base || u >= base + 32) {
      base = u;
      const int v = u + lane;
      if (v < total) mine = S.desc(v);
    }
    const int src = u - base;
    ChunkDesc d;
    d.off = __shfl_sync(0xffffffffu, mine.off, src);
    d.bytes = __shfl_sync(0xffffffffu, mine.bytes, src);
    d.nseg = 0;
    d.pos0 = __shfl_sync(0xffffffffu, mine.pos0, src);
    d.npos = __shfl_sync(0xffffffffu, mine.npos, src);
    return d;
  }
};

// Producer: the whole producer warp runs the loop (warp-uniform decisions), lane 0
// issues the TMA operations.
__device__ void producer(const Streams& S, Ctl* ctl, uint8_t* stages, double* rhsbuf, int nst,
                         int stage_bytes, int rhs_stride) {
  const bool lead = (threadIdx.x & 31) == 0;
  const int total = S.begin[S.nphase];
  int data_next = 0, rhs_next = 0;
  bool ready[4] = {false, false, false, false};
  DescCache cd, cr;
  // L2 prefetch cursor over the block's contiguous byte range of each phase
  int pf_phase = 0;
  int64_t pf_off = 0, pf_end = 0;
  auto phase_range = [&](int k, int64_t& lo, int64_t& hi) {
    const int n = S.begin[k + 1] - S.begin[k];
    if (n <= 0) {
      lo = hi = 0;
      return;
    }
    const ChunkDesc a = S.chunks[k][0], z = S.chunks[k][n - 1];
    lo = a.off;
    hi = z.off + z.bytes;
  };
  if (S.nphase > 0) phase_range(0, pf_off, pf_end);
  int64_t issued_bytes = 0, prefetched_bytes = 0;
  int st_d = 0, use_d = 0;  // stage / use count of data_next
  int st_r = 0;             // stage of rhs_next
  while (rhs_next < total) {
    bool did = false;
    if (data_next < total && (use_d == 0 || mbar_test(&ctl->empty[st_d], (uint32_t)((use_d - 1) & 1)))) {
      const ChunkDesc d = cd.get(S, data_next, total);
      const int k = S.phase_of(data_next);
      if (lead) {
        mbar_expect_tx(&ctl->full[st_d], (uint32_t)d.bytes);
        bulk_load(stages + (size_t)st_d * stage_bytes, S.data[k] + d.off, (uint32_t)d.bytes,
                  &ctl->full[st_d]);
      }
      issued_bytes += d.bytes;
      ++data_next;
      if (++st_d == nst) {
        st_d = 0;
        ++use_d;
      }
      did = true;
    }
    if (rhs_next < data_next) {
      const int k = S.phase_of(rhs_next);
      if (!ready[k] && mbar_test(&ctl->rhs_ready[k], 0)) {
        ready[k] = true;
        fence_proxy_async();
      }
      if (ready[k]) {
        const ChunkDesc d = cr.get(S, rhs_next, total);
        const int p0 = d.pos0 & ~1;
        const int cnt = (d.pos0 + d.npos - p0 + 1) & ~1;
        if (lead) {
          mbar_expect_tx(&ctl->full[st_r], (uint32_t)(cnt * 8));
          bulk_load(rhsbuf + (size_t)st_r * rhs_stride, S.rhs[k] + p0, (uint32_t)(cnt * 8),
                    &ctl->full[st_r]);
        }
        ++rhs_next;
        if (++st_r == nst) st_r = 0;
        did = true;
      }
    }
    // keep ~kL2Ahead bytes of the stream prefetched into L2 beyond the issued chunks
    while (pf_phase < S.nphase && prefetched_bytes < issued_bytes + kL2Ahead) {
      if (pf_off >= pf_end) {
        if (++pf_phase < S.nphase) phase_range(pf_phase, pf_off, pf_end);
        continue;
      }
      const int64_t len = (pf_end - pf_off) < 32768 ? (pf_end - pf_off) : 32768;
      if (lead) bulk_prefetch_l2(S.data[pf_phase] + pf_off, (uint32_t)len);
      pf_off += len;
      prefetched_bytes += len;
    }
    if (!did) __nanosleep(32);
  }
}


// Process the segments of one staged chunk.  A segment holds at most kStepThreads rows;
// consumer thread t owns row t.  Slab k holds entry k of rows [0, cnt_k); rows are sorted
// by length, so a warp stops at the first slab its leading row does not reach.
template <bool UPPER>
__device__ __forceinline__ void run_chunk(const StepConst& K, const uint8_t* buf,
                                          const double* rbuf, double* ring, int mask, int base,
                                          double* z, double* xout, const double* __restrict__ cadd) {
  const int32_t* h0 = reinterpret_cast<const int32_t*>(buf);
  const int nseg = h0[6];
  const int rbase = h0[7];
  const int t = threadIdx.x;
  for (int s = 0; s < nseg; ++s) {
    const int32_t* h = reinterpret_cast<const int32_t*>(buf);
    const int nrows = h[0], w = h[1], flags = h[2], pos0 = h[3], S = h[4], bytes = h[5];
    if (t < nrows) {
      // ELL segment (pack.cpp): info[S], [U: sd[S], invd[S]], val[w][S], slot[w][S]
      const int32_t* info = h + 8;
      const uint8_t* p = reinterpret_cast<const uint8_t*>(info + S);
      const double* sd = nullptr;
      const double* invd = nullptr;
      if (UPPER) {
        sd = reinterpret_cast<const double*>(p);
        invd = sd + S;
        p = reinterpret_cast<const uint8_t*>(invd + S);
      }
      const double* val = reinterpret_cast<const double*>(p) + t;
      const int32_t* slot = reinterpret_cast<const int32_t*>(reinterpret_cast<const double*>(p) + w * S) + t;
      const int gp = pos0 + t;
      double acc = rbuf[gp - rbase];
      if (UPPER) {
        const double sdv = sd[t];
        if (sdv != 1.0) acc = acc / sdv;  // x / 1.0 == x exactly: skip the division
      }
      // Padding entries are exact no-ops (0 * ring[zero slot] = 0), so every lane runs the
      // segment-uniform w steps in the reference's ascending-column order.
      if (!(flags & 2)) {
        int k = 0;
        for (; k + 4 <= w; k += 4) {
          const int s0 = slot[(k + 0) * S], s1 = slot[(k + 1) * S];
          const int s2 = slot[(k + 2) * S], s3 = slot[(k + 3) * S];
          const double v0 = val[(k + 0) * S], v1 = val[(k + 1) * S];
          const double v2 = val[(k + 2) * S], v3 = val[(k + 3) * S];
          const double z0 = ring[s0], z1 = ring[s1], z2 = ring[s2], z3 = ring[s3];
          acc = acc - v0 * z0;
          acc = acc - v1 * z1;
          acc = acc - v2 * z2;
          acc = acc - v3 * z3;
        }
        for (; k < w; ++k) acc = acc - val[k * S] * ring[slot[k * S]];
      } else {
        for (int k = 0; k < w; ++k) {
          const int sl = slot[k * S];
          const double zz = (sl >= 0) ? ring[sl] : z[sl & 0x7fffffff];
          acc = acc - val[k * S] * zz;
        }
      }
      ring[(gp - base) & mask] = acc;
      if (UPPER) {
        z[gp] = acc;
        const int row = info[t];
        double x = acc * invd[t];
        if (cadd) x = x + __ldg(cadd + row);
        xout[row] = x;
      } else {
        z[info[t]] = acc;
      }
    }
    if (flags & 1) {
      trace_ev(K, 40, nrows | (w << 16));
      consumer_sync();
      trace_ev(K, 41, 0);
    }
    buf += bytes;
  }
}

// Consumer side of one triangular phase.  Callers arrive right after a consumer barrier
// that follows the last write of the phase's rhs array.
template <bool UPPER>
__device__ void tri_phase(const StepConst& K, const Streams& S, Ctl* ctl, uint8_t* stages,
                          double* rhsbuf, int k, double* ring, int base, double* z, double* xout,
                          const double* cadd) {
  trace_ev(K, 10 + k, 0);
  if (threadIdx.x == 0) {
    __threadfence();
    fence_proxy_async();
    mbar_arrive(&ctl->rhs_ready[k]);
  }
  const int nst = K.nst;
  const int lane = threadIdx.x & 31;
  int st = S.begin[k] % nst;
  uint32_t par = (uint32_t)((S.begin[k] / nst) & 1);
  for (int u = S.begin[k]; u < S.begin[k + 1]; ++u) {
    mbar_wait(&ctl->full[st], par);
    trace_ev(K, 20, u);
    run_chunk<UPPER>(K, stages + (size_t)st * K.stage_bytes, rhsbuf + (size_t)st * K.rhs_stride, ring,
                     K.ring_mask, base, z, xout, cadd);
    __syncwarp();
    if (lane == 0) mbar_arrive(&ctl->empty[st]);
    trace_ev(K, 21, u);
    if (++st == nst) {
      st = 0;
      par ^= 1u;
    }
  }
  consumer_sync();
}

// Four SpMV rows at once (independent gathers in flight): s[j] = sum_e M_ij x_j in CSR
// order from 0 (scipy csr_matvec).  RO: x is read-only for this launch.
template <bool RO>
__device__ __forceinline__ void spmv4(const DevCsr& M, const int (&row)[4], const bool (&ok)[4],
                                      const double* x, double (&s)[4]) {
  int e0[4], e1[4];
  int len = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    e0[j] = ok[j] ? __ldg(M.ptr + row[j]) : 0;
    e1[j] = ok[j] ? __ldg(M.ptr + row[j] + 1) : 0;
    s[j] = 0.0;
    len = max(len, e1[j] - e0[j]);
  }
  for (int k = 0; k < len; ++k) {
    int c[4];
    double v[4];
    bool on[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      on[j] = e0[j] + k < e1[j];
      c[j] = on[j] ? __ldg(M.col + e0[j] + k) : 0;
      v[j] = on[j] ? __ldg(M.val + e0[j] + k) : 0.0;
    }
    double xv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xv[j] = on[j] ? (RO ? __ldg(x + c[j]) : x[c[j]]) : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (on[j]) s[j] = s[j] + v[j] * xv[j];
  }
}

__device__ __forceinline__ void iface_terms4(int kind, const int (&row)[4], const bool (&ok)[4],
                                             const StepArgs& a, const StepConst& K, double (&t)[4]) {
  switch (kind) {
    case IT_G:
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = ok[j] ? __ldg(a.g + row[j]) : 0.0;
      break;
    case IT_FX: spmv4<false>(K.F, row, ok, a.xb, t); break;
    case IT_CY: spmv4<true>(K.C, row, ok, a.yC, t); break;
    case IT_CGY: spmv4<true>(K.Cg, row, ok, a.yC, t); break;
    default:
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = 0.0;
  }
}

__global__ void __launch_bounds__(kBlockThreads, 1)
subdomain_step_kernel(const __grid_constant__ StepArgs a, const __grid_constant__ StepConst K) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int b = blockIdx.x;
  const bool do_b = a.b1 != BT_NONE;
  const bool do_i = a.i1 != IT_NONE;
  const bool do_c = do_i && a.do_c0;

  Ctl* ctl = reinterpret_cast<Ctl*>(smem);
  uint8_t* stages = smem + 256;
  double* rhsbuf = reinterpret_cast<double*>(stages + (size_t)K.nst * K.stage_bytes);
  double* ring = rhsbuf + (size_t)K.nst * K.rhs_stride;

  Streams S;
  S.nphase = 0;
  S.begin[0] = 0;
  auto add_phase = [&](const DevTri& T, const double* rhs) {
    const int c0 = T.blk_chunk[b], c1 = T.blk_chunk[b + 1];
    S.data[S.nphase] = T.data;
    S.chunks[S.nphase] = T.chunks + c0;
    S.rhs[S.nphase] = rhs;
    S.begin[S.nphase + 1] = S.begin[S.nphase] + (c1 - c0);
    S.nphase++;
  };
  if (do_b) {
    add_phase(K.LB, K.rhsB);
    add_phase(K.UB, K.zB);
  }
  if (do_c) {
    add_phase(K.LC, K.rhsC);
    add_phase(K.UC, K.zC);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < K.nst; ++s) {
      mbar_init(&ctl->full[s], 2);
      mbar_init(&ctl->empty[s], kConsumerWarps);
    }
    for (int k = 0; k < 4; ++k) mbar_init(&ctl->rhs_ready[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= kStepThreads) {  // producer warp (all 32 lanes)
    producer(S, ctl, stages, rhsbuf, K.nst, K.stage_bytes, K.rhs_stride);
    return;
  }
  trace_begin(K);
  trace_ev(K, 1, S.begin[S.nphase]);
  if (threadIdx.x == 0) ring[K.ring_mask + 1] = 0.0;  // the zero slot (visible after the next barrier)
  const int ph_LB = 0, ph_UB = 1;
  const int ph_LC = do_b ? 2 : 0, ph_UC = do_b ? 3 : 1;
  const int tid = threadIdx.x;

  if (do_b) {
    const int r0 = K.int_off[b], r1 = K.int_off[b + 1];
    // pass 1: every row gets b1's f term (or 0); independent loads, 4 rows in flight
    for (int row0 = r0 + tid; row0 < r1; row0 += 4 * kStepThreads) {
      double v[4];
      int pos[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int row = row0 + j * kStepThreads;
        const bool ok = row < r1;
        v[j] = (ok && a.b1 == BT_F) ? __ldg(a.f + row) : 0.0;
        pos[j] = ok ? __ldg(K.LB.lpos + row) : 0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (row0 + j * kStepThreads < r1) K.rhsB[pos[j]] = v[j];
    }
    // pass 2: rows with E entries get the E y term: f - E y, or E y alone
    if (a.b1 == BT_EY || a.b2 == BT_EY) {
      consumer_sync();
      const int e0 = K.erow_off[b], e1 = K.erow_off[b + 1];
      for (int i0 = e0 + tid; i0 < e1; i0 += 4 * kStepThreads) {
        int row[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + j * kStepThreads;
          ok[j] = i < e1;
          row[j] = ok[j] ? __ldg(K.erows + i) : 0;
        }
        double s[4];
        spmv4<true>(K.E, row, ok, a.yE, s);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!ok[j]) continue;
          const double v = (a.b1 == BT_F) ? (__ldg(a.f + row[j]) - s[j]) : s[j];
          K.rhsB[__ldg(K.LB.lpos + row[j])] = v;
        }
      }
    }
    consumer_sync();
    trace_ev(K, 3, 0);
    tri_phase<false>(K, S, ctl, stages, rhsbuf, ph_LB, ring, r0, K.zB, nullptr, nullptr);
    tri_phase<true>(K, S, ctl, stages, rhsbuf, ph_UB, ring, r0, K.zB, a.xb, nullptr);
  }
  if (do_i) {
    const int r0 = K.ifc_off[b], r1 = K.ifc_off[b + 1];
    for (int row0 = r0 + tid; row0 < r1; row0 += 4 * kStepThreads) {
      int row[4];
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        row[j] = row0 + j * kStepThreads;
        ok[j] = row[j] < r1;
      }
      double w[4], t2[4];
      iface_terms4(a.i1, row, ok, a, K, w);
      if (a.i2 != IT_NONE) {
        iface_terms4(a.i2, row, ok, a, K, t2);
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = a.i2_sub ? (w[j] - t2[j]) : (w[j] + t2[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!ok[j]) continue;
        if (do_c) {
          K.rhsC[__ldg(K.LC.lpos + row[j])] = w[j];
        } else {
          double y = w[j];
          if (a.cadd) y = y + __ldg(a.cadd + row[j]);
          a.yout[row[j]] = y;
        }
      }
    }
    consumer_sync();
    trace_ev(K, 30, 0);
    if (do_c) {
      tri_phase<false>(K, S, ctl, stages, rhsbuf, ph_LC, ring, r0, K.zC, nullptr, nullptr);
      tri_phase<true>(K, S, ctl, stages, rhsbuf, ph_UC, ring, r0, K.zC, a.yout, a.cadd);
    }
  }
}

int configure_step_kernel(int smem_bytes) {
  return (int)cudaFuncSetAttribute(subdomain_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem_bytes);
}

int launch_step(const pslr_ctx* ctx, const StepArgs& a, cudaStream_t st) {
  if (ctx->s == 0) return 0;
  subdomain_step_kernel<<<(unsigned)ctx->s, kBlockThreads, ctx->K.smem_bytes, st>>>(a, ctx->K);
  return (int)cudaGetLastError();
}

}  // namespace pslr
