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

constexpr int kBlockThreads = kStepThreads + 32;  // + one producer warp (the launch bound)
// Consumer threads of a launch: a template parameter NT of the kernel (kStepThreads, or
// kNarrowThreads for systems of narrow levels: a cheaper level barrier, fewer idle warps
// walking the segment headers; StepConst::nthr, chosen per context by capi.cu); the block is
// launched with NT + 32 threads.  A compile-time count keeps the barrier's operand immediate
// (a runtime count cost the cfg5 apply 1.2 %).
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
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity);
// spin on test_wait (no hardware suspend): timing experiment PSLR_DBG bit 2048
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  while (!mbar_test(bar, parity)) {
  }
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
// the same copy with an L2 cache policy (createpolicy): the kept blocks' factor streams
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
// every consumer thread after writing a phase's right-hand-side array (global, generic
// proxy) and before the barrier after which the producer's TMA reads it (async proxy);
// a CTA-local ordering, unlike a GPU-scope membar
__device__ __forceinline__ void fence_rhs_written() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// barrier among the consumer warps only (the producer warp never joins)
template <int NT>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
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

// Optional timeline of one CTA: (code<<32|arg, %globaltimer ns) pairs, recorded only by a
// trace build (make EXTRA=-DPSLR_TRACE_BUILD=1) run with PSLR_TRACE=1; in the normal build
// trace_ev compiles to nothing (even a predicated-off check costs the level loop ~10
// instructions per call).  Thread 0 of CTA 0 reserves a window with one atomic per launch.
#ifndef PSLR_TRACE_BUILD
#define PSLR_TRACE_BUILD 0
#endif
__shared__ long long* g_trace_ptr;
__shared__ int g_trace_n;
__shared__ int g_trace_tag;
__shared__ long long g_wait_cyc;  // trace builds: thread 0's chunk-wait cycles / transitions
__shared__ int g_wait_n, g_wait_big;

constexpr int kTraceWindow = 1 << 15;

__device__ __forceinline__ void trace_begin(const StepConst& K) {
  if (PSLR_TRACE_BUILD && K.trace && blockIdx.x == K.trace_block && threadIdx.x == 0) {
    const unsigned long long i =
        atomicAdd(reinterpret_cast<unsigned long long*>(K.trace), (unsigned long long)kTraceWindow);
    g_trace_ptr = (i + kTraceWindow <= (unsigned long long)K.trace_cap) ? K.trace + 2 + 2 * i : nullptr;
    g_trace_n = 0;
  }
}
__device__ __forceinline__ void trace_ev(const StepConst& K, int code, int arg) {
  if (PSLR_TRACE_BUILD && K.trace && blockIdx.x == K.trace_block && threadIdx.x == 0 && g_trace_ptr &&
      g_trace_n < kTraceWindow) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    g_trace_ptr[2 * g_trace_n] = ((long long)code << 32) | (unsigned)arg;
    g_trace_ptr[2 * g_trace_n + 1] = (long long)ns;
    ++g_trace_n;
  }
}

// =3 builds: one (code|arg, clock64) record per level-loop step, cheap enough (no
// %globaltimer) to time individual levels in cycles
__device__ __forceinline__ void trace_clk(const StepConst& K, int code, int arg) {
  if (PSLR_TRACE_BUILD == 3 && K.trace && blockIdx.x == K.trace_block && threadIdx.x == 0 && g_trace_ptr &&
      g_trace_n < kTraceWindow) {
    g_trace_ptr[2 * g_trace_n] = ((long long)code << 32) | (unsigned)arg;
    g_trace_ptr[2 * g_trace_n + 1] = clock64();
    ++g_trace_n;
  }
}

// trace builds: every CTA stamps its phase boundaries (slot 0 start, 1 prepass done,
// 2..5 phase k start, 6 end) into row 1024 + 64 * (launch kind) + b of the counter area
// (the last launch of each kind wins; b < 64)
__device__ __forceinline__ void trace_cta(const StepConst& K, int slot) {
  if (PSLR_TRACE_BUILD && K.trace && threadIdx.x == 0 && K.trace_cap >= (1 << 20) && blockIdx.x < 64) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    K.trace[2 + 2 * K.trace_cap - 8 * 4096 + (1024 + 64 * (g_trace_tag & 15) + blockIdx.x) * 8 + slot] =
        (long long)ns;
  }
}

// per-chunk / per-level events: only in PSLR_TRACE_BUILD=2 builds (they perturb the level
// loop's timing; =1 records the phase boundaries only)
__device__ __forceinline__ void trace_fine(const StepConst& K, int code, int arg) {
  if (PSLR_TRACE_BUILD >= 2) trace_ev(K, code, arg);
}

// The kernel's dynamic shared memory (file scope: the level loop addresses staged
// segments by 32-bit offsets into it, which keeps its pointers in one register each)
extern __shared__ __align__(128) uint8_t smem[];
template <class T>
__device__ __forceinline__ const T* sp(uint32_t off) {
  return reinterpret_cast<const T*>(smem + off);
}

// Shared-memory control block
struct Ctl {
  uint4 dq[16];           // producer: descriptors of the next chunks (cp.async ring)
  uint64_t full[8];       // data + rhs landed (2 arrivals + tx bytes)
  uint64_t empty[8];      // all consumer warps done with the stage (kConsumerWarps arrivals)
  uint64_t rhs_ready[4];  // phase k's rhs array is final (1 arrival)
  int4 rrec[8];           // per stage: rhs slice (first position, bytes, offset in the stage) of its chunk
};

// The chunks of up to four factor streams of this CTA's block form one sequence.
struct Streams {
  int nphase;
  int begin[5];
  const uint8_t* data[4];
  const ChunkDesc* chunks[4];  // this block's first chunk of the phase
  const double* rhs[4];        // position-ordered right-hand-side array of each phase
  uint32_t pf_lo[4], pf_hi[4]; // byte range of this block's chunks in data[k] (L2 prefetch)
};

__device__ __forceinline__ ChunkDesc load_desc(const ChunkDesc* p) {
  const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
  ChunkDesc d;
  d.off16 = v.x;
  d.bytes = v.y;
  d.rpos = (int32_t)v.z;
  d.rbytes = v.w;
  return d;
}

static_assert(sizeof(Ctl) <= kCtlBytes, "the control block must fit the header of the shared memory plan");

// Producer: one thread (lane 0 of the producer warp) streams the chunks of the launch's
// phases, in order, into the nst stages with TMA bulk copies: chunk u's packed segments
// into stage u % nst, and its right-hand-side slice (a contiguous piece of the phase's
// position-ordered rhs array) into the stage's rhs buffer, both completing on full[st].
// A slice can only be copied once its phase's rhs is final (rhs_ready, signalled by the
// consumers at the phase start), so slices of chunks staged ahead of their phase are
// deferred and issued as soon as the phase is seen ready.
//
// The stream's rate is bounded by this ONE thread's dependent-instruction latency per
// chunk (measured: ~800 cycles per chunk for a loop that re-derived every quantity,
// i.e. ~55 GB/s per SM at 22 KB chunks): the steady-state path is a handful of
// instructions — poll the stage, read the next descriptor (prefetched into shared
// memory by cp.async twelve chunks ahead and into registers one chunk ahead), two
// expect_tx + bulk-copy pairs.  Phase bookkeeping only runs at phase boundaries.
__device__ void producer(const Streams& S, Ctl* ctl, uint8_t* stages, int nst,
                         int stage_bytes, int nv, long long* g_dbg_out, int dbg,
                         long long* g_tma, long long l2ahead, int keep) {
  if ((threadIdx.x & 31) != 0) return;
  const uint64_t pol = keep ? policy_evict_last() : 0ull;
  const int np = S.nphase;
  const int total = S.begin[np];
  if (total == 0) return;
  // descriptor queue: chunk u's 16-B descriptor is copied into ctl->dq[u & 15]
  int q_u = 0, q_k = 0, q_base = 0, q_end = S.begin[1];
  auto q_issue = [&]() {
    if (q_u < total) {
      while (q_u >= q_end) {
        ++q_k;
        q_base = S.begin[q_k];
        q_end = S.begin[q_k + 1];
      }
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_addr(&ctl->dq[q_u & 15])),
                   "l"(S.chunks[q_k] + (q_u - q_base))
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    ++q_u;
  };
  for (int i = 0; i < 12; ++i) q_issue();
  asm volatile("cp.async.wait_group 11;" ::: "memory");
  uint4 dv = ctl->dq[0];  // chunk u's descriptor: off16, bytes, rpos, rbytes
  // data cursor: phase k of chunk u, its end, data and rhs arrays
  int k = 0;
  while (S.begin[k + 1] == 0) ++k;
  int k_end = S.begin[k + 1];
  const uint8_t* data = S.data[k];
  const double* rhs = S.rhs[k];
  bool k_ready = false;
  // deferred slices: chunks [r_u, r_hi) of phase r_k (always the current or the next phase)
  int r_u = 0, r_hi = 0, r_k = k;
  // the rhs slice lands in the chunk's stage right behind its data (dbytes)
  auto rhs_copy = [&](int st, const double* src, uint32_t rpos, uint32_t rbytes, uint32_t dbytes) {
    if (dbg & 64) {
      mbar_arrive(&ctl->full[st]);
    } else {
      mbar_expect_tx(&ctl->full[st], rbytes * nv);  // nv interleaved right-hand sides
      bulk_load(stages + (size_t)st * stage_bytes + dbytes, src + (size_t)rpos * nv, rbytes * nv, &ctl->full[st]);
    }
  };
  auto phase_test = [&](int kk, bool block) -> bool {
    if (block) {
      mbar_wait(&ctl->rhs_ready[kk], 0);
    } else if (!mbar_test(&ctl->rhs_ready[kk], 0)) {
      return false;
    }
    fence_proxy_async();  // the consumers' generic-proxy rhs writes, before TMA reads them
    return true;
  };
  // issue the deferred slices once their phase is ready (block: wait for it)
  auto flush = [&](bool block) {
    if (r_u == r_hi) return;
    if (!phase_test(r_k, block)) return;
    for (; r_u < r_hi; ++r_u) {
      const int st = r_u % nst;
      const int4 rr = ctl->rrec[st];
      rhs_copy(st, S.rhs[r_k], (uint32_t)rr.x, (uint32_t)rr.y, (uint32_t)rr.z);
    }
    if (r_k == k) k_ready = true;
  };
  int st = 0;
  uint32_t par = 1;  // parity of the empty-barrier phase a reused stage waits for
  // L2 prefetch cursor: phase kp, byte offset pf; bytes copied / prefetched so far
  int kp = 0;
  while (kp < np && S.pf_hi[kp] == S.pf_lo[kp]) ++kp;
  uint32_t pf = kp < np ? S.pf_lo[kp] : 0u;
  long long issued = 0, prefetched = 0;
  const long long c_all = clock64();
  for (int u = 0; u < total; ++u) {
    if (u == k_end) {  // next phase (its slices are deferred until it is ready)
      flush(true);     // the previous phase's deferred slices (consumers need them first)
      do {
        ++k;
      } while (S.begin[k + 1] == S.begin[k]);
      k_end = S.begin[k + 1];
      data = S.data[k];
      rhs = S.rhs[k];
      k_ready = false;
      r_k = k;
      r_u = r_hi = u;
    }
    if (u >= nst) {
      // the stage's previous occupant (chunk u - nst) must be consumable: its slice issued
      if (r_u < r_hi && r_u <= u - nst) flush(true);
      while (!mbar_test(&ctl->empty[st], par)) {
        flush(false);
        __nanosleep(20);
      }
    }
    mbar_expect_tx(&ctl->full[st], dv.y);
    if (keep)
      bulk_load_hint(stages + (size_t)st * stage_bytes, data + (size_t)dv.x * 16, dv.y, &ctl->full[st], pol);
    else
      bulk_load(stages + (size_t)st * stage_bytes, data + (size_t)dv.x * 16, dv.y, &ctl->full[st]);
    if (l2ahead > 0) {  // keep the factor stream l2ahead bytes ahead in L2 (phases in order)
      issued += dv.y;
      while (prefetched < issued + l2ahead && kp < np) {
        const uint32_t n = min(32768u, S.pf_hi[kp] - pf);
        if (n) bulk_prefetch_l2(S.data[kp] + pf, n);
        pf += n;
        prefetched += n;
        if (pf >= S.pf_hi[kp] && ++kp < np) pf = S.pf_lo[kp];
      }
    }
    if (PSLR_TRACE_BUILD && g_tma && u < 8192) {
      g_tma[2 * u] = clock64();
      g_tma[2 * 8192 + u] = dv.y;
    }
    if (!k_ready && r_u == r_hi && phase_test(k, false)) k_ready = true;  // cheap once known
    if (k_ready) {
      rhs_copy(st, rhs, dv.z, dv.w, dv.y);
      r_u = r_hi = u + 1;
    } else {
      ctl->rrec[st] = make_int4((int32_t)dv.z, (int)dv.w, (int)dv.y, 0);
      r_hi = u + 1;
    }
    // next descriptor (its cp.async landed long ago) and the one twelve chunks ahead
    q_issue();
    asm volatile("cp.async.wait_group 11;" ::: "memory");
    dv = ctl->dq[(u + 1) & 15];
    if (++st == nst) {
      st = 0;
      par ^= 1u;
    }
  }
  flush(true);  // the last phase's deferred slices
  if (g_dbg_out) {
    atomicAdd(reinterpret_cast<unsigned long long*>(g_dbg_out + 7), (unsigned long long)(clock64() - c_all));
    atomicAdd(reinterpret_cast<unsigned long long*>(g_dbg_out + 4), (unsigned long long)total);
  }
}

// ---------------------------------------------------------------------------------------
// Right-hand sides per launch: NV = 1, or NV = 2 independent vectors stored interleaved
// ([row][2]) in every array the step kernel reads or writes.  The two chains of a row share
// every factor load and interleave (each is the single-vector arithmetic bit for bit).
template <int NV> struct VecT;
template <> struct VecT<1> { using T = double; };
template <> struct VecT<2> { using T = double2; };
template <int NV> using vt = typename VecT<NV>::T;

template <int NV> __device__ __forceinline__ vt<NV> vzero();
template <> __device__ __forceinline__ double vzero<1>() { return 0.0; }
template <> __device__ __forceinline__ double2 vzero<2>() { return make_double2(0.0, 0.0); }
template <int NV> __device__ __forceinline__ vt<NV> vld(const double* p, int64_t i);
template <> __device__ __forceinline__ double vld<1>(const double* p, int64_t i) { return p[i]; }
template <> __device__ __forceinline__ double2 vld<2>(const double* p, int64_t i) {
  return reinterpret_cast<const double2*>(p)[i];
}
template <int NV> __device__ __forceinline__ vt<NV> vldg(const double* p, int64_t i);
template <> __device__ __forceinline__ double vldg<1>(const double* p, int64_t i) { return __ldg(p + i); }
template <> __device__ __forceinline__ double2 vldg<2>(const double* p, int64_t i) {
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}
__device__ __forceinline__ void vst(double* p, int64_t i, double v) { p[i] = v; }
__device__ __forceinline__ void vst(double* p, int64_t i, double2 v) { reinterpret_cast<double2*>(p)[i] = v; }
// a - v * z, a + v * x, a - b, a + b, a * s  (separately rounded, per component)
__device__ __forceinline__ double vmsub(double a, double v, double z) { return a - v * z; }
__device__ __forceinline__ double2 vmsub(double2 a, double v, double2 z) {
  return make_double2(a.x - v * z.x, a.y - v * z.y);
}
__device__ __forceinline__ double vmadd(double a, double v, double x) { return a + v * x; }
__device__ __forceinline__ double2 vmadd(double2 a, double v, double2 x) {
  return make_double2(a.x + v * x.x, a.y + v * x.y);
}
__device__ __forceinline__ double vsub(double a, double b) { return a - b; }
__device__ __forceinline__ double2 vsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double vadd(double a, double b) { return a + b; }
__device__ __forceinline__ double2 vadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double vmul(double a, double s) { return a * s; }
__device__ __forceinline__ double2 vmul(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// Consumer side: the level loop.
//
// A level's critical path is: barrier -> ring gathers -> the row's DMUL/DADD chain ->
// ring store -> barrier.  Two things decide how close a level gets to it:
//  * ISSUE: all consumer warps walk the segment stream, but most levels have far fewer
//    rows than threads, so a warp owning no row of a segment must cost almost nothing.
//    The first 16 bytes of a segment header say everything needed to follow the stream
//    (rows, first thread, flags, size); a warp without rows reads that one word and
//    moves on (and arrives on the stage's empty barrier once per chunk).
//  * LATENCY: the header of the segment after next is read two ahead (a chunk
//    transition and its mbarrier wait happen a level early); the next row's raw
//    operands (slots, info, right-hand side) are loaded before the barrier and consumed
//    after it (the Markstein division overlaps the gathers); values and U's invd are
//    loaded after the barrier beside the gathers; the chain has w entries rounded up to
//    an even count (w = the segment's longest row; rows of a level are sorted by length,
//    shorter rows fold exact no-ops 0 * 0), not 4-entry groups.
// Inactive lanes of an active warp compute on row 0 of the segment and skip the stores.
//
// Segment layout (pack.cpp, pslr_internal.h); consumer thread tb + t owns row t.
constexpr int kLevelEnd = 1, kFar = 2, kExplicitSd = 4, kChunkEnd = 8, kFarRing = 16;

// one row's operands, loaded before the barrier of the level that precedes it
template <int NV>
struct RowOps {
  int t;          // row in the segment (0 for inactive lanes)
  bool active;    // this lane owns a row
  int info;       // L: U-position ; U: row id | bit 31 sd = 1 - 2^-53 | bit 30 far target
  uint32_t vals;  // smem offsets (computed before the barrier: no address arithmetic between
  uint32_t far;   //   the barrier and the gathers): val[0][0][t], the far list, U's invd[t]
  uint32_t invd;
  vt<NV> rhs;     // raw right-hand side(s)
  uint2 s0, s1;   // slot groups 0 and 1 (zero slot when absent)
  vt<NV> cadd;    // U epilogue addend
  int fsl;        // far-ring slot + 1 (0: the row is not a far-ring target)
};

__device__ __forceinline__ int hdr_rows(int4 h) { return h.x & 0xffff; }
__device__ __forceinline__ int hdr_w(int4 h) { return h.x >> 16; }
__device__ __forceinline__ int hdr_S(int4 h) { return ((h.x & 0xffff) + 3) & ~3; }
// bytes of a segment's per-row far-ring slots (uint16, present when flag bit 4 is set)
__device__ __forceinline__ uint32_t fsl_bytes(int S, int flags) {
  return (flags & kFarRing) ? (uint32_t)((2 * S + 15) & ~15) : 0u;
}
__device__ __forceinline__ uint32_t pre_bytes(bool upper, int S, int flags) {
  return 48 + 4 * S + fsl_bytes(S, flags) + (upper ? ((flags & kExplicitSd) ? 24 : 8) * S : 0);
}
// does this warp own rows of the segment?
__device__ __forceinline__ bool warp_owns(int4 h) {
  const int tb = h.y >> 8, w0 = (int)threadIdx.x & ~31;
  return w0 < tb + hdr_rows(h) && w0 + 32 > tb;
}

template <bool UPPER, int NV>
__device__ __forceinline__ void load_ops(uint32_t seg, int4 h, uint32_t rbuf, int rbase, int zslot,
                                         RowOps<NV>& r) {
  int t = (int)threadIdx.x - (h.y >> 8);
  r.active = (unsigned)t < (unsigned)hdr_rows(h);
  t = r.active ? t : 0;  // inactive lanes read row 0 (in bounds); their results are not stored
  r.t = t;
  const int S = hdr_S(h), G = max(1, (hdr_w(h) + 3) >> 2);
  r.far = seg + (uint32_t)sp<int32_t>(seg)[5];
  r.info = sp<int32_t>(seg + 48)[t];
  r.rhs = vld<NV>(sp<double>(rbuf), h.z + t - rbase);
  const uint32_t slots = seg + pre_bytes(UPPER, S, h.y) + 8 * t;
  r.s0 = *sp<uint2>(slots);
  const unsigned z2 = (unsigned)zslot | ((unsigned)zslot << 16);
  r.s1 = (hdr_w(h) > 4) ? *sp<uint2>(slots + 8 * S) : make_uint2(z2, z2);
  r.vals = slots + 8 * G * S + 8 * t;  // val[0][0][t] = pre + 8GS + 16t
  r.invd = seg + 48 + 4 * S + fsl_bytes(S, h.y) + 8 * t;
  r.fsl = (h.y & kFarRing) ? (int)sp<uint16_t>(seg + 48 + 4 * S)[t] : 0;
}

// U rows start from rhs / sd.  rcp = RN(1/sd): q0 = RN(x rcp) is within an ulp of x/sd
// and one fma-corrected step gives RN(x/sd) (Markstein); sd == 1 keeps x as is.
__device__ __forceinline__ double div_sd(double x, double sd, double rcp) {
  const double q0 = x * rcp;
  const double q = fma(fma(-q0, sd, x), rcp, q0);
  return (sd == 1.0) ? x : q;
}
__device__ __forceinline__ double2 div_sd(double2 x, double sd, double rcp) {
  return make_double2(div_sd(x.x, sd, rcp), div_sd(x.y, sd, rcp));
}

// dependency value: near -> ring slot, far (bit 15) -> the segment's far list -> global
// position-ordered array
template <bool FAR, int NV>
__device__ __forceinline__ vt<NV> gather(const double* ring, const double* z, uint32_t far, unsigned sl) {
  return (FAR && (sl & 0x8000u)) ? vld<NV>(z, sp<int32_t>(far)[sl & 0x7fffu]) : vld<NV>(ring, sl);
}

__device__ __forceinline__ unsigned slot_of(const uint2 s0, const uint2 s1, int k) {
  const uint32_t w = (k < 4) ? ((k < 2) ? s0.x : s0.y) : ((k < 6) ? s1.x : s1.y);
  return (k & 1) ? (w >> 16) : (w & 0xffffu);
}

// acc -= val_k * z_k for the first NE (even, <= 8) entries in the reference's
// ascending-column order; prep() yields the starting value after the loads are issued.
template <int NE, bool FAR, int NV, class Prep>
__device__ __forceinline__ vt<NV> fold_n(const RowOps<NV>& r, int S, uint32_t vals, uint32_t far,
                                         const double* ring, const double* z, Prep&& prep) {
  vt<NV> zz[NE];
#pragma unroll
  for (int k = 0; k < NE; ++k) zz[k] = gather<FAR, NV>(ring, z, far, slot_of(r.s0, r.s1, k));
  double2 d[NE / 2];
#pragma unroll
  for (int p = 0; p < NE / 2; ++p) d[p] = *sp<double2>(vals + 16 * S * p);
  vt<NV> acc = prep();
#pragma unroll
  for (int k = 0; k < NE; ++k) acc = vmsub(acc, (k & 1) ? d[k >> 1].y : d[k >> 1].x, zz[k]);
  return acc;
}

// rows longer than 8 entries: groups of four beyond the first two (padding: exact
// no-ops), slots straight from the staged segment (out of line: rare)
template <bool FAR, int NV>
__device__ __noinline__ vt<NV> fold_tail(vt<NV> acc, uint32_t slots, uint32_t vals, uint32_t far, int S, int G,
                                         const double* ring, const double* z) {
  for (int g = 2; g < G; ++g) {
    const uint2 sg = *sp<uint2>(slots + 8 * g * S);
    const vt<NV> z0 = gather<FAR, NV>(ring, z, far, sg.x & 0xffffu), z1 = gather<FAR, NV>(ring, z, far, sg.x >> 16);
    const vt<NV> z2 = gather<FAR, NV>(ring, z, far, sg.y & 0xffffu), z3 = gather<FAR, NV>(ring, z, far, sg.y >> 16);
    const double2 a = *sp<double2>(vals + 16 * S * (2 * g));
    const double2 b = *sp<double2>(vals + 16 * S * (2 * g + 1));
    acc = vmsub(acc, a.x, z0);
    acc = vmsub(acc, a.y, z1);
    acc = vmsub(acc, b.x, z2);
    acc = vmsub(acc, b.y, z3);
  }
  return acc;
}

template <bool FAR, int NV, class Prep>
__device__ __forceinline__ vt<NV> fold_w(const RowOps<NV>& r, int w, int S, uint32_t vals,
                                         uint32_t far, const double* ring, const double* z, Prep&& prep) {
  // two chain lengths (one uniform branch): a padded entry costs one dependent DADD,
  // a finer dispatch costs more in branch resolution
  if (w <= 4) return fold_n<4, FAR, NV>(r, S, vals, far, ring, z, prep);
  if (w <= 8) return fold_n<8, FAR, NV>(r, S, vals, far, ring, z, prep);
  const int G = (w + 3) >> 2;
  return fold_tail<FAR, NV>(fold_n<8, FAR, NV>(r, S, vals, far, ring, z, prep), vals - 8 * G * S - 8 * r.t, vals,
                            far, S, G, ring, z);
}

// compute one row of the segment (seg, h): gathers, chain, publish
template <bool UPPER, int NV, bool XPOS>
__device__ __forceinline__ void compute_row(const StepConst& K, uint32_t seg, int4 h, const RowOps<NV>& r,
                                            double* ring, int base, double* z, double* xout, const double* cadd) {
  const int S = hdr_S(h), w = hdr_w(h), flags = h.y;
  const uint32_t vals = r.vals, far = r.far;
  const double invd = UPPER ? *sp<double>(r.invd) : 0.0;  // beside the gathers
  auto prep = [&]() -> vt<NV> {
    if (!UPPER) return r.rhs;
    if (flags & kExplicitSd) {  // explicit sd / rcp arrays
      const double* d = sp<double>(r.invd);
      return div_sd(r.rhs, d[S], d[2 * S]);
    }
    // info bit 31: sd = 1 - 2^-53 (rcp = 1 + 2^-52), else sd = 1
    return (r.info < 0) ? div_sd(r.rhs, 0x1.fffffffffffffp-1, 0x1.0000000000001p+0) : r.rhs;
  };
  const vt<NV> acc = (flags & kFar) ? fold_w<true, NV>(r, w, S, vals, far, ring, z, prep)
                                    : fold_w<false, NV>(r, w, S, vals, far, ring, z, prep);
  if (r.active) {
    const int gp = h.z + r.t;
    vst(ring, (gp - base) & K.ring_mask, acc);
    if (r.fsl) vst(ring, K.ring_mask + 1 + r.fsl, acc);  // kept for its far readers
    if (UPPER) {
      if (r.info & 0x40000000) vst(z, gp, acc);  // only far-dependency targets go to global z
      vt<NV> x = vmul(acc, invd);
      if (cadd) x = vadd(x, r.cadd);
      vst(xout, XPOS ? gp : (r.info & 0x3fffffff), x);  // U-position order when only F reads x
    } else {
      vst(z, r.info, acc);  // the U phase's right-hand side, at the row's U-position
    }
  }
}

// Consumer side of one triangular phase.  Callers arrive right after a consumer barrier
// that follows the last write of the phase's rhs array; the phase ends with the barrier
// of its last level.  rel: the release cursor over the stages (carried across phases).
template <int NT, bool UPPER, int NV, bool XPOS = false>
__device__ __forceinline__ void tri_phase(const StepConst& K, const Streams& Sm, Ctl* ctl, uint8_t* stages_p,
                          int k, double* ring, int base, double* z, double* xout,
                          const double* cadd) {
  trace_ev(K, 10 + k, 0);
  trace_cta(K, 2 + k);
  if (threadIdx.x == 0) mbar_arrive(&ctl->rhs_ready[k]);  // writers fenced before the last barrier
  int u = Sm.begin[k];
  const int u1 = Sm.begin[k + 1];
  if (u == u1) return;
  const uint32_t stages = (uint32_t)(stages_p - smem);
  const int nst = K.nst, zslot = K.ring_mask + 1;
  int st = u % nst;
  uint32_t par = (uint32_t)((u / nst) & 1);
  if (K.dbg & 16) {  // timing experiment: the stream alone (every chunk waited for and released)
    for (; u < u1; ++u) {
      if (K.dbg & 2048)
        mbar_spin(&ctl->full[st], par);
      else
        mbar_wait(&ctl->full[st], par);
      if (PSLR_TRACE_BUILD && K.trace && blockIdx.x == K.trace_block && threadIdx.x == 0 && u < 8192)
        K.trace[2 + 2 * 65536 + 2 * u + 1] = clock64();
      if (PSLR_TRACE_BUILD && K.trace && blockIdx.x == K.trace_block && (threadIdx.x & 31) == 0 && u < 8192)
        atomicMax(reinterpret_cast<unsigned long long*>(K.trace + 2 + 2 * 65536 + 3 * 8192 + u),
                  (unsigned long long)clock64());  // the last warp to see the chunk
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&ctl->empty[st]);
      if (++st == nst) {
        st = 0;
        par ^= 1u;
      }
    }
    consumer_sync<NT>();
    return;
  }
  // segment A (computed this step), B (its operands loaded this step), C (header read)
  mbar_wait(&ctl->full[st], par);
  uint32_t segA = stages + (uint32_t)(st * K.stage_bytes);
  int stA = st, stB = st;  // stages holding A and B (released after their chunk's last segment)
  uint32_t rbuf = segA + (uint32_t)sp<int32_t>(segA)[7];  // the rhs slice behind the chunk's data
  int rbase = sp<int32_t>(segA)[6];
  int4 hA = *sp<int4>(segA);
  bool actA = warp_owns(hA);
  RowOps<NV> ra;
  if (actA) load_ops<UPPER, NV>(segA, hA, rbuf, rbase, zslot, ra);
  // the cursor moves to the segment after `seg` (header h); false at the end of the phase
  auto next = [&](uint32_t seg, int4 h, uint32_t& nseg) -> bool {
    if (h.y & kChunkEnd) {
      if (++u == u1) return false;
      if (++st == nst) {
        st = 0;
        par ^= 1u;
      }
      long long tw0 = 0;
      if (PSLR_TRACE_BUILD && threadIdx.x == 0) tw0 = clock64();
      mbar_wait(&ctl->full[st], par);
      if (PSLR_TRACE_BUILD && threadIdx.x == 0) {
        const long long dw = clock64() - tw0;
        g_wait_cyc += dw;
        g_wait_n += 1;
        g_wait_big += dw > 200 ? 1 : 0;
      }
      if (PSLR_TRACE_BUILD && K.trace && blockIdx.x == K.trace_block && threadIdx.x == 0 && u < 8192)
        K.trace[2 + 2 * 65536 + 2 * u + 1] = clock64();  // the chunk seen by the look-ahead
      nseg = stages + (uint32_t)(st * K.stage_bytes);
      rbuf = nseg + (uint32_t)sp<int32_t>(nseg)[7];
      rbase = sp<int32_t>(nseg)[6];
    } else {
      nseg = seg + (uint32_t)h.w;
    }
    return true;
  };
  uint32_t segB = 0;
  uint32_t rbufB = rbuf;
  int rbaseB = rbase;
  bool validB = next(segA, hA, segB);
  stB = st;
  int4 hB = validB ? *sp<int4>(segB) : make_int4(0, 0, 0, 0);
  if (validB) {
    rbufB = rbuf;
    rbaseB = rbase;
  }
  if (UPPER && actA) ra.cadd = (cadd && ra.active) ? vldg<NV>(cadd, ra.info & 0x3fffffff) : vzero<NV>();
  for (;;) {
    trace_clk(K, 50, (hA.x & 0xffff) | ((hA.y & 0xf) << 16) | (min(hdr_w(hA), 15) << 20) | ((int)UPPER << 24));
    if (actA && !(K.dbg & 1)) compute_row<UPPER, NV, XPOS>(K, segA, hA, ra, ring, base, z, xout, cadd);
    trace_clk(K, 52, 0);
    if (hA.y & kChunkEnd) {  // this warp no longer reads A's stage
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&ctl->empty[stA]);
    }
    const int flagsA = hA.y;
    if (!validB) {
      fence_rhs_written();  // z (an L phase's output) is the next phase's right-hand side
      if (flagsA & kLevelEnd) consumer_sync<NT>();
      break;
    }
    // B: this warp's row operands (before the barrier; consumed after it)
    const bool actB = warp_owns(hB);
    if (actB && !(K.dbg & 2)) load_ops<UPPER, NV>(segB, hB, rbufB, rbaseB, zslot, ra);
    trace_clk(K, 53, 0);
    // C: the header after B
    uint32_t segC = 0;
    const bool validC = next(segB, hB, segC);
    const int4 hC = validC ? *sp<int4>(segC) : make_int4(0, 0, 0, 0);
    trace_clk(K, 54, 0);
    if (flagsA & kLevelEnd) consumer_sync<NT>();
    if (UPPER && actB)  // the epilogue addend: a global load a level ahead of its use
      ra.cadd = (cadd && ra.active) ? vldg<NV>(cadd, ra.info & 0x3fffffff) : vzero<NV>();
    segA = segB;
    hA = hB;
    actA = actB;
    stA = stB;
    stB = st;
    segB = segC;
    hB = hC;
    validB = validC;
    rbufB = rbuf;
    rbaseB = rbase;
  }
}


// Four SpMV rows at once (independent gathers in flight): s[j] = sum_e M_ij x_j in CSR
// order from 0 (scipy csr_matvec).  RO: x is read-only for this launch.
template <bool RO, int NV>
__device__ __forceinline__ void spmv4(const DevCsr& M, const int (&row)[4], const bool (&ok)[4],
                                      const double* x, vt<NV> (&s)[4]) {
  int e0[4], e1[4];
  int len = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    e0[j] = ok[j] ? __ldg(M.ptr + row[j]) : 0;
    e1[j] = ok[j] ? __ldg(M.ptr + row[j] + 1) : 0;
    s[j] = vzero<NV>();
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
    vt<NV> xv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xv[j] = on[j] ? (RO ? vldg<NV>(x, c[j]) : vld<NV>(x, c[j])) : vzero<NV>();
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (on[j]) s[j] = vmadd(s[j], v[j], xv[j]);
  }
}

template <int NV, bool XPOS>
__device__ __forceinline__ void iface_terms4(int kind, const int (&row)[4], const bool (&ok)[4],
                                             const StepArgs& a, const StepConst& K, vt<NV> (&t)[4]) {
  switch (kind) {
    case IT_G:
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = ok[j] ? vldg<NV>(a.g, row[j]) : vzero<NV>();
      break;
    case IT_FX: spmv4<false, NV>(XPOS ? K.Fpos : K.F, row, ok, a.xb, t); break;
    case IT_CY: spmv4<true, NV>(K.C, row, ok, a.yC, t); break;
    case IT_CGY: spmv4<true, NV>(K.Cg, row, ok, a.yC, t); break;
    case IT_PRE:
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = ok[j] ? vldg<NV>(a.pre, row[j]) : vzero<NV>();
      break;
    default:
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = vzero<NV>();
  }
}

// Right-hand-side transform of a level-merged factor (pack.cpp merge_levels), for this
// CTA's block, in place: arr[pos_i] -= c0 arr[pos_j0] + c1 arr[pos_j1] + c2 arr[pos_j2].
// The records read only unmerged rows and write only merged ones (no ordering among them).
// Callers fence and barrier before the phase that reads arr.
template <int NV, int NT>
__device__ __forceinline__ void xform_block(const DevXform& X, int b, double* arr) {
  const int r0 = __ldg(X.blk + b), r1 = __ldg(X.blk + b + 1);
  constexpr int kIn = 4;  // records in flight per thread (two dependent global round trips)
  const int4* idx = reinterpret_cast<const int4*>(X.idx);
  const double2* val = reinterpret_cast<const double2*>(X.val);
  for (int i0 = r0 + (int)threadIdx.x; i0 < r1; i0 += kIn * NT) {
    int4 id[kIn];
    double2 c01[kIn], c2[kIn];
#pragma unroll
    for (int j = 0; j < kIn; ++j) {
      const int i = i0 + j * NT;
      const bool ok = i < r1;
      id[j] = ok ? __ldg(idx + i) : make_int4(0, 0, 0, 0);
      c01[j] = ok ? __ldg(val + 2 * i) : make_double2(0.0, 0.0);
      c2[j] = ok ? __ldg(val + 2 * i + 1) : make_double2(0.0, 0.0);
    }
    vt<NV> a[kIn], z0[kIn], z1[kIn], z2[kIn];
#pragma unroll
    for (int j = 0; j < kIn; ++j) {
      a[j] = vld<NV>(arr, id[j].x);
      z0[j] = vld<NV>(arr, id[j].y);
      z1[j] = vld<NV>(arr, id[j].z);
      z2[j] = vld<NV>(arr, id[j].w);
    }
#pragma unroll
    for (int j = 0; j < kIn; ++j) {
      vt<NV> t = vmul(z0[j], c01[j].x);
      t = vmadd(t, c01[j].y, z1[j]);
      t = vmadd(t, c2[j].x, z2[j]);
      if (i0 + j * NT < r1) vst(arr, id[j].x, vsub(a[j], t));
    }
  }
}

// prepass loads in flight per thread (the prepass is latency-bound: three dependent global
// loads per E row; more rows in flight per thread = fewer round trips)
#ifndef PSLR_PRE_F
#define PSLR_PRE_F 8
#endif
#ifndef PSLR_PRE_E
#define PSLR_PRE_E 8
#endif
#ifndef PSLR_STEP_MINB
#define PSLR_STEP_MINB 1
#endif
template <int NV, bool XPOS, int NT>
__global__ void __launch_bounds__(NT + 32, PSLR_STEP_MINB)
subdomain_step_kernel(const __grid_constant__ StepArgs a, const __grid_constant__ StepConst K) {
  const int b = blockIdx.x;
  const bool do_b = a.b1 != BT_NONE;
  const bool do_i = a.i1 != IT_NONE;
  const bool do_c = do_i && a.do_c0;

  Ctl* ctl = reinterpret_cast<Ctl*>(smem);
  // [Ctl][ring: (W + zero slot + far-ring) x NV, padded to 128 B][nst stages: chunk data + its rhs slice]
  // The ring sits at a constant offset, so a gather is one address op on its slot.
  double* ring = reinterpret_cast<double*>(smem + kCtlBytes);
  // [ring W | zero slot | far-ring] padded to 128 B, then the stages
  uint8_t* stages = smem + kCtlBytes + (((size_t)(K.ring_mask + 2 + K.far_slots) * 8 * NV + 127) / 128) * 128;

  // The stream table lives in shared memory: dynamically indexed per-thread arrays would
  // spill to local memory, which misses the small L1 left beside 229 KB of shared memory.
  __shared__ Streams s_streams;
  Streams& S = s_streams;
  if (threadIdx.x == 0) {
    S.nphase = 0;
    S.begin[0] = 0;
    auto add_phase = [&](const DevTri& T, const double* rhs) {
      const int c0 = T.blk_chunk[b], c1 = T.blk_chunk[b + 1];
      S.data[S.nphase] = T.data;
      S.chunks[S.nphase] = T.chunks + c0;
      S.rhs[S.nphase] = rhs;
      if (K.l2ahead > 0 && c1 > c0) {
        const ChunkDesc d0 = load_desc(T.chunks + c0), d1 = load_desc(T.chunks + c1 - 1);
        S.pf_lo[S.nphase] = d0.off16 * 16u;
        S.pf_hi[S.nphase] = d1.off16 * 16u + d1.bytes;
      } else {
        S.pf_lo[S.nphase] = S.pf_hi[S.nphase] = 0;
      }
      S.begin[S.nphase + 1] = S.begin[S.nphase] + (c1 - c0);
      S.nphase++;
    };
    if (do_b) {
      add_phase(K.LB, a.fL ? a.fL : (a.b1 == BT_EY && a.b2 == BT_NONE) ? K.rhsE : K.rhsB);
      add_phase(K.UB, K.zB);
    }
    if (do_c) {
      add_phase(K.LC, K.rhsC);
      add_phase(K.UC, K.zC);
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < K.nst; ++s) {
      mbar_init(&ctl->full[s], 2);
      mbar_init(&ctl->empty[s], NT / 32);
    }
    for (int k = 0; k < 4; ++k) mbar_init(&ctl->rhs_ready[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= NT) {  // producer warp (all 32 lanes)
    producer(S, ctl, stages, K.nst, K.stage_bytes, NV,
             (K.trace && K.trace_cap >= (1 << 20)) ? K.trace + 2 + 2 * K.trace_cap - 8 * 4096 + b * 8
                                                   : nullptr,
             K.dbg,
             (PSLR_TRACE_BUILD && K.trace && b == K.trace_block) ? K.trace + 2 + 2 * 65536 : nullptr,
             K.l2ahead, K.l2keep ? (int)K.l2keep[b] : 0);
    return;
  }
  // Programmatic dependent launch: this grid may start while the previous kernel of the
  // stream finishes (setup above and the producer's factor stream do not depend on it);
  // consumers wait here for its completion before reading any vector it produced or
  // writing any buffer it may still read.  A no-op for ordinary launches.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (PSLR_TRACE_BUILD && threadIdx.x == 0) {
    g_trace_tag = a.tag;
    g_wait_cyc = 0;
    g_wait_n = g_wait_big = 0;
  }
  trace_begin(K);
  trace_ev(K, 1, S.begin[S.nphase]);
  trace_cta(K, 0);
  if (threadIdx.x == 0) vst(ring, K.ring_mask + 1, vzero<NV>());  // the zero slot (visible after the next barrier)
  const int ph_LB = 0, ph_UB = 1;
  const int ph_LC = do_b ? 2 : 0, ph_UC = do_b ? 3 : 1;
  const int tid = threadIdx.x;

  if (do_b) {
    const int r0 = K.int_off[b], r1 = K.int_off[b + 1];
    // pass 1: rhs = f scattered to the L-positions (stores do not stall, so scatter
    // beats a gather here), or a coalesced zero fill.  With a.fL the all-SM permute_f
    // kernel has done it: the L phase reads fL and only the E rows are rewritten.
    const bool ey_only = a.b1 == BT_EY && a.b2 == BT_NONE;
    double* rhs = a.fL ? a.fL : ey_only ? K.rhsE : K.rhsB;
    if (a.fL || ey_only) {
      // fL holds f already; rhsE's non-E positions are permanently 0
    } else if (a.b1 == BT_F) {
      constexpr int kIn = PSLR_PRE_F;  // independent loads in flight per thread
      for (int row0 = r0 + tid; row0 < r1; row0 += kIn * NT) {
        vt<NV> v[kIn];
        int pos[kIn];
#pragma unroll
        for (int j = 0; j < kIn; ++j) {
          const int row = row0 + j * NT;
          const bool ok = row < r1;
          v[j] = ok ? vldg<NV>(a.f, row) : vzero<NV>();
          pos[j] = ok ? __ldg(K.LB.lpos + row) : 0;
        }
#pragma unroll
        for (int j = 0; j < kIn; ++j)
          if (row0 + j * NT < r1) vst(K.rhsB, pos[j], v[j]);
      }
      if (K.XLB.nrec) {  // level-merged L_B: f' = (I - N) f in place
        consumer_sync<NT>();
        xform_block<NV, NT>(K.XLB, b, K.rhsB);
      }
    } else {
      for (int p = r0 + tid; p < r1; p += NT) vst(K.rhsB, p, vzero<NV>());
    }
    // pass 2: rows with E entries get the E y term: f - E y, or E y alone (scipy
    // csr_matvec order), kIn rows per thread in flight; one int4 record per row
    if ((a.b1 == BT_EY || a.b2 == BT_EY) && !a.ey_done) {
      if (!a.fL && !ey_only) consumer_sync<NT>();
      constexpr int kIn = PSLR_PRE_E;  // E rows in flight per thread (dependent chain: record, E entry, y)
      const int e0 = K.erow_off[b], e1 = K.erow_off[b + 1];
      const int4* rec = reinterpret_cast<const int4*>(K.erows);
      for (int i0 = e0 + tid; i0 < e1; i0 += kIn * NT) {
        int4 r[kIn];
        vt<NV> fv[kIn], sum[kIn];
        int len = 0;
#pragma unroll
        for (int j = 0; j < kIn; ++j) {
          const int i = i0 + j * NT;
          r[j] = i < e1 ? __ldg(rec + i) : make_int4(0, 0, 0, 0);
          len = max(len, r[j].w - r[j].z);
          sum[j] = vzero<NV>();
        }
#pragma unroll
        for (int j = 0; j < kIn; ++j)
          fv[j] = (a.b1 == BT_F && r[j].w > r[j].z) ? vld<NV>(rhs, r[j].x) : vzero<NV>();  // f (pass 1)
        for (int k = 0; k < len; ++k) {
          int c[kIn];
          double v[kIn];
          vt<NV> yv[kIn];
#pragma unroll
          for (int j = 0; j < kIn; ++j) {
            const bool on = r[j].z + k < r[j].w;
            c[j] = on ? __ldg(K.E.col + r[j].z + k) : 0;
            v[j] = on ? __ldg(K.E.val + r[j].z + k) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < kIn; ++j) yv[j] = (r[j].z + k < r[j].w) ? vldg<NV>(a.yE, c[j]) : vzero<NV>();
#pragma unroll
          for (int j = 0; j < kIn; ++j)
            if (r[j].z + k < r[j].w) sum[j] = vmadd(sum[j], v[j], yv[j]);
        }
#pragma unroll
        for (int j = 0; j < kIn; ++j)
          if (i0 + j * NT < e1) vst(rhs, r[j].x, (a.b1 == BT_F) ? vsub(fv[j], sum[j]) : sum[j]);
      }
    }
    fence_rhs_written();  // the L_B right-hand side (f / E y rows) is read by TMA next
    consumer_sync<NT>();
    trace_ev(K, 3, 0);
    trace_cta(K, 1);
    tri_phase<NT, false, NV>(K, S, ctl, stages, ph_LB, ring, r0, K.zB, nullptr, nullptr);
    if (K.XUB.nrec) {  // level-merged U_B: y' = (I - M) y in place (y: L_B's output)
      xform_block<NV, NT>(K.XUB, b, K.zB);
      fence_rhs_written();
      consumer_sync<NT>();
    }
    tri_phase<NT, true, NV, XPOS>(K, S, ctl, stages, ph_UB, ring, r0, K.zB, a.xb, nullptr);
  }
  if (do_i) {
    trace_cta(K, 7);
    const int r0 = K.ifc_off[b], r1 = K.ifc_off[b + 1];
    for (int row0 = r0 + tid; row0 < r1 && !a.ifc_done; row0 += 4 * NT) {
      int row[4];
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        row[j] = row0 + j * NT;
        ok[j] = row[j] < r1;
      }
      vt<NV> w[4], t2[4];
      iface_terms4<NV, XPOS>(a.i1, row, ok, a, K, w);
      if (a.i2 != IT_NONE) {
        iface_terms4<NV, XPOS>(a.i2, row, ok, a, K, t2);
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = a.i2_sub ? vsub(w[j], t2[j]) : vadd(w[j], t2[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!ok[j]) continue;
        if (do_c) {
          vst(K.rhsC, __ldg(K.LC.lpos + row[j]), w[j]);
        } else {
          vt<NV> y = w[j];
          if (a.cadd) y = vadd(y, vldg<NV>(a.cadd, row[j]));
          vst(a.yout, row[j], y);
        }
      }
    }
    fence_rhs_written();  // rhsC is the L_C0 right-hand side
    consumer_sync<NT>();
    trace_ev(K, 30, 0);
    if (do_c) {
      if (K.XLC.nrec) {  // level-merged L_C0: w' = (I - N) w in place
        xform_block<NV, NT>(K.XLC, b, K.rhsC);
        fence_rhs_written();
        consumer_sync<NT>();
      }
      tri_phase<NT, false, NV>(K, S, ctl, stages, ph_LC, ring, r0, K.zC, nullptr, nullptr);
      if (K.XUC.nrec) {  // level-merged U_C0
        xform_block<NV, NT>(K.XUC, b, K.zC);
        fence_rhs_written();
        consumer_sync<NT>();
      }
      tri_phase<NT, true, NV>(K, S, ctl, stages, ph_UC, ring, r0, K.zC, a.yout, a.cadd);
    }
  }
  trace_cta(K, 6);
  if (PSLR_TRACE_BUILD && K.trace && threadIdx.x == 0 && K.trace_cap >= (1 << 20) && blockIdx.x < 64) {
    long long* w = K.trace + 2 + 2 * K.trace_cap - 8 * 4096 + (3072 + 64 * (g_trace_tag & 15) + blockIdx.x) * 8;
    w[0] = g_wait_cyc;
    w[1] = g_wait_n;
    w[2] = g_wait_big;
  }
}

// The parts of a step that only need vectors of earlier launches, for every block at once
// on all SMs (in the step kernel they run on the one SM per block, as dependent global
// loads on the critical path — the E y prepass alone took 13-17 us before the L phase):
//   threads [0, ne): the E y rows of the L_B right-hand side, rhs[pos] = E_row y (ey_only)
//                    or rhs[pos] = rhs[pos] - E_row y (the last step, rhs = f in L order);
//   threads [ne, ne + nq): cgy[i] = C_g row i . y, the interface phase's C_g term.
// Every row is summed in CSR order from 0 (scipy csr_matvec), exactly as the step kernel.
template <int NV>
__global__ void __launch_bounds__(256) pre_step_kernel(const int4* __restrict__ erows, int ne, DevCsr E,
                                                       const double* __restrict__ yE, double* rhs, int sub,
                                                       DevCsr Cg, const double* __restrict__ yC, double* cgy,
                                                       int nq) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ne) {
    const int4 r = __ldg(erows + i);
    vt<NV> sum = vzero<NV>();
    for (int e = r.z; e < r.w; ++e) sum = vmadd(sum, __ldg(E.val + e), vldg<NV>(yE, __ldg(E.col + e)));
    if (sub) {
      vst(rhs, r.x, vsub(vld<NV>(rhs, r.x), sum));
    } else {
      vst(rhs, r.x, sum);
    }
  } else if (i - ne < nq) {
    const int row = i - ne;
    vt<NV> sum = vzero<NV>();
    const int e1 = __ldg(Cg.ptr + row + 1);
    for (int e = __ldg(Cg.ptr + row); e < e1; ++e) sum = vmadd(sum, __ldg(Cg.val + e), vldg<NV>(yC, __ldg(Cg.col + e)));
    vst(cgy, row, sum);
  }
}

// One term of the interface phase for one row (the step kernel's iface_terms4, one row):
// an SpMV row is summed in CSR order from 0 (scipy csr_matvec) exactly as there.
template <int NV>
__device__ __forceinline__ vt<NV> spmv_row1(const DevCsr& M, int row, const double* __restrict__ x) {
  vt<NV> s = vzero<NV>();
  const int e1 = __ldg(M.ptr + row + 1);
  for (int e = __ldg(M.ptr + row); e < e1; ++e) s = vmadd(s, __ldg(M.val + e), vldg<NV>(x, __ldg(M.col + e)));
  return s;
}
template <int NV, bool XPOS>
__device__ __forceinline__ vt<NV> iface_term1(int kind, int row, const StepArgs& a, const StepConst& K) {
  switch (kind) {
    case IT_G: return vldg<NV>(a.g, row);
    case IT_FX: return spmv_row1<NV>(XPOS ? K.Fpos : K.F, row, a.xb);
    case IT_CY: return spmv_row1<NV>(K.C, row, a.yC);
    case IT_CGY: return spmv_row1<NV>(K.Cg, row, a.yC);
    case IT_PRE: return vldg<NV>(a.pre, row);
    default: return vzero<NV>();
  }
}

// The interface phase of a step for every block at once (all SMs, one interface row per
// thread), between the launch of the B phases (x_B written) and the launch of the C0 phases:
// on the one SM per block it was 40-50 us of dependent gathers (F x_B, C_g y) on the
// critical block.  w = i1 (-|+) i2 ; do_c0: rhsC[L_C0 position] = w, else yout = w [+ cadd].
template <int NV, bool XPOS>
__global__ void __launch_bounds__(256) iface_kernel(const __grid_constant__ StepArgs a,
                                                    const __grid_constant__ StepConst K, int q) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= q) return;
  vt<NV> w = iface_term1<NV, XPOS>(a.i1, row, a, K);
  if (a.i2 != IT_NONE) {
    const vt<NV> t2 = iface_term1<NV, XPOS>(a.i2, row, a, K);
    w = a.i2_sub ? vsub(w, t2) : vadd(w, t2);
  }
  if (a.do_c0) {
    vst(K.rhsC, __ldg(K.LC.lpos + row), w);
  } else {
    if (a.cadd) w = vadd(w, vldg<NV>(a.cadd, row));
    vst(a.yout, row, w);
  }
}

int configure_step_kernel(int nv, int smem_bytes) {
  auto set = [&](auto kern) {
    return (int)cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  };
  int e;
  if (nv == 2) {
    if ((e = set(subdomain_step_kernel<2, false, kWide2Threads>))) return e;
    if ((e = set(subdomain_step_kernel<2, true, kWide2Threads>))) return e;
    if ((e = set(subdomain_step_kernel<2, false, kNarrowThreads>))) return e;
    return set(subdomain_step_kernel<2, true, kNarrowThreads>);
  }
  if ((e = set(subdomain_step_kernel<1, false, kStepThreads>))) return e;
  if ((e = set(subdomain_step_kernel<1, true, kStepThreads>))) return e;
  if ((e = set(subdomain_step_kernel<1, false, kNarrowThreads>))) return e;
  return set(subdomain_step_kernel<1, true, kNarrowThreads>);
}

int launch_step_kernel(const pslr_ctx* ctx, const StepArgs& a, const StepConst& K, cudaStream_t st, int nv);

int launch_step(const pslr_ctx* ctx, const StepArgs& a_in, cudaStream_t st, int nv) {
  if (ctx->s == 0) return 0;
  // x_B is read only by this launch's F SpMV: store it in U-position order (coalesced
  // stores from the level loop) and read it through the position-mapped F.  Launches
  // whose x_B leaves the kernel (the last step, solve_B) keep row order.
  StepArgs a = a_in;
  a.xpos = (a.b1 != BT_NONE && (a.i1 == IT_FX || a.i2 == IT_FX)) ? 1 : 0;
  const StepConst& K = (nv == 2) ? ctx->K2 : ctx->K;
  // E y rows of the L right-hand side (when the rhs array is one the prepass would only
  // patch at the E rows: E y alone into rhsE, or f - E y into fL) and the C_g y term of the
  // interface phase, by the all-SM pre-kernel
  const bool ey_only = a.b1 == BT_EY && a.b2 == BT_NONE;
  const bool f_ey = a.fL && a.b1 == BT_F && a.b2 == BT_EY;
  const int ne = ((ey_only || f_ey) && ctx->ey_all_sm) ? K.nerows : 0;
  const int nq = (a.i2 == IT_CGY && K.cgy && ctx->ey_all_sm) ? (int)K.Cg.nrows : 0;
  // A halo exchange of yC's ghost columns may still be in flight on the communication stream
  // (comm.cu comm_halo_async).  Only C_g reads ghosts: with the split interface phase the E y
  // rows and the B phases run first and the stream waits for the halo between the B launch
  // and the C_g y kernel; every other launch shape waits here.
  cudaEvent_t halo_ev = ctx->pending_halo;
  ctx->pending_halo = nullptr;
  const bool split = ctx->split_iface && a.i1 != IT_NONE && (a.b1 != BT_NONE || a.do_c0) && !a.ifc_done;
  const bool defer_cgy = halo_ev && nq > 0 && split && a.b1 != BT_NONE;
  if (halo_ev && !defer_cgy) {
    const cudaError_t e = cudaStreamWaitEvent(st, halo_ev, 0);
    if (e != cudaSuccess) return (int)e;
    halo_ev = nullptr;
  }
  auto pre_launch = [&](int ne_, int nq_) -> int {
    cudaLaunchConfig_t ec = {};
    ec.gridDim = dim3((unsigned)((ne_ + nq_ + 255) / 256));
    ec.blockDim = dim3(256);
    ec.stream = st;
    cudaLaunchAttribute eat[1];
    eat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    eat[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
    ec.attrs = eat;
    ec.numAttrs = 1;
    double* rhs = ey_only ? K.rhsE : a.fL;
    const int sub = f_ey ? 1 : 0;
    const int4* er = reinterpret_cast<const int4*>(K.erows);
    return (int)((nv == 2)
                     ? cudaLaunchKernelEx(&ec, pre_step_kernel<2>, er, ne_, K.E, a.yE, rhs, sub, K.Cg, a.yC, K.cgy, nq_)
                     : cudaLaunchKernelEx(&ec, pre_step_kernel<1>, er, ne_, K.E, a.yE, rhs, sub, K.Cg, a.yC, K.cgy, nq_));
  };
  if (ne > 0 || (nq > 0 && !defer_cgy)) {
    const int e = pre_launch(ne, defer_cgy ? 0 : nq);
    if (e) return e;
  }
  if (ne > 0) a.ey_done = 1;
  if (nq > 0) {
    a.i2 = IT_PRE;
    a.pre = K.cgy;
  }
  // programmatic stream serialization: the step kernel's CTAs (one per subdomain, far
  // fewer than the 148 SMs) launch and stage their first factor chunks while the
  // previous kernel drains; griddepcontrol.wait orders the data accesses
  // The interface phase of a launch that also has a B phase (or a C0 phase) runs as its own
  // all-SM kernel: [B phases] -> iface_kernel -> [C0 phases], the two step launches being
  // the same kernel with the other phases switched off (bit for bit the same results).
  if (split) {
    if (a.b1 != BT_NONE) {
      StepArgs ab = a;
      ab.i1 = ab.i2 = IT_NONE;
      ab.do_c0 = 0;
      ab.yout = nullptr;
      const int e = launch_step_kernel(ctx, ab, K, st, nv);
      if (e) return e;
    }
    if (defer_cgy) {  // the ghosts of yC have landed: C_g y, then the interface phase
      cudaError_t e = cudaStreamWaitEvent(st, halo_ev, 0);
      if (e != cudaSuccess) return (int)e;
      const int e2 = pre_launch(0, nq);
      if (e2) return e2;
    }
    cudaLaunchConfig_t ic = {};
    ic.gridDim = dim3((unsigned)((ctx->q + 255) / 256));
    ic.blockDim = dim3(256);
    ic.stream = st;
    cudaLaunchAttribute iat[1];
    iat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    iat[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
    ic.attrs = iat;
    ic.numAttrs = 1;
    const int q = (int)ctx->q;
    cudaError_t e;
    if (nv == 2)
      e = a.xpos ? cudaLaunchKernelEx(&ic, iface_kernel<2, true>, a, K, q)
                 : cudaLaunchKernelEx(&ic, iface_kernel<2, false>, a, K, q);
    else
      e = a.xpos ? cudaLaunchKernelEx(&ic, iface_kernel<1, true>, a, K, q)
                 : cudaLaunchKernelEx(&ic, iface_kernel<1, false>, a, K, q);
    if (e != cudaSuccess) return (int)e;
    if (!a.do_c0) return 0;
    StepArgs ac = a;
    ac.b1 = ac.b2 = BT_NONE;
    ac.ifc_done = 1;
    ac.xpos = 0;
    ac.tag = a.tag | 8;  // trace builds: the C0 launch of a split step stamps its own row
    return launch_step_kernel(ctx, ac, K, st, nv);
  }
  return launch_step_kernel(ctx, a, K, st, nv);
}

int launch_step_kernel(const pslr_ctx* ctx, const StepArgs& a, const StepConst& K, cudaStream_t st, int nv) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctx->s);
  cfg.blockDim = dim3((unsigned)(K.nthr + 32));
  cfg.dynamicSmemBytes = (size_t)K.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) { return (int)cudaLaunchKernelEx(&cfg, kern, a, K); };
  const bool narrow = K.nthr == kNarrowThreads && kNarrowThreads != (nv == 2 ? kWide2Threads : kStepThreads);
  if (!narrow && K.nthr != (nv == 2 ? kWide2Threads : kStepThreads)) return (int)cudaErrorInvalidValue;
  if (nv == 2) {
    if (narrow)
      return a.xpos ? go(subdomain_step_kernel<2, true, kNarrowThreads>) : go(subdomain_step_kernel<2, false, kNarrowThreads>);
    return a.xpos ? go(subdomain_step_kernel<2, true, kWide2Threads>) : go(subdomain_step_kernel<2, false, kWide2Threads>);
  }
  if (narrow)
    return a.xpos ? go(subdomain_step_kernel<1, true, kNarrowThreads>) : go(subdomain_step_kernel<1, false, kNarrowThreads>);
  return a.xpos ? go(subdomain_step_kernel<1, true, kStepThreads>) : go(subdomain_step_kernel<1, false, kStepThreads>);
}

}  // namespace pslr
