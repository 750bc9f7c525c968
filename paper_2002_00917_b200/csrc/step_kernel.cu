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

// Shared-memory control block
struct Ctl {
  uint64_t full[8];       // data + rhs landed (2 arrivals + tx bytes)
  uint64_t empty[8];      // all consumer warps done with the stage (kConsumerWarps arrivals)
  uint64_t rhs_ready[4];  // phase k's rhs array is final (1 arrival)
  int2 rrec[8];           // per stage: rhs slice (first position, bytes) of the staged chunk
};

// The chunks of up to four factor streams of this CTA's block form one sequence.
struct Streams {
  int nphase;
  int begin[5];
  const uint8_t* data[4];
  const ChunkDesc* chunks[4];  // this block's first chunk of the phase
  const double* rhs[4];        // position-ordered right-hand-side array of each phase
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

// Producer: one thread (lane 0 of the producer warp).  The loop is latency-bound on a
// single thread, so everything per chunk is precomputed (ChunkDesc) and the next
// descriptor load is in flight while the producer waits for a free stage.
//   data cursor: chunk d_u goes to stage d_u % nst once the consumers released it;
//   rhs cursor:  chunk r_u < d_u gets its rhs slice once its phase's rhs is final;
//   L2 cursor:   bulk prefetch kL2Ahead bytes beyond the issued data.
__device__ void producer(const Streams& S, Ctl* ctl, uint8_t* stages, double* rhsbuf, int nst,
                         int stage_bytes, int rhs_stride, int nv, long long* g_dbg_out) {
  if ((threadIdx.x & 31) != 0) return;
  const int np = S.nphase;
  const int total = S.begin[np];
  if (total == 0) return;
  const int64_t l2ahead = kL2Ahead;
  // data cursor
  int d_u = 0, d_k = 0;
  while (S.begin[d_k + 1] == 0) ++d_k;
  int d_end = S.begin[d_k + 1], d_base = 0;
  const uint8_t* d_data = S.data[d_k];
  const ChunkDesc* d_ops = S.chunks[d_k];
  ChunkDesc dop = load_desc(d_ops);
  int st_d = 0, use_d = 0;
  // rhs cursor
  int r_u = 0, r_k = d_k, r_end = d_end, st_r = 0;
  const double* r_rhs = S.rhs[r_k];
  uint32_t ready = 0;
  // L2 cursor over the byte ranges of the phases (chunks of a phase are contiguous)
  int pf_k = d_k;
  int64_t pf_off = 0, pf_hi = 0, issued = 0, prefetched = 0;
  auto pf_range = [&](int k) {
    const int n = S.begin[k + 1] - S.begin[k];
    if (n == 0) {
      pf_off = pf_hi = 0;
      return;
    }
    const ChunkDesc a = load_desc(S.chunks[k]), z = load_desc(S.chunks[k] + n - 1);
    pf_off = (int64_t)a.off16 * 16;
    pf_hi = (int64_t)z.off16 * 16 + z.bytes;
  };
  pf_range(pf_k);
  long long c_idle = 0, n_it = 0;
  const long long c_all = clock64();
  while (r_u < total) {
    bool did = false;
    ++n_it;
    const long long c_it = clock64();
    if (d_u < total && (use_d == 0 || mbar_test(&ctl->empty[st_d], (uint32_t)((use_d - 1) & 1)))) {
      mbar_expect_tx(&ctl->full[st_d], dop.bytes);
      bulk_load(stages + (size_t)st_d * stage_bytes, d_data + (size_t)dop.off16 * 16, dop.bytes,
                &ctl->full[st_d]);
      ctl->rrec[st_d] = make_int2(dop.rpos, (int)dop.rbytes);
      issued += dop.bytes;
      if (++st_d == nst) {
        st_d = 0;
        ++use_d;
      }
      if (++d_u < total) {
        while (d_u >= d_end) {
          ++d_k;
          d_base = S.begin[d_k];
          d_end = S.begin[d_k + 1];
          d_data = S.data[d_k];
          d_ops = S.chunks[d_k];
        }
        dop = load_desc(d_ops + (d_u - d_base));
      }
      did = true;
    }
    if (r_u < d_u) {
      while (r_u >= r_end) {
        ++r_k;
        r_end = S.begin[r_k + 1];
        r_rhs = S.rhs[r_k];
      }
      if (!(ready & (1u << r_k)) && mbar_test(&ctl->rhs_ready[r_k], 0)) {
        ready |= 1u << r_k;
        fence_proxy_async();
      }
      if (ready & (1u << r_k)) {
        const int2 rr = ctl->rrec[st_r];
        mbar_expect_tx(&ctl->full[st_r], (uint32_t)(rr.y * nv));  // nv interleaved right-hand sides
        bulk_load(rhsbuf + (size_t)st_r * rhs_stride, r_rhs + (size_t)rr.x * nv, (uint32_t)(rr.y * nv),
                  &ctl->full[st_r]);
        ++r_u;
        if (++st_r == nst) st_r = 0;
        did = true;
      }
    }
    while (prefetched < issued + l2ahead && pf_k < np) {
      if (pf_off >= pf_hi) {
        if (++pf_k < np) pf_range(pf_k);
        continue;
      }
      const int64_t len = (pf_hi - pf_off) < 32768 ? (pf_hi - pf_off) : 32768;
      bulk_prefetch_l2(S.data[pf_k] + pf_off, (uint32_t)len);
      pf_off += len;
      prefetched += len;
    }
    if (!did) {
      __nanosleep(20);
      c_idle += clock64() - c_it;
    }
  }
  if (g_dbg_out) {
    atomicAdd(reinterpret_cast<unsigned long long*>(g_dbg_out + 5), (unsigned long long)c_idle);
    atomicAdd(reinterpret_cast<unsigned long long*>(g_dbg_out + 7), (unsigned long long)(clock64() - c_all));
    atomicAdd(reinterpret_cast<unsigned long long*>(g_dbg_out + 4), (unsigned long long)n_it);
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
// A level's critical path is latency: gather the dependencies from the ring, the
// sequential DADD chain, store, barrier.  Everything that does not depend on the
// previous level is loaded one segment ahead: the next segment's header, the row's
// slots (two groups), its first four values, rhs, U's invd / cadd.  The step is written
// as straight-line code (no per-row branches: inactive lanes compute on row 0 of the
// segment and skip the stores).
//
// Segment layout (pack.cpp, pslr_internal.h); consumer thread tb + t owns row t
// (tb = flags >> 8), so the segments of one level run side by side.
template <int NV>
struct Row {
  const uint8_t* slots;  // &slot[0][t]  (4 x u16 per row and group)
  const uint8_t* vals;   // &val[0][0][t]
  const int32_t* far;    // the segment's far list (U-positions)
  int bytes, flags, G, S, nrows;
  bool wact;             // the warp owns rows of this segment (warp-uniform)
  bool active;           // this lane owns a row
  int ridx;              // ring slot of the row
  int zidx;              // z index: L: U-position ; U: position (-1: not a far target)
  int xidx;              // U: xout index (row id)
  vt<NV> acc;            // right-hand side(s) (U: already divided by sd)
  double invd;           // U epilogue
  vt<NV> cadd;
  uint2 s0, s1;          // slot groups 0 and 1 (zero slot when absent)
  double2 va, vb;        // group-0 values
};

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

template <bool UPPER, int NV, bool XPOS = false>
__device__ __forceinline__ void load_row(const uint8_t* seg, const int4 h0, const int4 h1, const double* rbuf,
                                         int rbase, int base, int mask, int zslot,
                                         const double* __restrict__ cadd, Row<NV>& r) {
  const int S = h1.x;
  const int G = max(1, (h0.y + 3) >> 2);
  r.flags = h0.z;
  r.S = S;
  r.G = G;
  r.nrows = h0.x;
  r.bytes = h1.y;
  // warps owning no row of the segment skip it entirely (the four schedulers are shared
  // by all consumer warps, so idle warps must not spend issue slots)
  const int tb = h0.z >> 8, w0 = (int)threadIdx.x & ~31;
  r.wact = w0 < tb + h0.x && w0 + 32 > tb;
  if (!r.wact) return;
  int t = (int)threadIdx.x - tb;
  r.active = (unsigned)t < (unsigned)h0.x;
  t = r.active ? t : 0;  // inactive lanes read row 0 (in bounds); their results are not stored
  const int32_t* info = reinterpret_cast<const int32_t*>(seg + 48);
  const uint8_t* p = seg + 48 + 4 * S;
  const int gp = h0.w + t;
  r.ridx = (gp - base) & mask;
  vt<NV> x = vld<NV>(rbuf, gp - rbase);
  const int inf = info[t];
  if (UPPER) {
    const double* d = reinterpret_cast<const double*>(p);
    r.invd = d[t];
    if (h0.z & 4) {  // explicit sd / rcp arrays
      x = div_sd(x, d[S + t], d[2 * S + t]);
      p += 24 * S;
    } else {         // info bit 31: sd = 1 - 2^-53 (rcp = 1 + 2^-52), else sd = 1
      if (inf < 0) x = div_sd(x, 0x1.fffffffffffffp-1, 0x1.0000000000001p+0);
      p += 8 * S;
    }
    const int row = inf & 0x3fffffff;
    r.zidx = (inf & 0x40000000) ? gp : -1;  // only far-dependency targets go to global z
    r.xidx = XPOS ? gp : row;  // x in U-position order when only this kernel's F reads it
    r.cadd = (cadd && r.active) ? vldg<NV>(cadd, row) : vzero<NV>();
  } else {
    r.zidx = inf;
  }
  r.acc = x;
  r.slots = p + 8 * t;
  r.s0 = *reinterpret_cast<const uint2*>(r.slots);
  const unsigned z2 = (unsigned)zslot | ((unsigned)zslot << 16);
  r.s1 = (G > 1) ? *reinterpret_cast<const uint2*>(r.slots + 8 * S) : make_uint2(z2, z2);
  r.vals = p + 8 * G * S + 16 * t;
  r.va = *reinterpret_cast<const double2*>(r.vals);
  r.vb = *reinterpret_cast<const double2*>(r.vals + 16 * S);
  r.far = reinterpret_cast<const int32_t*>(seg + h1.z);
}

// dependency value: near -> ring slot, far (bit 15) -> the segment's far list -> global
// position-ordered array
template <bool FAR, int NV>
__device__ __forceinline__ vt<NV> gather(const double* ring, const double* z, const int32_t* far, unsigned sl) {
  return (FAR && (sl & 0x8000u)) ? vld<NV>(z, far[sl & 0x7fffu]) : vld<NV>(ring, sl);
}

template <bool FAR, int NV>
__device__ __forceinline__ vt<NV> fold4(vt<NV> acc, uint2 s, double2 va, double2 vb, const double* ring,
                                        const double* z, const int32_t* far) {
  const vt<NV> z0 = gather<FAR, NV>(ring, z, far, s.x & 0xffffu), z1 = gather<FAR, NV>(ring, z, far, s.x >> 16);
  const vt<NV> z2 = gather<FAR, NV>(ring, z, far, s.y & 0xffffu), z3 = gather<FAR, NV>(ring, z, far, s.y >> 16);
  acc = vmsub(acc, va.x, z0);
  acc = vmsub(acc, va.y, z1);
  acc = vmsub(acc, vb.x, z2);
  acc = vmsub(acc, vb.y, z3);
  return acc;
}

// acc -= val_k * z_k over the row's groups in the reference's ascending-column order
// (padding entries: 0 * 0); group 0's slots and values are in registers.
template <bool FAR, int NV>
__device__ __forceinline__ vt<NV> fold_row(vt<NV> acc, const Row<NV>& r, const double* ring, const double* z) {
  acc = fold4<FAR, NV>(acc, r.s0, r.va, r.vb, ring, z, r.far);
  if (r.G > 1) {
    const uint8_t* v = r.vals + 32 * r.S;  // group 1 values
    acc = fold4<FAR, NV>(acc, r.s1, *reinterpret_cast<const double2*>(v),
                         *reinterpret_cast<const double2*>(v + 16 * r.S), ring, z, r.far);
    for (int g = 2; g < r.G; ++g) {  // long rows: the rest straight from the staged segment
      const uint2 sg = *reinterpret_cast<const uint2*>(r.slots + 8 * g * r.S);
      const uint8_t* w = r.vals + 32 * g * r.S;
      acc = fold4<FAR, NV>(acc, sg, *reinterpret_cast<const double2*>(w),
                           *reinterpret_cast<const double2*>(w + 16 * r.S), ring, z, r.far);
    }
  }
  return acc;
}

struct Cursor {
  int u, u1, st, nst, si, nseg, rbase;
  uint32_t par;
  const uint8_t* seg;
  const double* rbuf;
};

template <bool UPPER, int NV, bool XPOS = false>
__device__ __forceinline__ bool level_step(const StepConst& K, Ctl* ctl, uint8_t* stages, double* rhsbuf,
                                           Cursor& c, Row<NV>& cur, const double* ring_c,
                                           double* ring, int base, double* z, double* xout,
                                           const double* cadd) {
  const int mask = K.ring_mask, zslot = K.ring_mask + 1;
  // C: locate the next segment (next chunk: wait for it; it is normally staged already)
  //    and issue its header loads, so they are in flight while this row is computed
  const uint8_t* nseg_ptr = c.seg + cur.bytes;
  const int cur_st = c.st;
  bool chunk_done = false, more = true;
  if (++c.si == c.nseg) {
    chunk_done = true;
    if (++c.u == c.u1) {
      more = false;
    } else {
      if (++c.st == c.nst) {
        c.st = 0;
        c.par ^= 1u;
      }
      trace_fine(K, 19, c.u);
#if PSLR_TRACE_BUILD == 3
      const long long tw0 = clock64();
      mbar_wait(&ctl->full[c.st], c.par);
      trace_clk(K, 51, (int)(clock64() - tw0));
#else
      mbar_wait(&ctl->full[c.st], c.par);
#endif
      trace_fine(K, 20, c.u);
      nseg_ptr = stages + (size_t)c.st * K.stage_bytes;
      c.rbuf = rhsbuf + (size_t)c.st * K.rhs_stride;
      c.nseg = reinterpret_cast<const int32_t*>(nseg_ptr)[6];
      c.rbase = reinterpret_cast<const int32_t*>(nseg_ptr)[7];
      c.si = 0;
    }
  }
  int4 nh0 = make_int4(0, 0, 0, 0), nh1 = make_int4(0, 0, 0, 0);
  if (more) {
    nh0 = *reinterpret_cast<const int4*>(nseg_ptr);
    nh1 = make_int4(reinterpret_cast<const int32_t*>(nseg_ptr)[4], reinterpret_cast<const int32_t*>(nseg_ptr)[5],
                    reinterpret_cast<const int32_t*>(nseg_ptr)[8], 0);  // S, bytes, far_off
  }
  if (cur.wact) {
    // A + D: gathers and the chain
    const vt<NV> acc = (cur.flags & 2) ? fold_row<true, NV>(cur.acc, cur, ring_c, z)
                                       : fold_row<false, NV>(cur.acc, cur, ring_c, z);
    // F: publish the row
    if (cur.active) {
      vst(ring, cur.ridx, acc);
      if (!UPPER || cur.zidx >= 0) vst(z, cur.zidx, acc);
      if (UPPER) {
        vt<NV> x = vmul(acc, cur.invd);
        if (cadd) x = vadd(x, cur.cadd);
        vst(xout, cur.xidx, x);
      }
    }
  }
  const int cur_flags = cur.flags;
  const int cur_info = (cur.G << 2) | (cur.nrows << 8);
  // E: the next segment's row, loaded in place (everything it needs before its gathers)
  if (more) load_row<UPPER, NV, XPOS>(nseg_ptr, nh0, nh1, c.rbuf, c.rbase, base, mask, zslot, cadd, cur);
  c.seg = nseg_ptr;
  if (chunk_done) {  // the staged chunk is no longer read by this warp
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&ctl->empty[cur_st]);
  }
  if (cur_flags & 1) {
    trace_fine(K, 40, 0);
    consumer_sync();
    trace_fine(K, 41, 0);
  }
  trace_clk(K, 50, (cur_flags & 1) | (chunk_done ? 2 : 0) | cur_info);
  return more;
}

// Consumer side of one triangular phase.  Callers arrive right after a consumer barrier
// that follows the last write of the phase's rhs array; the phase ends with the barrier
// of its last level.
template <bool UPPER, int NV, bool XPOS = false>
__device__ void tri_phase(const StepConst& K, const Streams& S, Ctl* ctl, uint8_t* stages,
                          double* rhsbuf, int k, double* ring, int base, double* z, double* xout,
                          const double* cadd) {
  trace_ev(K, 10 + k, 0);
  trace_cta(K, 2 + k);
  if (threadIdx.x == 0) {
    __threadfence();
    fence_proxy_async();
    mbar_arrive(&ctl->rhs_ready[k]);
  }
  Cursor c;
  c.u = S.begin[k];
  c.u1 = S.begin[k + 1];
  if (c.u == c.u1) return;
  c.nst = K.nst;
  c.st = c.u % c.nst;
  c.par = (uint32_t)((c.u / c.nst) & 1);
  mbar_wait(&ctl->full[c.st], c.par);
  trace_fine(K, 20, c.u);
  c.seg = stages + (size_t)c.st * K.stage_bytes;
  c.rbuf = rhsbuf + (size_t)c.st * K.rhs_stride;
  c.nseg = reinterpret_cast<const int32_t*>(c.seg)[6];
  c.rbase = reinterpret_cast<const int32_t*>(c.seg)[7];
  c.si = 0;
  Row<NV> row;
  {
    const int32_t* h = reinterpret_cast<const int32_t*>(c.seg);
    load_row<UPPER, NV, XPOS>(c.seg, *reinterpret_cast<const int4*>(c.seg), make_int4(h[4], h[5], h[8], 0), c.rbuf,
                        c.rbase, base, K.ring_mask, K.ring_mask + 1, cadd, row);
  }
  const double* ring_c = ring;
  while (level_step<UPPER, NV, XPOS>(K, ctl, stages, rhsbuf, c, row, ring_c, ring, base, z, xout, cadd)) {
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
    default:
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = vzero<NV>();
  }
}

#ifndef PSLR_STEP_MINB
#define PSLR_STEP_MINB 1
#endif
template <int NV, bool XPOS>
__global__ void __launch_bounds__(kBlockThreads, PSLR_STEP_MINB)
subdomain_step_kernel(const __grid_constant__ StepArgs a, const __grid_constant__ StepConst K) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int b = blockIdx.x;
  const bool do_b = a.b1 != BT_NONE;
  const bool do_i = a.i1 != IT_NONE;
  const bool do_c = do_i && a.do_c0;

  Ctl* ctl = reinterpret_cast<Ctl*>(smem);
  // [Ctl 256 B][ring: (W + zero slot) x NV, padded to 128 B][nst stages][nst rhs slices]
  // The ring sits at a constant offset, so a gather is one address op on its slot.
  double* ring = reinterpret_cast<double*>(smem + 256);
  uint8_t* stages = smem + 256 + (size_t)(K.ring_mask + 1) * 8 * NV + 128;
  double* rhsbuf = reinterpret_cast<double*>(stages + (size_t)K.nst * K.stage_bytes);

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
      mbar_init(&ctl->empty[s], kConsumerWarps);
    }
    for (int k = 0; k < 4; ++k) mbar_init(&ctl->rhs_ready[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= kStepThreads) {  // producer warp (all 32 lanes)
    producer(S, ctl, stages, rhsbuf, K.nst, K.stage_bytes, K.rhs_stride, NV,
             (K.trace && K.trace_cap >= (1 << 20)) ? K.trace + 2 + 2 * K.trace_cap - 8 * 4096 + b * 8
                                                   : nullptr);
    return;
  }
  // Programmatic dependent launch: this grid may start while the previous kernel of the
  // stream finishes (setup above and the producer's factor stream do not depend on it);
  // consumers wait here for its completion before reading any vector it produced or
  // writing any buffer it may still read.  A no-op for ordinary launches.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (PSLR_TRACE_BUILD && threadIdx.x == 0) g_trace_tag = a.tag;
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
      constexpr int kIn = 8;  // independent loads in flight per thread
      for (int row0 = r0 + tid; row0 < r1; row0 += kIn * kStepThreads) {
        vt<NV> v[kIn];
        int pos[kIn];
#pragma unroll
        for (int j = 0; j < kIn; ++j) {
          const int row = row0 + j * kStepThreads;
          const bool ok = row < r1;
          v[j] = ok ? vldg<NV>(a.f, row) : vzero<NV>();
          pos[j] = ok ? __ldg(K.LB.lpos + row) : 0;
        }
#pragma unroll
        for (int j = 0; j < kIn; ++j)
          if (row0 + j * kStepThreads < r1) vst(K.rhsB, pos[j], v[j]);
      }
    } else {
      for (int p = r0 + tid; p < r1; p += kStepThreads) vst(K.rhsB, p, vzero<NV>());
    }
    // pass 2: rows with E entries get the E y term: f - E y, or E y alone (scipy
    // csr_matvec order), kIn rows per thread in flight; one int4 record per row
    if (a.b1 == BT_EY || a.b2 == BT_EY) {
      if (!a.fL && !ey_only) consumer_sync();
      constexpr int kIn = 4;
      const int e0 = K.erow_off[b], e1 = K.erow_off[b + 1];
      const int4* rec = reinterpret_cast<const int4*>(K.erows);
      for (int i0 = e0 + tid; i0 < e1; i0 += kIn * kStepThreads) {
        int4 r[kIn];
        vt<NV> fv[kIn], sum[kIn];
        int len = 0;
#pragma unroll
        for (int j = 0; j < kIn; ++j) {
          const int i = i0 + j * kStepThreads;
          r[j] = i < e1 ? __ldg(rec + i) : make_int4(0, 0, 0, 0);
          len = max(len, r[j].w - r[j].z);
          sum[j] = vzero<NV>();
        }
#pragma unroll
        for (int j = 0; j < kIn; ++j)
          fv[j] = (a.b1 == BT_F && r[j].w > r[j].z) ? (a.fL ? vld<NV>(a.fL, r[j].x) : vldg<NV>(a.f, r[j].y))
                                                    : vzero<NV>();
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
          if (i0 + j * kStepThreads < e1) vst(rhs, r[j].x, (a.b1 == BT_F) ? vsub(fv[j], sum[j]) : sum[j]);
      }
    }
    consumer_sync();
    trace_ev(K, 3, 0);
    trace_cta(K, 1);
    tri_phase<false, NV>(K, S, ctl, stages, rhsbuf, ph_LB, ring, r0, K.zB, nullptr, nullptr);
    tri_phase<true, NV, XPOS>(K, S, ctl, stages, rhsbuf, ph_UB, ring, r0, K.zB, a.xb, nullptr);
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
    consumer_sync();
    trace_ev(K, 30, 0);
    if (do_c) {
      tri_phase<false, NV>(K, S, ctl, stages, rhsbuf, ph_LC, ring, r0, K.zC, nullptr, nullptr);
      tri_phase<true, NV>(K, S, ctl, stages, rhsbuf, ph_UC, ring, r0, K.zC, a.yout, a.cadd);
    }
  }
  trace_cta(K, 6);
}

int configure_step_kernel(int nv, int smem_bytes) {
  auto set = [&](auto kern) {
    return (int)cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  };
  if (nv == 2) {
    const int e = set(subdomain_step_kernel<2, false>);
    return e ? e : set(subdomain_step_kernel<2, true>);
  }
  const int e = set(subdomain_step_kernel<1, false>);
  return e ? e : set(subdomain_step_kernel<1, true>);
}

int launch_step(const pslr_ctx* ctx, const StepArgs& a_in, cudaStream_t st, int nv) {
  if (ctx->s == 0) return 0;
  // x_B is read only by this launch's F SpMV: store it in U-position order (coalesced
  // stores from the level loop) and read it through the position-mapped F.  Launches
  // whose x_B leaves the kernel (the last step, solve_B) keep row order.
  StepArgs a = a_in;
  a.xpos = (a.b1 != BT_NONE && (a.i1 == IT_FX || a.i2 == IT_FX)) ? 1 : 0;
  const StepConst& K = (nv == 2) ? ctx->K2 : ctx->K;
  // programmatic stream serialization: the step kernel's CTAs (one per subdomain, far
  // fewer than the 148 SMs) launch and stage their first factor chunks while the
  // previous kernel drains; griddepcontrol.wait orders the data accesses
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctx->s);
  cfg.blockDim = dim3(kBlockThreads);
  cfg.dynamicSmemBytes = (size_t)K.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (nv == 2)
    return (int)(a.xpos ? cudaLaunchKernelEx(&cfg, subdomain_step_kernel<2, true>, a, K)
                        : cudaLaunchKernelEx(&cfg, subdomain_step_kernel<2, false>, a, K));
  return (int)(a.xpos ? cudaLaunchKernelEx(&cfg, subdomain_step_kernel<1, true>, a, K)
                      : cudaLaunchKernelEx(&cfg, subdomain_step_kernel<1, false>, a, K));
}

}  // namespace pslr
