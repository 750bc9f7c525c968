// capi.cu — the C-ABI of libpslr.so: device context (upload + streamed-factor
// packing), the hot-path operators of Alg. 3.2 and their launch-level profiling.
// Krylov drivers (Arnoldi, GMRES/FGMRES) are in krylov.cu.  Every entry point
// cites the reference function it replaces (see include/pslr.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pslr_internal.h"
#include "pslr_ops.h"

namespace pslr {

static thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <class T>
static int upload(pslr_ctx* ctx, const std::vector<T>& h, const T** out) {
  if (h.empty()) {
    *out = nullptr;
    return PSLR_OK;
  }
  void* d = nullptr;
  CK(cudaMalloc(&d, h.size() * sizeof(T)));
  ctx->allocations.push_back(d);
  ctx->device_bytes += (int64_t)(h.size() * sizeof(T));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = static_cast<const T*>(d);
  return PSLR_OK;
}

int alloc_scratch(pslr_ctx* ctx, double** p, int64_t count) {
  *p = nullptr;
  if (count <= 0) count = 1;
  void* d = nullptr;
  CK(cudaMalloc(&d, (size_t)count * sizeof(double)));
  CK(cudaMemset(d, 0, (size_t)count * sizeof(double)));
  ctx->allocations.push_back(d);
  ctx->device_bytes += count * (int64_t)sizeof(double);
  *p = static_cast<double*>(d);
  return PSLR_OK;
}

void free_ptr(pslr_ctx* ctx, void* p) {
  if (!p) return;
  auto it = std::find(ctx->allocations.begin(), ctx->allocations.end(), p);
  if (it == ctx->allocations.end()) return;  // not this context's (a clone's shared data)
  ctx->allocations.erase(it);
  cudaFree(p);
}

int ensure(pslr_ctx* ctx, double** p, int64_t* len, int64_t need) {
  if (*len >= need) return PSLR_OK;
  free_ptr(ctx, *p);
  RET(alloc_scratch(ctx, p, need));
  *len = need;
  return PSLR_OK;
}

static int64_t env_int(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoll(v) : dflt;
}

static int check_csr(const pslr_csr& M, int64_t nr, int64_t nc, const char* name) {
  if (M.nrows != nr || M.ncols != nc)
    return fail(PSLR_EDIM, std::string(name) + " has the wrong shape");
  if (M.nnz > 0x7fffffffLL || nr > 0x7fffffffLL)
    return fail(PSLR_EINVAL, std::string(name) + " exceeds the int32 device index range");
  if (nr > 0 && (M.indptr == nullptr || M.indptr[nr] != M.nnz))
    return fail(PSLR_EDIM, std::string(name) + ": indptr does not match nnz");
  return PSLR_OK;
}

static int upload_csr(pslr_ctx* ctx, const pslr_csr& M, DevCsr* out) {
  out->nrows = (int32_t)M.nrows;
  out->ncols = (int32_t)M.ncols;
  out->nnz = (int32_t)M.nnz;
  std::vector<int32_t> ptr(M.nrows + 1, 0);
  for (int64_t i = 0; i <= M.nrows; ++i) ptr[i] = M.nrows ? (int32_t)M.indptr[i] : 0;
  std::vector<int32_t> col(M.indices, M.indices + M.nnz);
  std::vector<double> val(M.data, M.data + M.nnz);
  RET(upload(ctx, ptr, &out->ptr));
  RET(upload(ctx, col, &out->col));
  RET(upload(ctx, val, &out->val));
  return PSLR_OK;
}

// ---------------------------------------------------------------- the packed format
// Everything pslr_ctx_create derives on the host before uploading (level analysis +
// streamed factor chunks): serialisable, so a setup cache can skip it.
struct PackedFactor {
  TriHost H;
  std::vector<int32_t> pos_of_row, row_at_pos;  // L factors: the rhs placement (lpos / lrow)
};
struct PackedSystem {
  int64_t n = 0, p = 0, q = 0, s = 0;
  int64_t W = 0, SB = 0, reach = 0, far = 0;
  int64_t nthr = kStepThreads;       // consumer threads per step CTA = rows per segment
  int64_t levels[4] = {0, 0, 0, 0}, depth[4] = {0, 0, 0, 0}, nnz[4] = {0, 0, 0, 0};
  PackedFactor F[4];                 // LB, UB, LC, UC
  // the factor streams again at the two-vector launches' chunk size SB2 (empty: SB2 == SB):
  // one vector per launch (the latency a GMRES iteration sees) prefers larger chunks and
  // fewer stages, two vectors per launch (whose ring and rhs slices are twice as large)
  // more stages
  int64_t SB2 = 0;
  TriHost H2[4];
  std::vector<int32_t> ub_pos;       // U_B: row -> U-position (x order, Fpos columns)
  std::vector<int32_t> lb_pos;       // L_B: row -> L-position (E rows' rhs placement)
  // level-merged factors (PSLR_MERGE bit f/2: 1 = L_B/U_B, 2 = L_C0/U_C0; pack.cpp
  // merge_levels): each factor's rhs transform in the position space of the array it
  // rewrites, and L_B's again in row space (permute_f, E' = E - N E)
  int64_t merged = 0;
  std::vector<int32_t> blk_levels;   // per block: L_B + U_B dependency levels (L2 residency)
  MergeXf X[4];
  MergeXf XLBrow;
};

constexpr uint64_t kPackMagic = 0x37764b4150524c53ull;  // "SLRPAKv7" (v6 + the two-vector packing's own segment height)

// Stages of the step kernel's pipeline for chunk size sb and nv vectors per launch: what
// the shared memory holds beside the control block and the (nv-wide) value ring, at most 8
// (PSLR_MAX_STAGES caps it); a chunk's rhs slice travels inside its stage.
static int64_t stage_count(int64_t smem_optin, int64_t W, int64_t sb, int64_t nv) {
  const int64_t n = (smem_optin - 1024 - kCtlBytes - W * 8 * nv - 128) / sb;
  const int64_t cap = nv == 1 ? env_int("PSLR_MAX_STAGES", 8) : env_int("PSLR_MAX_STAGES2", 8);
  return std::min<int64_t>(n, std::min<int64_t>(8, cap));
}

// Level analysis of the four factors, the ring size W (from the reach and the device's
// shared memory) and the streamed chunks of every block (pack.cpp).
// PSLR_MERGE: 0 = the reference's factors as they are (bit-exact), 1 = level-merged B
// factors, 2 = level-merged C0 factors (default), 3 = both.  PSLR_MERGE_W / _WC: merge only
// level pairs of at most that many rows (B: kStepThreads, C0: 0 = every pair)
// The blob key: mode bits 0-1, the B width limit from bit 2, the C0 width limit from bit 32,
// PSLR_LIST_SCHED (list-scheduled steps, pack.cpp) in bit 31, PSLR_ALT_GROUPS (alternating
// warp groups, pack.cpp) in bits 61-62
static int64_t merge_mode() {
  const int64_t mode = env_int("PSLR_MERGE", 2) & 3;
  const int64_t wB = std::min<int64_t>(std::max<int64_t>(env_int("PSLR_MERGE_W", kStepThreads), 0), (1 << 29) - 1);
  const int64_t wC = std::min<int64_t>(std::max<int64_t>(env_int("PSLR_MERGE_WC", 0), 0), (1 << 29) - 1);
  const int64_t alt = env_int("PSLR_ALT_GROUPS", 1) & 3;
  const int64_t sched = env_int("PSLR_LIST_SCHED", 1) ? 1 : 0;
  return mode | (wB << 2) | (sched << 31) | (wC << 32) | (alt << 61);
}

static int64_t step_threads_for(int64_t levels_LB, int64_t levels_UB, int64_t p) {
  int64_t t = env_int("PSLR_STEP_THREADS_RT", 0);
  if (t <= 0) {
    const int64_t lv = std::max<int64_t>(1, std::min(levels_LB, levels_UB));
    t = (p / lv < 40) ? kNarrowThreads : kStepThreads;  // rows per level of the shallower B factor
  }
  return t <= kNarrowThreads ? kNarrowThreads : kStepThreads;  // the kernel's two instantiations
}

// the two-vector packing's consumer threads (pslr_internal.h kWide2Threads), and whether the
// two-vector launches need a packing of their own (another chunk size or segment height)
static int64_t nthr2_for(int64_t nthr) { return nthr == kStepThreads ? kWide2Threads : nthr; }
static bool separate2(int64_t SB, int64_t SB2, int64_t nthr) { return SB2 != SB || nthr2_for(nthr) != nthr; }

static int pack_system(const pslr_system* sys, const std::vector<int64_t>& ioff, const std::vector<int64_t>& foff,
                       int64_t smem_optin, int64_t SB, int64_t SB2, int64_t wmax, PackedSystem& P) {
  P.n = sys->n;
  P.SB2 = SB2;
  P.p = sys->p;
  P.q = sys->q;
  P.s = sys->s;
  P.SB = SB;
  // level merging (depth halving, pack.cpp merge_levels): the streams carry the merged rows
  P.merged = merge_mode();
  HostCsr mf[4];
  pslr_csr LB = sys->LB, UB = sys->UB, LC = sys->LC, UC = sys->UC;
  if (P.merged & 1) {
    const int64_t wB = (P.merged >> 2) & ((1 << 29) - 1);  // (bit 31: list scheduling)
    RET(merge_levels(sys->LB, ioff, false, wB, mf[0], P.X[0], "L_B"));
    RET(merge_levels(sys->UB, ioff, true, wB, mf[1], P.X[1], "U_B"));
    LB = mf[0].view();
    UB = mf[1].view();
  }
  if (P.merged & 2) {
    const int64_t wC = (P.merged >> 32) & ((1 << 29) - 1);
    RET(merge_levels(sys->LC, foff, false, wC, mf[2], P.X[2], "L_C0"));
    RET(merge_levels(sys->UC, foff, true, wC, mf[3], P.X[3], "U_C0"));
    LC = mf[2].view();
    UC = mf[3].view();
  }
  TriAnalysis aLB, aUB, aLC, aUC;
  // rows of levels wider than a launch's consumer threads are list-scheduled into full steps
  // (pack.cpp list_schedule; PSLR_LIST_SCHED=0: the ASAP dependency levels as they are)
  const int64_t scap = ((P.merged >> 31) & 1) ? std::max<int64_t>(32, env_int("PSLR_SCHED_CAP", kStepThreads)) : 0;
  const int64_t sdel = std::max<int64_t>(0, env_int("PSLR_SCHED_DELAY", 16));
  RET(analyze_factor(LB, ioff, false, aLB, "L_B", scap, sdel));
  RET(analyze_factor(UB, ioff, true, aUB, "U_B", scap, sdel));
  RET(analyze_factor(LC, foff, false, aLC, "L_C0", scap, sdel));
  RET(analyze_factor(UC, foff, true, aUC, "U_C0", scap, sdel));
  P.reach = std::max({aLB.reach, aUB.reach, aLC.reach, aUC.reach, (int64_t)1});
  int64_t W = 2048;  // >= 2048: the ring doubles as the V^T y reduction scratch
  while (W < P.reach && W < wmax) W *= 2;
  while (W > 2048 && (smem_optin - 1024 - kCtlBytes - W * 8 - 128) / SB < 2) W /= 2;
  P.W = W;
  // Consumer threads per step CTA (= rows per segment).  Systems whose B levels are narrow
  // (2D grids: cfg4 averages 18 rows per level, cfg1 2) run with 4 consumer warps instead of
  // 15: the level barrier and the idle warps' header walks are most of such a level (cfg4
  // solve_B 1,083 -> 937 us, cfg1 445 -> 377 us; the 3D configs, 50-500 rows per level, are
  // 15-30 % slower with 128 threads and keep 480).  PSLR_STEP_THREADS_RT overrides.
  P.nthr = step_threads_for(aLB.levels, aUB.levels, sys->p);
  const TriAnalysis* an[4] = {&aLB, &aUB, &aLC, &aUC};
  const pslr_csr* M[4] = {&LB, &UB, &LC, &UC};
  const pslr_csr* M0[4] = {&sys->LB, &sys->UB, &sys->LC, &sys->UC};
  const char* nm[4] = {"L_B", "U_B", "L_C0", "U_C0"};
  for (int f = 0; f < 4; ++f) {
    P.levels[f] = an[f]->levels;
    P.depth[f] = an[f]->depth_max;
    P.nnz[f] = M0[f]->nnz;  // the system's factors (blob validation)
  }
  // the merged rows' rhs transforms: L_B's in row space too, then every record in the
  // position space of the array it rewrites (L: L-positions, U: U-positions)
  P.XLBrow = P.X[0];
  for (int f = 0; f < 4; ++f)
    for (auto& v : P.X[f].rows) v = an[f]->pos_of_row[v];
  // far-ring capacity of each launch width: the shared memory a launch's stage plan leaves
  // beside the ring (PSLR_FAR_SLOTS caps it; 0 = every far dependency read from global)
  auto far_cap = [&](int64_t sb, int64_t nv) -> int64_t {
    const int64_t nst = stage_count(smem_optin, W, sb, nv);
    const int64_t left = smem_optin - 1024 - kCtlBytes - nst * sb;
    return std::max<int64_t>(0, std::min<int64_t>(left / (8 * nv) - W - 17, env_int("PSLR_FAR_SLOTS", 1 << 14)));
  };
  const bool sep2 = separate2(SB, SB2, P.nthr);
  const int64_t fr1 = sep2 ? far_cap(SB, 1) : std::min(far_cap(SB, 1), far_cap(SB, 2));
  const int64_t fr2 = far_cap(SB2, 2);
  // a chunk's rhs slice shares its stage (8 B per row and vector)
  const int64_t rr1 = sep2 ? 8 : 16, rr2 = 16;
  // U first: L's output lands at the U-positions, where every value lives globally
  for (int pair = 0; pair < 2; ++pair) {
    const TriAnalysis& AL = *an[2 * pair];
    const TriAnalysis& AU = *an[2 * pair + 1];
    // narrow levels on alternating consumer warp groups (pack.cpp emit_factor): bit 0 the
    // one-vector packing, bit 1 the two-vector packing
    const bool alt1 = (P.merged >> 61) & 1, alt2 = (P.merged >> 62) & 1;
    const int64_t nr = M[2 * pair]->nrows;
    std::vector<int32_t> row_id(nr);
    for (int64_t i = 0; i < nr; ++i) row_id[i] = (int32_t)i;
    const auto& off = pair == 0 ? ioff : foff;
    RET(emit_factor(*M[2 * pair + 1], off, AU, W, SB, P.nthr, AU.pos_of_row, row_id, fr1, rr1,
                    P.F[2 * pair + 1].H, nm[2 * pair + 1], alt1));
    RET(emit_factor(*M[2 * pair], off, AL, W, SB, P.nthr, AU.pos_of_row, AU.pos_of_row, fr1, rr1,
                    P.F[2 * pair].H, nm[2 * pair], alt1));
    if (sep2) {
      RET(emit_factor(*M[2 * pair + 1], off, AU, W, SB2, nthr2_for(P.nthr), AU.pos_of_row, row_id, fr2, rr2,
                      P.H2[2 * pair + 1], nm[2 * pair + 1], alt2));
      RET(emit_factor(*M[2 * pair], off, AL, W, SB2, nthr2_for(P.nthr), AU.pos_of_row, AU.pos_of_row, fr2, rr2,
                      P.H2[2 * pair], nm[2 * pair], alt2));
    }
    P.F[2 * pair].pos_of_row = AL.pos_of_row;
    P.F[2 * pair].row_at_pos = AL.row_at_pos;
    P.far += P.F[2 * pair].H.far + P.F[2 * pair + 1].H.far;
  }
  P.ub_pos = aUB.pos_of_row;
  P.lb_pos = aLB.pos_of_row;
  P.blk_levels.assign(P.s, 0);
  for (int64_t b = 0; b < P.s; ++b) P.blk_levels[b] = aLB.blk_depth[b] + aUB.blk_depth[b];
  return PSLR_OK;
}

namespace {
struct Writer {
  std::vector<uint8_t> b;
  template <class T> void put(const T& v) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  template <class T> void vec(const std::vector<T>& v) {
    put<int64_t>((int64_t)v.size());
    const uint8_t* p = reinterpret_cast<const uint8_t*>(v.data());
    b.insert(b.end(), p, p + v.size() * sizeof(T));
  }
};
struct Reader {
  const uint8_t* p;
  int64_t left;
  bool ok = true;
  template <class T> T get() {
    T v{};
    if (left < (int64_t)sizeof(T)) {
      ok = false;
      return v;
    }
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    left -= sizeof(T);
    return v;
  }
  template <class T> void vec(std::vector<T>& v) {
    const int64_t cnt = get<int64_t>();
    if (!ok || cnt < 0 || cnt * (int64_t)sizeof(T) > left) {
      ok = false;
      return;
    }
    v.resize(cnt);
    std::memcpy(v.data(), p, cnt * sizeof(T));
    p += cnt * sizeof(T);
    left -= cnt * sizeof(T);
  }
};
}  // namespace

static void serialize(const PackedSystem& P, std::vector<uint8_t>& out) {
  Writer w;
  w.put(kPackMagic);
  w.put<int64_t>(P.nthr);
  w.put<int64_t>(kChunkRows);
  for (int64_t v : {P.n, P.p, P.q, P.s, P.W, P.SB, P.SB2, P.reach, P.far}) w.put(v);
  for (int f = 0; f < 4; ++f) {
    w.put(P.levels[f]);
    w.put(P.depth[f]);
    w.put(P.nnz[f]);
    w.vec(P.F[f].H.data);
    w.vec(P.F[f].H.chunks);
    w.vec(P.F[f].H.blk_chunk);
    w.put(P.F[f].H.far);
    w.put(P.F[f].H.far_slots);
    w.put(P.H2[f].far_slots);
    w.vec(P.F[f].pos_of_row);
    w.vec(P.F[f].row_at_pos);
    w.vec(P.H2[f].data);
    w.vec(P.H2[f].chunks);
    w.vec(P.H2[f].blk_chunk);
  }
  w.vec(P.ub_pos);
  w.vec(P.lb_pos);
  w.put(P.merged);
  w.vec(P.blk_levels);
  for (int f = 0; f < 5; ++f) {
    const MergeXf& X = f < 4 ? P.X[f] : P.XLBrow;
    w.vec(X.rows);
    w.vec(X.c);
    w.vec(X.blk);
  }
  out.swap(w.b);
}

// a blob packed for this system, this build of the kernel and a ring / stage plan the
// device can hold; anything else is rejected (the caller repacks)
static bool deserialize(const void* blob, int64_t len, const pslr_system* sys, int64_t smem_optin, int64_t SB,
                        int64_t SB2, PackedSystem& P) {
  Reader r{static_cast<const uint8_t*>(blob), len};
  if (r.get<uint64_t>() != kPackMagic) return false;
  P.nthr = r.get<int64_t>();  // the packing's consumer-thread count (step_threads_for)
  if ((P.nthr != kNarrowThreads && P.nthr != kStepThreads) || r.get<int64_t>() != kChunkRows) return false;
  const int64_t want_thr = env_int("PSLR_STEP_THREADS_RT", 0);
  if (want_thr > 0 && P.nthr != (want_thr <= kNarrowThreads ? kNarrowThreads : kStepThreads)) return false;
  P.n = r.get<int64_t>();
  P.p = r.get<int64_t>();
  P.q = r.get<int64_t>();
  P.s = r.get<int64_t>();
  P.W = r.get<int64_t>();
  P.SB = r.get<int64_t>();
  P.SB2 = r.get<int64_t>();
  P.reach = r.get<int64_t>();
  P.far = r.get<int64_t>();
  if (!r.ok || P.n != sys->n || P.p != sys->p || P.q != sys->q || P.s != sys->s || P.SB != SB || P.SB2 != SB2)
    return false;
  const pslr_csr* M[4] = {&sys->LB, &sys->UB, &sys->LC, &sys->UC};
  for (int f = 0; f < 4; ++f) {
    P.levels[f] = r.get<int64_t>();
    P.depth[f] = r.get<int64_t>();
    P.nnz[f] = r.get<int64_t>();
    if (P.nnz[f] != M[f]->nnz) return false;
    r.vec(P.F[f].H.data);
    r.vec(P.F[f].H.chunks);
    r.vec(P.F[f].H.blk_chunk);
    P.F[f].H.far = r.get<int64_t>();
    P.F[f].H.far_slots = r.get<int64_t>();
    P.H2[f].far_slots = r.get<int64_t>();
    r.vec(P.F[f].pos_of_row);
    r.vec(P.F[f].row_at_pos);
    r.vec(P.H2[f].data);
    r.vec(P.H2[f].chunks);
    r.vec(P.H2[f].blk_chunk);
    if ((int64_t)P.F[f].H.blk_chunk.size() != P.s + 1) return false;
    if (separate2(SB, SB2, P.nthr) != ((int64_t)P.H2[f].blk_chunk.size() == P.s + 1)) return false;
  }
  r.vec(P.ub_pos);
  r.vec(P.lb_pos);
  P.merged = r.get<int64_t>();
  if (!r.ok || P.merged != merge_mode()) return false;
  r.vec(P.blk_levels);
  if ((int64_t)P.blk_levels.size() != P.s) return false;
  for (int f = 0; f < 5; ++f) {
    MergeXf& X = f < 4 ? P.X[f] : P.XLBrow;
    r.vec(X.rows);
    r.vec(X.c);
    r.vec(X.blk);
  }
  return r.ok && r.left == 0 && (int64_t)P.ub_pos.size() == P.p && (int64_t)P.lb_pos.size() == P.p &&
         stage_count(smem_optin, P.W, SB, 1) >= 2;
}

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// the fused single-context operators read Cg through internal q-vectors without ghosts
static int unsharded(const pslr_ctx* ctx) {
  if (ctx->nghost)
    return fail(PSLR_EINVAL, "sharded context: use the split apply (pslr_apply_first/mid/horner/last)");
  return PSLR_OK;
}

static int mark(pslr_ctx* ctx, int32_t kind, cudaStream_t st) {
  if (!ctx->prof_on) return PSLR_OK;
  cudaEvent_t ev;
  CK(cudaEventCreate(&ev));
  CK(cudaEventRecord(ev, st));
  ctx->prof_events.push_back(ev);
  ctx->prof_kinds.push_back(kind);
  return PSLR_OK;
}

static int run_step(pslr_ctx* ctx, const StepArgs& a, cudaStream_t st, int nv = 1) {
  CKL(launch_step(ctx, a, st, nv));
  return mark(ctx, a.tag, st);
}

static int run_core(pslr_ctx* ctx, cudaStream_t st) {
  CKL(launch_correction_core(ctx, st));
  return mark(ctx, LK_CORE, st);
}

int set_device(const pslr_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  return PSLR_OK;
}

// ---------------------------------------------------------------- composite operators
int op_solve_B(pslr_ctx* ctx, const double* f, double* x, cudaStream_t st) {
  StepArgs a;
  a.b1 = BT_F;
  a.f = f;
  a.xb = x;
  return run_step(ctx, a, st);
}

int op_solve_C0(pslr_ctx* ctx, const double* g, double* y, cudaStream_t st) {
  StepArgs a;
  a.i1 = IT_G;
  a.g = g;
  a.do_c0 = 1;
  a.yout = y;
  return run_step(ctx, a, st);
}

// out = [C0^{-1}] (F B^{-1} E v - Cg v) [+ cadd]
int op_es_step(pslr_ctx* ctx, const double* v, double* out, int do_c0, const double* cadd,
               cudaStream_t st) {
  StepArgs a;
  a.b1 = BT_EY;
  a.yE = v;
  a.xb = ctx->xb;
  a.i1 = IT_FX;
  a.i2 = IT_CGY;
  a.i2_sub = 1;
  a.yC = v;
  a.do_c0 = do_c0;
  a.cadd = cadd;
  a.yout = out;
  a.tag = (do_c0 && cadd) ? LK_HORNER : LK_STEP;
  return run_step(ctx, a, st);
}

// Horner recurrence of schur.py:89-101 starting from c = C0^{-1} v already in `c`.
int op_horner(pslr_ctx* ctx, int64_t m, const double* c, double* out, cudaStream_t st) {
  if (m == 0) {
    if (out != c) CK(cudaMemcpyAsync(out, c, ctx->q * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return PSLR_OK;
  }
  double* buf[2] = {ctx->y1, ctx->y2};
  const double* src = c;
  for (int64_t t = 1; t <= m; ++t) {
    double* dst = (t == m) ? out : buf[t & 1];
    if (dst == src) dst = buf[(t + 1) & 1];
    RET(op_es_step(ctx, src, dst, 1, c, st));
    src = dst;
  }
  if (src != out) CK(cudaMemcpyAsync(out, src, ctx->q * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return PSLR_OK;
}

int op_apply(pslr_ctx* ctx, int64_t m, const double* b, double* z, cudaStream_t st) {
  if (ctx->comm) return op_apply_sharded(ctx, m, b, z, st);
  const int64_t p = ctx->p, q = ctx->q;
  if (q == 0) return op_solve_B(ctx, b, z, st);
  // (0) f in L-position order, shared by the first and the last step
  if (p > 0) {
    CKL(launch_permute_f(ctx, b, st));
    RET(mark(ctx, LK_PERMUTE, st));
  }
  // (1) y0 = g - F B^{-1} f  (+ per-subdomain V^T y0 partials)   preconditioner.py:89
  {
    StepArgs a;
    a.b1 = BT_F;
    a.f = b;
    a.fL = ctx->fL;
    a.xb = ctx->xb;
    a.i1 = IT_G;
    a.g = b + p;
    a.i2 = IT_FX;
    a.i2_sub = 1;
    a.yout = ctx->y0;
    a.tag = LK_FIRST;
    RET(run_step(ctx, a, st));
  }
  // (2) y1 = y0 + V G V^T y0 (all-SM GEMV kernels) ; c = C0^{-1} y1   preconditioner.py:90, schur.py:97
  double* c = (m == 0) ? z + p : ctx->c;
  const double* y1 = ctx->y0;
  if (ctx->r > 0) {
    CKL(launch_vt_dot(ctx, ctx->y0, st));
    RET(mark(ctx, LK_CORE, st));
    CKL(launch_vu_add(ctx, ctx->y0, ctx->y1, st));
    RET(mark(ctx, LK_CORE, st));
    y1 = ctx->y1;
  }
  {
    StepArgs a;
    a.i1 = IT_G;
    a.g = y1;
    a.do_c0 = 1;
    a.yout = c;
    a.tag = LK_CORR;
    RET(run_step(ctx, a, st));
  }
  // (3) m Horner steps y = C0^{-1}(Es y) + c                     schur.py:99-100
  if (m > 0) RET(op_horner(ctx, m, c, z + p, st));
  // (4) x = B^{-1}(f - E y)                                      preconditioner.py:92
  {
    StepArgs a;
    a.b1 = BT_F;
    a.f = b;
    a.fL = ctx->fL;  // last reader of fL: its E rows become f - E y in place
    a.b2 = BT_EY;
    a.yE = z + p;
    a.xb = z;
    a.tag = LK_LAST;
    RET(run_step(ctx, a, st));
  }
  return PSLR_OK;
}

// ---------------------------------------------------------------- two right-hand sides
// Step constants and interleaved scratch for NV = 2 launches: the ring and the rhs slices
// double, the factor stages stay (fewer of them fit), the factors are shared with NV = 1.
static int ensure_nv2(pslr_ctx* ctx) {
  if (ctx->nv2_ready) return PSLR_OK;
  const int64_t p = ctx->p, q = ctx->q;
  StepConst K2 = ctx->K;
  K2.LB = ctx->tri2[0];
  K2.UB = ctx->tri2[1];
  K2.LC = ctx->tri2[2];
  K2.UC = ctx->tri2[3];
  const int64_t W = (int64_t)ctx->K.ring_mask + 1, SB = ctx->sb2, CTL = kCtlBytes;
  const int64_t nst = stage_count(ctx->smem_optin, W, SB, 2);
  if (nst < 2) return fail(PSLR_EINVAL, "not enough shared memory for two right-hand sides per launch");
  K2.nst = (int)nst;
  K2.nthr = (int)nthr2_for(ctx->K.nthr);
  K2.stage_bytes = (int)SB;
  K2.rhs_stride = 0;  // the rhs slice follows the data inside its stage
  K2.far_slots = (int)ctx->far2;
  K2.smem_bytes = (int)(CTL + (((W + 1 + ctx->far2) * 16 + 127) / 128) * 128 + nst * SB);
  if (configure_step_kernel(2, K2.smem_bytes) != 0)
    return fail(PSLR_ECUDA, "cannot configure the two-vector step kernel's shared memory");
  RET(alloc_scratch(ctx, &K2.rhsB, 2 * (p + 2)));
  RET(alloc_scratch(ctx, &K2.rhsE, 2 * (p + 2)));  // zeroed: only E rows are ever written
  RET(alloc_scratch(ctx, &K2.zB, 2 * (p + 2)));
  RET(alloc_scratch(ctx, &K2.cgy, 2 * (q + 1)));
  RET(alloc_scratch(ctx, &K2.rhsC, 2 * (q + 2)));
  RET(alloc_scratch(ctx, &K2.zC, 2 * (q + 2)));
  RET(alloc_scratch(ctx, &ctx->fL2, 2 * (p + 2)));
  RET(alloc_scratch(ctx, &ctx->g2, 2 * q));
  RET(alloc_scratch(ctx, &ctx->xb2, 2 * p));
  RET(alloc_scratch(ctx, &ctx->xF2, 2 * p));
  RET(alloc_scratch(ctx, &ctx->y0_2, 2 * q));
  RET(alloc_scratch(ctx, &ctx->y1_2, 2 * q));
  RET(alloc_scratch(ctx, &ctx->c2, 2 * q));
  RET(alloc_scratch(ctx, &ctx->yA2, 2 * q));
  RET(alloc_scratch(ctx, &ctx->yB2, 2 * q));
  RET(alloc_scratch(ctx, &ctx->yF2, 2 * q));
  RET(alloc_scratch(ctx, &ctx->io_b2, 2 * ctx->n));
  RET(alloc_scratch(ctx, &ctx->io_z2, 2 * ctx->n));
  CK(cudaDeviceSynchronize());
  ctx->K2 = K2;
  ctx->nv2_ready = true;
  return PSLR_OK;
}

// Alg. 3.2 for two vectors at once (b, z: two n-vectors, vector-major): op_apply with every
// vector interleaved; each vector's arithmetic is the single-vector one bit for bit.
int op_apply2(pslr_ctx* ctx, int64_t m, const double* b, double* z, cudaStream_t st) {
  RET(ensure_nv2(ctx));
  const int64_t q = ctx->q;
  CKL(launch_permute2(ctx, b, st));
  RET(mark(ctx, LK_PERMUTE, st));
  {  // (1) y0 = g - F B^{-1} f
    StepArgs a;
    a.b1 = BT_F;
    a.fL = ctx->fL2;
    a.xb = ctx->xb2;
    a.i1 = IT_G;
    a.g = ctx->g2;
    a.i2 = IT_FX;
    a.i2_sub = 1;
    a.yout = ctx->y0_2;
    a.tag = LK_FIRST;
    RET(run_step(ctx, a, st, 2));
  }
  // (2) y1 = y0 + V G V^T y0 per vector ; c = C0^{-1} y1
  const double* y1 = ctx->y0_2;
  if (ctx->r > 0) {
    for (int v = 0; v < 2; ++v) {
      CKL(launch_vt_dot_strided(ctx, ctx->y0_2 + v, 2, st));
      CKL(launch_vu_add_strided(ctx, ctx->y0_2 + v, 2, ctx->y1_2 + v, 2, st));
    }
    RET(mark(ctx, LK_CORE, st));
    y1 = ctx->y1_2;
  }
  double* c = (m == 0) ? ctx->yF2 : ctx->c2;
  {
    StepArgs a;
    a.i1 = IT_G;
    a.g = y1;
    a.do_c0 = 1;
    a.yout = c;
    a.tag = LK_CORR;
    RET(run_step(ctx, a, st, 2));
  }
  // (3) m Horner steps y = C0^{-1}(Es y) + c
  const double* src = c;
  for (int64_t t = 1; t <= m; ++t) {
    double* dst = (t == m) ? ctx->yF2 : ((t & 1) ? ctx->yA2 : ctx->yB2);
    StepArgs a;
    a.b1 = BT_EY;
    a.yE = src;
    a.xb = ctx->xb2;
    a.i1 = IT_FX;
    a.i2 = IT_CGY;
    a.i2_sub = 1;
    a.yC = src;
    a.do_c0 = 1;
    a.cadd = c;
    a.yout = dst;
    a.tag = LK_HORNER;
    RET(run_step(ctx, a, st, 2));
    src = dst;
  }
  {  // (4) x = B^{-1}(f - E y)
    StepArgs a;
    a.b1 = BT_F;
    a.fL = ctx->fL2;
    a.b2 = BT_EY;
    a.yE = ctx->yF2;
    a.xb = ctx->xF2;
    a.tag = LK_LAST;
    RET(run_step(ctx, a, st, 2));
  }
  (void)q;
  CKL(launch_deinterleave2(ctx, ctx->yF2, z, st));
  return PSLR_OK;
}

int op_apply_err(pslr_ctx* ctx, int64_t m, const double* v, double* out, cudaStream_t st) {
  if (ctx->comm) return op_apply_err_sharded(ctx, m, v, out, st);
  if (ctx->q == 0) return PSLR_OK;
  double* buf[2] = {ctx->y1, ctx->y2};
  RET(op_solve_C0(ctx, v, buf[0], st));
  const double* src = buf[0];
  for (int64_t t = 1; t <= m + 1; ++t) {
    const bool last = (t == m + 1);
    double* dst = last ? out : buf[t & 1];
    if (dst == src) dst = buf[(t + 1) & 1];
    RET(op_es_step(ctx, src, dst, last ? 0 : 1, nullptr, st));
    src = dst;
  }
  if (src != out) CK(cudaMemcpyAsync(out, src, ctx->q * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return PSLR_OK;
}

}  // namespace pslr

using namespace pslr;

extern "C" {

const char* pslr_last_error(void) { return g_last_error.c_str(); }
int pslr_abi_version(void) { return 2; }

int pslr_ctx_create(pslr_ctx** out, int device, const pslr_system* sys) {
  return pslr_ctx_create_packed(out, device, sys, nullptr, 0, nullptr, nullptr, nullptr);
}

void pslr_blob_free(void* blob) { std::free(blob); }

int pslr_ctx_create_packed(pslr_ctx** out, int device, const pslr_system* sys, const void* blob_in,
                           int64_t blob_len, void** blob_out, int64_t* blob_out_len, int* reused) {
  pslr::NvtxRange nvtx_("pslr_ctx_create");
  *out = nullptr;
  if (blob_out) *blob_out = nullptr;
  if (blob_out_len) *blob_out_len = 0;
  if (!sys) return fail(PSLR_EINVAL, "null system");
  const int64_t n = sys->n, p = sys->p, q = sys->q, s = sys->s;
  if (p + q != n || s < 1) return fail(PSLR_EDIM, "inconsistent system dimensions");
  RET(check_csr(sys->LB, p, p, "L_B"));
  RET(check_csr(sys->UB, p, p, "U_B"));
  RET(check_csr(sys->LC, q, q, "L_C0"));
  RET(check_csr(sys->UC, q, q, "U_C0"));
  RET(check_csr(sys->E, p, q, "E"));
  RET(check_csr(sys->F, q, p, "F"));
  // sharded contexts: C, Cg and A carry the same nghost ghost columns (include/pslr.h)
  const int64_t nghost = sys->Cg.ncols - q;
  if (nghost < 0) return fail(PSLR_EDIM, "Cg has the wrong shape");
  RET(check_csr(sys->C, q, q + nghost, "C"));
  RET(check_csr(sys->C0, q, q, "C0"));
  RET(check_csr(sys->Cg, q, q + nghost, "Cg"));
  RET(check_csr(sys->A, n, n + nghost, "A"));
  if (sys->interior_offsets[0] != 0 || sys->interior_offsets[s] != p ||
      sys->interface_offsets[0] != 0 || sys->interface_offsets[s] != q)
    return fail(PSLR_EDIM, "block offsets do not tile the system");
  auto* ctx = new pslr_ctx();
  ctx->device = device;
  ctx->n = n;
  ctx->p = p;
  ctx->q = q;
  ctx->s = s;
  ctx->nghost = nghost;
  ctx->interior_off.assign(sys->interior_offsets, sys->interior_offsets + s + 1);
  ctx->interface_off.assign(sys->interface_offsets, sys->interface_offsets + s + 1);
  int rc = PSLR_OK;
  auto bail = [&](int code) {
    pslr_ctx_destroy(ctx);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(PSLR_ECUDA, "cudaSetDevice failed"));
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (ctx->sm_count <= 0) ctx->sm_count = 148;
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (smem_optin <= 0) smem_optin = 232448;
  smem_optin = (int)std::min<int64_t>(smem_optin, env_int("PSLR_SMEM_CAP", smem_optin));
  pslr_ctx_info_t& I = ctx->info;

  // ---- the packed format: from the caller's blob when it fits this system and device,
  // else level analysis + ring plan + streamed chunks (pack_system)
  // Shared-memory plan: a W-slot value ring, nst stages of SB bytes (a chunk's data and its
  // rhs slice), the far-ring in what is left.
  // stage size (a chunk's data + its rhs slice) of the one-vector launches (SB) and of the
  // two-vector launches (SB2), cfg5 round 2 (tools/stage_plan_sweep.sh, tools/sb_bench.sh):
  // one vector at a time prefers 3 stages of 52 KB (far-ring 4.7 k slots; 56 KB and more
  // shrink the far-ring below the wide blocks' needs), two vectors 4 stages of 36 KB
  const int64_t SB = env_int("PSLR_STAGE_BYTES", 52 * 1024);
  const int64_t SB2 = env_int("PSLR_STAGE_BYTES2", 36 * 1024);
  PackedSystem P;
  const bool reuse = blob_in && blob_len > 0 && deserialize(blob_in, blob_len, sys, smem_optin, SB, SB2, P);
  if (reused) *reused = reuse ? 1 : 0;
  if (!reuse) {
    P = PackedSystem();
    if ((rc = pack_system(sys, ctx->interior_off, ctx->interface_off, smem_optin, SB, SB2,
                          env_int("PSLR_RING", 4096), P)))
      return bail(rc);
  }
  if (blob_out) {
    std::vector<uint8_t> bytes;
    serialize(P, bytes);
    void* mem = std::malloc(bytes.size());
    if (!mem) return bail(fail(PSLR_ENOMEM, "packed-format blob"));
    std::memcpy(mem, bytes.data(), bytes.size());
    *blob_out = mem;
    *blob_out_len = (int64_t)bytes.size();
  }
  const int64_t W = P.W, reach = P.reach;
  const int64_t CTL = kCtlBytes;  // mbarriers + descriptor queue
  const int64_t nst = stage_count(smem_optin, W, SB, 1);
  if (nst < 2) return bail(fail(PSLR_EINVAL, "not enough shared memory for the streamed solve"));
  int64_t fr1 = 0, fr2 = 0;  // far-ring slots of the one- and two-vector packings
  for (int f = 0; f < 4; ++f) {
    fr1 = std::max(fr1, P.F[f].H.far_slots);
    fr2 = std::max(fr2, separate2(SB, SB2, P.nthr) ? P.H2[f].far_slots : P.F[f].H.far_slots);
  }
  ctx->K.ring_mask = (int)(W - 1);
  ctx->K.nthr = (int)P.nthr;
  ctx->K.far_slots = (int)fr1;
  ctx->K.nst = (int)nst;
  ctx->K.stage_bytes = (int)SB;
  ctx->K.rhs_stride = 0;  // the rhs slice follows the data inside its stage
  // ring + zero slot + far-ring (padded to 128 B), then the stages
  ctx->K.smem_bytes = (int)(CTL + (((W + 1 + fr1) * 8 + 127) / 128) * 128 + nst * SB);
  ctx->far2 = fr2;
  ctx->smem_optin = smem_optin;
  if (configure_step_kernel(1, ctx->K.smem_bytes) != 0)
    return bail(fail(PSLR_ECUDA, "cannot configure the step kernel's shared memory"));
  ctx->pdl = env_int("PSLR_PDL", 1) != 0;
  ctx->ey_all_sm = env_int("PSLR_EY_ALLSM", 1) != 0;
  ctx->split_iface = env_int("PSLR_SPLIT_IFACE", 1) != 0;
  ctx->K.dbg = (int)env_int("PSLR_DBG", 0);
  ctx->K.l2ahead = env_int("PSLR_L2AHEAD", 0);
  {  // L2 residency of the deepest blocks' B factor streams (PSLR_L2KEEP_MB, default 0 = off: measured no gain on cfg5): blocks
     // in decreasing dependency depth while their L_B + U_B chunks fit the budget
    const int64_t budget = env_int("PSLR_L2KEEP_MB", 0) << 20;
    if (budget > 0 && s > 0) {
      std::vector<int64_t> order(s), bytes(s, 0);
      for (int64_t b = 0; b < s; ++b) {
        order[b] = b;
        for (int f = 0; f < 2; ++f)
          for (int32_t c = P.F[f].H.blk_chunk[b]; c < P.F[f].H.blk_chunk[b + 1]; ++c) bytes[b] += P.F[f].H.chunks[c].bytes;
      }
      std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t c) { return P.blk_levels[a] > P.blk_levels[c]; });
      std::vector<int8_t> keep(s, 0);
      int64_t used = 0;
      for (int64_t b : order) {
        if (used + bytes[b] > budget) break;
        used += bytes[b];
        keep[b] = 1;
      }
      if (used > 0 && (rc = upload(ctx, keep, &ctx->K.l2keep))) return bail(rc);
    }
  }
  if (env_int("PSLR_TRACE", 0)) {  // diagnostics: timeline of CTA 0 (pslr_debug_trace)
    const int64_t cap = 1 << 20;
    void* d = nullptr;
    if (cudaMalloc(&d, (2 + 2 * cap) * sizeof(long long)) != cudaSuccess)
      return bail(fail(PSLR_ECUDA, "cudaMalloc trace"));
    cudaMemset(d, 0, 16);
    ctx->allocations.push_back(d);
    ctx->K.trace = static_cast<long long*>(d);
    ctx->K.trace_cap = cap;
    ctx->K.trace_block = env_int("PSLR_TRACE_CTA", 0);
  }
  {
    DevTri* dt[4] = {&ctx->K.LB, &ctx->K.UB, &ctx->K.LC, &ctx->K.UC};
    for (int f = 0; f < 4; ++f) {
      const PackedFactor& F = P.F[f];
      dt[f]->nblocks = (int32_t)F.H.blk_chunk.size() - 1;
      dt[f]->nchunks = (int32_t)F.H.chunks.size();
      if ((rc = upload(ctx, F.H.data, &dt[f]->data))) return bail(rc);
      if ((rc = upload(ctx, F.H.chunks, &dt[f]->chunks))) return bail(rc);
      if ((rc = upload(ctx, F.H.blk_chunk, &dt[f]->blk_chunk))) return bail(rc);
      if (!(f & 1)) {  // L factors: rhs placement
        if ((rc = upload(ctx, F.pos_of_row, &dt[f]->lpos))) return bail(rc);
        if ((rc = upload(ctx, F.row_at_pos, &dt[f]->lrow))) return bail(rc);
      }
      // the two-vector launches' streams (same positions, other chunk boundaries)
      ctx->tri2[f] = *dt[f];
      if (separate2(SB, SB2, P.nthr)) {
        const TriHost& H2 = P.H2[f];
        ctx->tri2[f].nchunks = (int32_t)H2.chunks.size();
        if ((rc = upload(ctx, H2.data, &ctx->tri2[f].data))) return bail(rc);
        if ((rc = upload(ctx, H2.chunks, &ctx->tri2[f].chunks))) return bail(rc);
        if ((rc = upload(ctx, H2.blk_chunk, &ctx->tri2[f].blk_chunk))) return bail(rc);
      }
    }
    ctx->sb2 = SB2;
  }
  I.levels_LB = P.levels[0];
  I.levels_UB = P.levels[1];
  I.levels_LC = P.levels[2];
  I.levels_UC = P.levels[3];
  I.maxdepth_LB = P.depth[0];
  I.maxdepth_UB = P.depth[1];
  I.maxdepth_LC = P.depth[2];
  I.maxdepth_UC = P.depth[3];
  I.ring_slots = W;
  I.stages = nst;
  I.far_deps = P.far;
  I.reach = reach;

  // level-merged factors: the in-place rhs transforms of the merged rows; L_B's also as
  // the permute_f gather map (lrowx) and folded into E (E' = E - N E: the E y rows of the
  // L_B right-hand side arrive transformed)
  HostCsr Em;
  pslr_csr Eu = sys->E;
  {
    DevXform* dx[4] = {&ctx->K.XLB, &ctx->K.XUB, &ctx->K.XLC, &ctx->K.XUC};
    for (int f = 0; f < 4; ++f) {
      const MergeXf& X = P.X[f];
      if (X.blk.empty() || X.rows.empty()) continue;
      dx[f]->nrec = (int32_t)(X.rows.size() / kXfWidth1);
      if ((rc = upload(ctx, X.rows, &dx[f]->idx))) return bail(rc);
      if ((rc = upload(ctx, X.c, &dx[f]->val))) return bail(rc);
      if ((rc = upload(ctx, X.blk, &dx[f]->blk))) return bail(rc);
    }
    const MergeXf& XL = P.XLBrow;
    const int64_t nrec = (int64_t)(XL.rows.size() / kXfWidth1);
    if (nrec > 0) {
      std::vector<int32_t> lrowx = P.F[0].row_at_pos;
      for (int64_t k = 0; k < nrec; ++k) lrowx[P.lb_pos[XL.rows[kXfWidth1 * k]]] = (int32_t)(-(k + 1));
      if ((rc = upload(ctx, lrowx, &ctx->K.lrowx))) return bail(rc);
      if ((rc = upload(ctx, XL.rows, &ctx->K.xlb_rows))) return bail(rc);
      // E'_i = E_i - sum_j c_ij E_j over the record of each merged row i
      const pslr_csr& E = sys->E;
      std::vector<int64_t> rec_of(p, -1);
      for (int64_t k = 0; k < nrec; ++k) rec_of[XL.rows[kXfWidth1 * k]] = k;
      Em.nrows = E.nrows;
      Em.ncols = E.ncols;
      Em.indptr.assign(p + 1, 0);
      std::vector<double> acc(q, 0.0);
      std::vector<uint8_t> used(q, 0);
      std::vector<int32_t> cols;
      for (int64_t i = 0; i < p; ++i) {
        const int64_t k = rec_of[i];
        if (k < 0) {
          for (int64_t e = E.indptr[i]; e < E.indptr[i + 1]; ++e) {
            Em.indices.push_back(E.indices[e]);
            Em.data.push_back(E.data[e]);
          }
        } else {
          cols.clear();
          auto add = [&](int32_t j, double v) {
            if (!used[j]) {
              used[j] = 1;
              acc[j] = 0.0;
              cols.push_back(j);
            }
            acc[j] += v;
          };
          for (int64_t e = E.indptr[i]; e < E.indptr[i + 1]; ++e) add(E.indices[e], E.data[e]);
          for (int a = 0; a < kXfWidth; ++a) {
            const int64_t j = XL.rows[kXfWidth1 * k + 1 + a];
            const double c = XL.c[kXfWidth1 * k + a];
            if (c == 0.0) continue;
            for (int64_t e = E.indptr[j]; e < E.indptr[j + 1]; ++e) add(E.indices[e], -c * E.data[e]);
          }
          std::sort(cols.begin(), cols.end());
          for (int32_t j : cols) {
            used[j] = 0;
            Em.indices.push_back(j);
            Em.data.push_back(acc[j]);
          }
        }
        Em.indptr[i + 1] = (int64_t)Em.indices.size();
      }
      Em.nnz = (int64_t)Em.indices.size();
      Eu = Em.view();
    }
  }
  if ((rc = upload_csr(ctx, Eu, &ctx->K.E))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->F, &ctx->K.F))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->C, &ctx->K.C))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->C0, &ctx->C0))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->Cg, &ctx->K.Cg))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->A, &ctx->A))) return bail(rc);
  {
    std::vector<int32_t> io(s + 1), fo(s + 1);
    for (int64_t b = 0; b <= s; ++b) {
      io[b] = (int32_t)ctx->interior_off[b];
      fo[b] = (int32_t)ctx->interface_off[b];
    }
    if ((rc = upload(ctx, io, &ctx->K.int_off))) return bail(rc);
    if ((rc = upload(ctx, fo, &ctx->K.ifc_off))) return bail(rc);
    // interior rows that carry E entries (~30% on the stencil configs), per block, as
    // {L-position, row, E row start, E row end}: one 16-B load per row in the prepass
    std::vector<int32_t> er, eo(s + 1, 0);
    for (int64_t b = 0; b < s; ++b) {
      for (int64_t i = ctx->interior_off[b]; i < ctx->interior_off[b + 1]; ++i)
        if (Eu.indptr[i + 1] > Eu.indptr[i]) {
          er.push_back(P.lb_pos[i]);
          er.push_back((int32_t)i);
          er.push_back((int32_t)Eu.indptr[i]);
          er.push_back((int32_t)Eu.indptr[i + 1]);
        }
      eo[b + 1] = (int32_t)(er.size() / 4);
    }
    ctx->K.nerows = eo[s];
    if (er.empty()) er.assign(4, 0);
    if ((rc = upload(ctx, er, &ctx->K.erows))) return bail(rc);
    if ((rc = upload(ctx, eo, &ctx->K.erow_off))) return bail(rc);
  }
  // position-ordered rhs arrays: +2 so a chunk's even-aligned TMA slice stays in bounds
  if ((rc = alloc_scratch(ctx, &ctx->K.rhsB, p + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.rhsE, p + 2))) return bail(rc);  // zeroed
  if ((rc = alloc_scratch(ctx, &ctx->K.zB, p + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.cgy, q + 1))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.rhsC, q + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.zC, q + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->xb, p))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->fL, p + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->y0, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->y1, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->y2, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->c, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->kw, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->kt, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->kr, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->io_b, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->io_z, n))) return bail(rc);
  {
    void* d = nullptr;
    if (cudaMalloc(&d, 64) != cudaSuccess) return bail(fail(PSLR_ECUDA, "cudaMalloc counter"));
    cudaMemset(d, 0, 64);
    ctx->allocations.push_back(d);
    ctx->counter = static_cast<unsigned int*>(d);
  }
  I.n = n;
  I.p = p;
  I.q = q;
  I.s = s;
  I.nnz_LB = sys->LB.nnz;
  I.nnz_UB = sys->UB.nnz;
  I.nnz_LC = sys->LC.nnz;
  I.nnz_UC = sys->UC.nnz;
  I.nnz_E = sys->E.nnz;
  I.nnz_F = sys->F.nnz;
  I.nnz_C = sys->C.nnz;
  I.nnz_C0 = sys->C0.nnz;
  I.nnz_Cg = sys->Cg.nnz;
  I.nnz_A = sys->A.nnz;
  I.sm_count = ctx->sm_count;
  I.nghost = nghost;
  {  // F over U-positions: same rows, entry order and values, columns renumbered (allocated
     // last: the other arrays keep the placement they were tuned with)
    pslr_csr Fp = sys->F;
    std::vector<int32_t> pcol(sys->F.indices, sys->F.indices + sys->F.nnz);
    for (auto& j : pcol) j = P.ub_pos[j];
    Fp.indices = pcol.data();
    if ((rc = upload_csr(ctx, Fp, &ctx->K.Fpos))) return bail(rc);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(PSLR_ECUDA, "upload failed"));
  *out = ctx;
  return PSLR_OK;
}

int pslr_workspace_create(pslr_ctx** out, int device) {
  *out = nullptr;
  auto* ctx = new pslr_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return fail(PSLR_ECUDA, "cudaSetDevice failed");
  }
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (ctx->sm_count <= 0) ctx->sm_count = 148;
  void* d = nullptr;
  if (cudaMalloc(&d, 64) != cudaSuccess) {
    delete ctx;
    return fail(PSLR_ECUDA, "cudaMalloc counter");
  }
  cudaMemset(d, 0, 64);
  ctx->allocations.push_back(d);
  ctx->counter = static_cast<unsigned int*>(d);
  *out = ctx;
  return PSLR_OK;
}

void pslr_ctx_destroy(pslr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  comm_destroy(ctx);
  for (void* p : ctx->allocations) cudaFree(p);
  for (cudaEvent_t ev : ctx->prof_events) cudaEventDestroy(ev);
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  for (cudaEvent_t ev : ctx->kev)
    if (ev) cudaEventDestroy(ev);
  delete ctx;
}

int pslr_ctx_info(const pslr_ctx* ctx, pslr_ctx_info_t* info) {
  *info = ctx->info;
  info->rank = ctx->r;
  info->device_bytes = ctx->device_bytes;
  return PSLR_OK;
}

static int set_correction_common(pslr_ctx* ctx, int64_t r, const double* V, bool V_on_device,
                                 const double* G) {
  if (r < 0) return fail(PSLR_EDIM, "rank must be >= 0");
  if (ctx->parent) return fail(PSLR_EINVAL, "a cloned context shares its parent's correction");
  if (ctx->family.use_count() > 1)
    return fail(PSLR_EINVAL, "the context has live clones sharing its correction: destroy them first");
  RET(set_device(ctx));
  free_ptr(ctx, ctx->V);
  free_ptr(ctx, ctx->G);
  free_ptr(ctx, ctx->partials);
  free_ptr(ctx, ctx->u);
  ctx->V = ctx->G = ctx->partials = ctx->u = nullptr;
  ctx->r = 0;
  ctx->K.V = nullptr;
  ctx->K.r = 0;
  if (r == 0 || ctx->q == 0) return PSLR_OK;
  RET(alloc_scratch(ctx, &ctx->V, ctx->q * r));
  RET(alloc_scratch(ctx, &ctx->G, r * r));
  RET(alloc_scratch(ctx, &ctx->partials, ctx->s * r));
  RET(alloc_scratch(ctx, &ctx->u, 2 * r));
  CK(cudaMemcpy(ctx->V, V, ctx->q * r * sizeof(double),
                V_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->G, G, r * r * sizeof(double), cudaMemcpyHostToDevice));
  ctx->r = r;
  ctx->K.V = ctx->V;
  ctx->K.r = (int)r;
  // per-CTA partials of the V^T y reduction
  RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)vt_grid(ctx->q, ctx->sm_count) * r + 8));
  return PSLR_OK;
}

int pslr_ctx_set_correction(pslr_ctx* ctx, int64_t r, const double* V, const double* G) {
  return set_correction_common(ctx, r, V, false, G);
}

int pslr_ctx_set_correction_device(pslr_ctx* ctx, int64_t r, const double* V_dev, const double* G) {
  return set_correction_common(ctx, r, V_dev, true, G);
}

int pslr_solve_B(pslr_ctx* ctx, const double* f, double* x, void* stream) {
  pslr::NvtxRange nvtx_("pslr_solve_B");
  RET(set_device(ctx));
  return op_solve_B(ctx, f, x, S(stream));
}

int pslr_solve_C0(pslr_ctx* ctx, const double* g, double* y, void* stream) {
  pslr::NvtxRange nvtx_("pslr_solve_C0");
  RET(set_device(ctx));
  return op_solve_C0(ctx, g, y, S(stream));
}

int pslr_apply_Es(pslr_ctx* ctx, const double* v, double* out, void* stream) {
  RET(unsharded(ctx));
  RET(set_device(ctx));
  return op_es_step(ctx, v, out, 0, nullptr, S(stream));
}

int pslr_apply_S(pslr_ctx* ctx, const double* v, double* out, void* stream) {
  RET(unsharded(ctx));
  RET(set_device(ctx));
  StepArgs a;
  a.b1 = BT_EY;
  a.yE = v;
  a.xb = ctx->xb;
  a.i1 = IT_CY;
  a.yC = v;
  a.i2 = IT_FX;
  a.i2_sub = 1;
  a.yout = out;
  return run_step(ctx, a, S(stream));
}

int pslr_apply_neumann(pslr_ctx* ctx, int64_t m, const double* v, double* out, void* stream) {
  RET(unsharded(ctx));
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  RET(set_device(ctx));
  RET(op_solve_C0(ctx, v, ctx->c, S(stream)));
  return op_horner(ctx, m, ctx->c, out, S(stream));
}

int pslr_apply_Err(pslr_ctx* ctx, int64_t m, const double* v, double* out, void* stream) {
  pslr::NvtxRange nvtx_("pslr_apply_Err");
  if (!ctx->comm) RET(unsharded(ctx));
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  RET(set_device(ctx));
  return op_apply_err(ctx, m, v, out, S(stream));
}

int pslr_apply_correction(pslr_ctx* ctx, const double* y, double* out, void* stream) {
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  if (ctx->r == 0) {
    if (out != y) CK(cudaMemcpyAsync(out, y, ctx->q * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return PSLR_OK;
  }
  CKL(launch_vt_dot(ctx, y, st));     // u = G V^T y
  CKL(launch_vu_add(ctx, y, out, st));  // out = y + V u
  return PSLR_OK;
}

int pslr_apply(pslr_ctx* ctx, int64_t m, const double* b, double* z, void* stream) {
  pslr::NvtxRange nvtx_("pslr_apply");
  if (!ctx->comm) RET(unsharded(ctx));  // with a communicator: the sharded apply (comm.cu)
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  RET(set_device(ctx));
  return op_apply(ctx, m, b, z, S(stream));
}

// ---------------------------------------------------------------- sharded apply
int pslr_apply_first(pslr_ctx* ctx, const double* b, double* y0, double* s, void* stream) {
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  if (ctx->q == 0) return PSLR_OK;
  if (ctx->p > 0) CKL(launch_permute_f(ctx, b, st));  // kept for pslr_apply_last
  StepArgs a;
  a.b1 = BT_F;
  a.f = b;
  a.fL = ctx->fL;
  a.xb = ctx->xb;
  a.i1 = IT_G;
  a.g = b + ctx->p;
  a.i2 = IT_FX;
  a.i2_sub = 1;
  a.yout = y0;
  a.tag = LK_FIRST;
  RET(run_step(ctx, a, st));
  if (ctx->r > 0) CKL(launch_vt_local(ctx, y0, s, st));
  return PSLR_OK;
}

int pslr_apply_mid(pslr_ctx* ctx, const double* y0, const double* s, double* c, void* stream) {
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  if (ctx->q == 0) return PSLR_OK;
  const double* y1 = y0;
  if (ctx->r > 0) {
    CKL(launch_gs(ctx, s, st));
    CKL(launch_vu_add(ctx, y0, ctx->y1, st));
    y1 = ctx->y1;
  }
  StepArgs a;
  a.i1 = IT_G;
  a.g = y1;
  a.do_c0 = 1;
  a.yout = c;
  a.tag = LK_CORR;
  return run_step(ctx, a, st);
}

int pslr_apply_horner(pslr_ctx* ctx, const double* y, const double* c, double* out, void* stream) {
  RET(set_device(ctx));
  if (ctx->q == 0) return PSLR_OK;
  return op_es_step(ctx, y, out, 1, c, S(stream));
}

int pslr_apply_es_step(pslr_ctx* ctx, const double* v, double* out, int do_c0, void* stream) {
  RET(set_device(ctx));
  if (ctx->q == 0) return PSLR_OK;
  return op_es_step(ctx, v, out, do_c0 ? 1 : 0, nullptr, S(stream));
}

int pslr_halo_pending(pslr_ctx* ctx, void* event) {
  if (!ctx) return fail(PSLR_EINVAL, "null context");
  ctx->pending_halo = static_cast<cudaEvent_t>(event);
  return PSLR_OK;
}

int pslr_apply_last(pslr_ctx* ctx, const double* b, const double* y, double* z, void* stream) {
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  if (ctx->q > 0 && z + ctx->p != y)
    CK(cudaMemcpyAsync(z + ctx->p, y, ctx->q * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (ctx->q == 0) return op_solve_B(ctx, b, z, st);
  StepArgs a;
  a.b1 = BT_F;
  a.f = b;
  a.fL = ctx->fL;  // permuted by pslr_apply_first of the same b
  a.b2 = BT_EY;
  a.yE = y;
  a.xb = z;
  a.tag = LK_LAST;
  return run_step(ctx, a, st);
}

// ---- the split apply for two right-hand sides (op_apply2 cut where ranks exchange data):
// b, z two vector-major local n-vectors; y0, c, y, out interleaved interface vectors
// ([i][v], ghosts after the q local rows); s two r-vectors (vector-major).
static int split2_ok(pslr_ctx* ctx) {
  if (ctx->p == 0 || ctx->q == 0) return fail(PSLR_EINVAL, "two-vector split apply needs p > 0 and q > 0");
  return ensure_nv2(ctx);
}

int pslr_apply2_first(pslr_ctx* ctx, const double* b, double* y0, double* s, void* stream) {
  RET(set_device(ctx));
  RET(split2_ok(ctx));
  cudaStream_t st = S(stream);
  CKL(launch_permute2(ctx, b, st));  // fL2 kept for pslr_apply2_last
  StepArgs a;
  a.b1 = BT_F;
  a.fL = ctx->fL2;
  a.xb = ctx->xb2;
  a.i1 = IT_G;
  a.g = ctx->g2;
  a.i2 = IT_FX;
  a.i2_sub = 1;
  a.yout = y0;
  a.tag = LK_FIRST;
  RET(run_step(ctx, a, st, 2));
  if (ctx->r > 0)
    for (int v = 0; v < 2; ++v) CKL(launch_vt_local_strided(ctx, y0 + v, 2, s + v * ctx->r, st));
  return PSLR_OK;
}

int pslr_apply2_mid(pslr_ctx* ctx, const double* y0, const double* s, double* c, void* stream) {
  RET(set_device(ctx));
  RET(split2_ok(ctx));
  cudaStream_t st = S(stream);
  const double* y1 = y0;
  if (ctx->r > 0) {
    for (int v = 0; v < 2; ++v) {
      CKL(launch_gs(ctx, s + v * ctx->r, st));
      CKL(launch_vu_add_strided(ctx, y0 + v, 2, ctx->y1_2 + v, 2, st));
    }
    y1 = ctx->y1_2;
  }
  StepArgs a;
  a.i1 = IT_G;
  a.g = y1;
  a.do_c0 = 1;
  a.yout = c;
  a.tag = LK_CORR;
  return run_step(ctx, a, st, 2);
}

int pslr_apply2_horner(pslr_ctx* ctx, const double* y, const double* c, double* out, void* stream) {
  RET(set_device(ctx));
  RET(split2_ok(ctx));
  StepArgs a;
  a.b1 = BT_EY;
  a.yE = y;
  a.xb = ctx->xb2;
  a.i1 = IT_FX;
  a.i2 = IT_CGY;
  a.i2_sub = 1;
  a.yC = y;
  a.do_c0 = 1;
  a.cadd = c;
  a.yout = out;
  a.tag = LK_HORNER;
  return run_step(ctx, a, S(stream), 2);
}

int pslr_apply2_last(pslr_ctx* ctx, const double* b, const double* y, double* z, void* stream) {
  RET(set_device(ctx));
  RET(split2_ok(ctx));
  (void)b;  // its permuted copy fL2 is from pslr_apply2_first of the same b
  cudaStream_t st = S(stream);
  StepArgs a;
  a.b1 = BT_F;
  a.fL = ctx->fL2;
  a.b2 = BT_EY;
  a.yE = y;
  a.xb = ctx->xF2;
  a.tag = LK_LAST;
  RET(run_step(ctx, a, st, 2));
  CKL(launch_deinterleave2(ctx, y, z, st));
  return PSLR_OK;
}

int pslr_spmv(pslr_ctx* ctx, int which, const double* x, double* y, void* stream) {
  RET(set_device(ctx));
  const DevCsr* M = nullptr;
  switch (which) {
    case 0: M = &ctx->A; break;
    case 1: M = &ctx->K.E; break;
    case 2: M = &ctx->K.F; break;
    case 3: M = &ctx->C0; break;
    case 4: M = &ctx->K.Cg; break;
    case 5: M = &ctx->K.C; break;
    default: return fail(PSLR_EINVAL, "unknown matrix selector");
  }
  CKL(launch_spmv(*M, x, y, S(stream)));
  return PSLR_OK;
}

int pslr_apply_profiled(pslr_ctx* ctx, int64_t m, const double* b, double* z, void* stream,
                        double* launch_ms, int32_t* launch_kind, int64_t cap, int64_t* nlaunch) {
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  for (cudaEvent_t ev : ctx->prof_events) cudaEventDestroy(ev);
  ctx->prof_events.clear();
  ctx->prof_kinds.clear();
  ctx->prof_on = true;
  int rc = mark(ctx, -1, st);
  if (rc == PSLR_OK) rc = op_apply(ctx, m, b, z, st);
  ctx->prof_on = false;
  RET(rc);
  CK(cudaStreamSynchronize(st));
  const int64_t nl = (int64_t)ctx->prof_events.size() - 1;
  *nlaunch = nl;
  for (int64_t i = 0; i < nl && i < cap; ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->prof_events[i], ctx->prof_events[i + 1]));
    launch_ms[i] = ms;
    launch_kind[i] = ctx->prof_kinds[i + 1];
  }
  for (cudaEvent_t ev : ctx->prof_events) cudaEventDestroy(ev);
  ctx->prof_events.clear();
  ctx->prof_kinds.clear();
  return PSLR_OK;
}

int pslr_debug_trace(pslr_ctx* ctx, int64_t* out, int64_t cap, int64_t* count) {
  *count = 0;
  if (!ctx->K.trace) return PSLR_OK;
  RET(set_device(ctx));
  long long n = 0;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&n, ctx->K.trace, sizeof(long long), cudaMemcpyDeviceToHost));
  n = std::min<long long>(n, ctx->K.trace_cap);
  n = std::min<long long>(n, cap / 2);
  if (cap >= 2 * ctx->K.trace_cap) {  // whole buffer (events + per-CTA cycle counters)
    CK(cudaMemcpy(out, ctx->K.trace + 2, 2 * ctx->K.trace_cap * sizeof(long long),
                  cudaMemcpyDeviceToHost));
    CK(cudaMemset(ctx->K.trace + 2 + 2 * ctx->K.trace_cap - 8 * 4096, 0, 8 * 4096 * sizeof(long long)));
  } else if (n > 0) {
    CK(cudaMemcpy(out, ctx->K.trace + 2, 2 * n * sizeof(long long), cudaMemcpyDeviceToHost));
  }
  CK(cudaMemset(ctx->K.trace, 0, 16));
  *count = n;
  return PSLR_OK;
}

int pslr_apply_multi(pslr_ctx* ctx, int64_t m, int64_t nv, const double* b, double* z, void* stream) {
  pslr::NvtxRange nvtx_("pslr_apply_multi");
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  if (nv < 0) return fail(PSLR_EDIM, "number of vectors must be >= 0");
  if (!ctx->comm) RET(unsharded(ctx));
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  const int64_t n = ctx->n;
  int64_t v = 0;
  if (ctx->comm) {  // sharded: pairs through one launch sequence + one set of collectives
    for (; v + 2 <= nv; v += 2) RET(op_apply2_sharded(ctx, m, b + v * n, z + v * n, st));
    for (; v < nv; ++v) RET(op_apply_sharded(ctx, m, b + v * n, z + v * n, st));
    return PSLR_OK;
  }
  if (ctx->q > 0 && ctx->p > 0)
    for (; v + 2 <= nv; v += 2) RET(op_apply2(ctx, m, b + v * n, z + v * n, st));
  for (; v < nv; ++v) RET(op_apply(ctx, m, b + v * n, z + v * n, st));
  return PSLR_OK;
}

// ---------------------------------------------------------------- clones (concurrent applies)
int pslr_ctx_clone(const pslr_ctx* src, pslr_ctx** out) {
  *out = nullptr;
  if (!src) return fail(PSLR_EINVAL, "null context");
  RET(set_device(src));
  auto* ctx = new pslr_ctx(*src);  // shares every read-only device array of src
  ctx->parent = src->parent ? src->parent : src;
  // ctx->family (copied) now counts this clone until pslr_ctx_destroy deletes it
  ctx->allocations.clear();
  ctx->prof_events.clear();
  ctx->prof_kinds.clear();
  ctx->prof_on = false;
  ctx->device_bytes = 0;
  ctx->K.trace = nullptr;
  ctx->K.trace_cap = 0;
  ctx->kv = ctx->kz = ctx->h_dev = nullptr;
  ctx->kv_len = ctx->kz_len = ctx->h_len = 0;
  ctx->gr = ctx->gw = ctx->gt = nullptr;
  ctx->g_len = ctx->gw_len = ctx->gt_len = 0;
  ctx->red = nullptr;  // reduction partials are per context (Krylov / dnorm on a clone)
  ctx->red_len = 0;
  ctx->comm = nullptr;  // a clone has no communicator of its own
  ctx->comm_stream = nullptr;
  ctx->ev_y = ctx->ev_halo = nullptr;
  ctx->pending_halo = nullptr;
  ctx->world = 1;
  ctx->rank = 0;
  ctx->halo_idx = nullptr;
  ctx->halo_buf = nullptr;
  ctx->halo_nsend = 0;
  ctx->sh_a = ctx->sh_b = ctx->sh_c = ctx->sh_s = ctx->sh_x = nullptr;
  ctx->sh_a_len = ctx->sh_b_len = ctx->sh_c_len = ctx->sh_s_len = ctx->sh_x_len = 0;
  ctx->sh2_y0 = ctx->sh2_a = ctx->sh2_b = ctx->sh2_c = ctx->halo_buf2 = nullptr;
  ctx->sh2_y0_len = ctx->sh2_a_len = ctx->sh2_b_len = ctx->sh2_c_len = ctx->halo_buf2_len = 0;
  ctx->halo_send_cnt.assign(ctx->halo_send_cnt.size(), 0);
  ctx->halo_recv_cnt.assign(ctx->halo_recv_cnt.size(), 0);
  ctx->hpin = nullptr;  // host staging and events are per context
  ctx->hpin_len = 0;
  ctx->kev[0] = ctx->kev[1] = nullptr;
  ctx->nv2_ready = false;  // its own two-vector scratch, on first use
  auto bail = [&](int rc) {
    pslr_ctx_destroy(ctx);
    return rc;
  };
  const int64_t n = ctx->n, p = ctx->p, q = ctx->q;
  int rc;
  // private scratch: every array a launch writes
  if ((rc = alloc_scratch(ctx, &ctx->K.rhsB, p + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.rhsE, p + 2))) return bail(rc);  // zeroed
  if ((rc = alloc_scratch(ctx, &ctx->K.zB, p + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.cgy, q + 1))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.rhsC, q + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->K.zC, q + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->xb, p))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->fL, p + 2))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->y0, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->y1, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->y2, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->c, q))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->kw, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->kt, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->kr, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->io_b, n))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->io_z, n))) return bail(rc);
  {
    void* d = nullptr;
    if (cudaMalloc(&d, 64) != cudaSuccess) return bail(fail(PSLR_ECUDA, "cudaMalloc counter"));
    cudaMemset(d, 0, 64);
    ctx->allocations.push_back(d);
    ctx->counter = static_cast<unsigned int*>(d);
  }
  if (ctx->r > 0) {  // V and G are shared; the reduction scratch is private
    ctx->partials = ctx->u = nullptr;
    if ((rc = alloc_scratch(ctx, &ctx->partials, ctx->s * ctx->r))) return bail(rc);
    if ((rc = alloc_scratch(ctx, &ctx->u, 2 * ctx->r))) return bail(rc);
    if ((rc = ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)vt_grid(ctx->q, ctx->sm_count) * ctx->r + 8)))
      return bail(rc);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(PSLR_ECUDA, "clone failed"));
  *out = ctx;
  return PSLR_OK;
}

int pslr_apply_host_async(pslr_ctx* ctx, int64_t m, const double* b_host, double* z_host, void* stream) {
  pslr::NvtxRange nvtx_("pslr_apply_host_async");
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  RET(unsharded(ctx));
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  CK(cudaMemcpyAsync(ctx->io_b, b_host, ctx->n * sizeof(double), cudaMemcpyHostToDevice, st));
  RET(op_apply(ctx, m, ctx->io_b, ctx->io_z, st));
  CK(cudaMemcpyAsync(z_host, ctx->io_z, ctx->n * sizeof(double), cudaMemcpyDeviceToHost, st));
  return PSLR_OK;
}

int pslr_apply_multi_host_async(pslr_ctx* ctx, int64_t m, int64_t nv, const double* b_host,
                                double* z_host, void* stream) {
  pslr::NvtxRange nvtx_("pslr_apply_multi_host_async");
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  if (nv < 0) return fail(PSLR_EDIM, "number of vectors must be >= 0");
  RET(unsharded(ctx));
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  const int64_t n = ctx->n;
  int64_t v = 0;
  if (ctx->q > 0 && ctx->p > 0 && nv >= 2) {
    RET(ensure_nv2(ctx));
    for (; v + 2 <= nv; v += 2) {
      CK(cudaMemcpyAsync(ctx->io_b2, b_host + v * n, 2 * n * sizeof(double), cudaMemcpyHostToDevice, st));
      RET(op_apply2(ctx, m, ctx->io_b2, ctx->io_z2, st));
      CK(cudaMemcpyAsync(z_host + v * n, ctx->io_z2, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
  }
  for (; v < nv; ++v) {
    CK(cudaMemcpyAsync(ctx->io_b, b_host + v * n, n * sizeof(double), cudaMemcpyHostToDevice, st));
    RET(op_apply(ctx, m, ctx->io_b, ctx->io_z, st));
    CK(cudaMemcpyAsync(z_host + v * n, ctx->io_z, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  return PSLR_OK;
}

int pslr_apply_host(pslr_ctx* ctx, int64_t m, const double* b_host, double* z_host, void* stream) {
  pslr::NvtxRange nvtx_("pslr_apply_host");
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  CK(cudaMemcpyAsync(ctx->io_b, b_host, ctx->n * sizeof(double), cudaMemcpyHostToDevice, st));
  RET(op_apply(ctx, m, ctx->io_b, ctx->io_z, st));
  CK(cudaMemcpyAsync(z_host, ctx->io_z, ctx->n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PSLR_OK;
}

}  // extern "C"
