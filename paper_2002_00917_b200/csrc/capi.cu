// capi.cu — the C-ABI of libpslr.so: device context (upload + level-schedule
// packing), the hot-path operators of Alg. 3.2, device Arnoldi and GMRES/FGMRES.
// Every entry point cites the reference function it replaces (see include/pslr.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "pslr_internal.h"

namespace pslr {

static thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// launchers (kernels.cu)
int launch_step(const pslr_ctx* ctx, const StepArgs& a, cudaStream_t st);
int launch_correction_core(const pslr_ctx* ctx, cudaStream_t st);
int launch_spmv(const DevCsr& M, const double* x, double* y, cudaStream_t st);
int launch_multidot(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* y, int64_t n,
                    double* out, cudaStream_t st);
int launch_gemv_sub(const double* X, int64_t ld, int k, const double* h, double* w, int64_t n,
                    cudaStream_t st);
int launch_gemv(const double* X, int64_t ld, int k, const double* h, double* y, int64_t n,
                cudaStream_t st);
int launch_sub(const double* a, const double* b, double* y, int64_t n, cudaStream_t st);
int launch_add_inplace(double* y, const double* a, int64_t n, cudaStream_t st);
int launch_div_scalar(const double* x, const double* s, double* y, int64_t n, cudaStream_t st);
int launch_transpose_basis(const double* X, int64_t q, int r, double* Y, cudaStream_t st);
int dot_grid(int64_t n, int sm_count);

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return ::pslr::fail(PSLR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)
#define CKL(expr)                                                                      \
  do {                                                                                 \
    int _e = (expr);                                                                   \
    if (_e != 0)                                                                       \
      return ::pslr::fail(PSLR_ECUDA, std::string(#expr) + ": " +                      \
                                          cudaGetErrorString((cudaError_t)_e));        \
  } while (0)
#define RET(expr)              \
  do {                         \
    int _r = (expr);           \
    if (_r != PSLR_OK) return _r; \
  } while (0)

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

static int alloc_scratch(pslr_ctx* ctx, double** p, int64_t count) {
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

static void free_ptr(pslr_ctx* ctx, void* p) {
  if (!p) return;
  auto it = std::find(ctx->allocations.begin(), ctx->allocations.end(), p);
  if (it != ctx->allocations.end()) ctx->allocations.erase(it);
  cudaFree(p);
}

// grow-on-demand scratch
static int ensure(pslr_ctx* ctx, double** p, int64_t* len, int64_t need) {
  if (*len >= need) return PSLR_OK;
  free_ptr(ctx, *p);
  RET(alloc_scratch(ctx, p, need));
  *len = need;
  return PSLR_OK;
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

// Level-schedule and pack one block-diagonal triangular factor.
static int pack_tri(pslr_ctx* ctx, const pslr_csr& M, const std::vector<int64_t>& off, bool upper,
                    DevTri* out, int64_t* levels_total, int64_t* maxdepth, const char* name) {
  const int64_t nb = (int64_t)off.size() - 1;
  std::vector<int32_t> blk_lvl(nb + 1, 0), lvl_pos{0}, pos_row, pos_ent{0}, col;
  std::vector<double> val, sd, invd;
  std::vector<int32_t> lev;
  std::vector<double> dinv;  // per row (block-local) 1/diag for the U pre-scaling
  int64_t depth_max = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = off[b], hi = off[b + 1], nr = hi - lo;
    lev.assign(nr, 0);
    if (upper) {
      dinv.assign(nr, 0.0);
      std::vector<double> dg(nr, 0.0);
      for (int64_t i = 0; i < nr; ++i) {
        bool found = false;
        for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
          const int64_t j = M.indices[e];
          if (j < lo || j >= hi) return fail(PSLR_EINVAL, std::string(name) + " is not block diagonal");
          if (j < lo + i) return fail(PSLR_EINVAL, std::string(name) + " is not upper triangular");
          if (j == lo + i) {
            dg[i] = M.data[e];
            found = true;
          }
        }
        if (!found || dg[i] == 0.0)
          return fail(PSLR_ESINGULAR, std::string(name) + ": A is singular: zero entry on diagonal.");
        dinv[i] = 1.0 / dg[i];
      }
      for (int64_t i = nr - 1; i >= 0; --i) {
        int32_t lv = 0;
        for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
          const int64_t j = M.indices[e] - lo;
          if (j > i) lv = std::max(lv, lev[j] + 1);
        }
        lev[i] = lv;
      }
      // stash the diagonal for sd/invd
      for (int64_t i = 0; i < nr; ++i) (void)dg[i];
      // pack below, recomputing sd from dg
      int32_t depth = 0;
      for (int64_t i = 0; i < nr; ++i) depth = std::max(depth, lev[i] + 1);
      if (nr == 0) depth = 0;
      depth_max = std::max<int64_t>(depth_max, depth);
      std::vector<int32_t> cnt(depth + 1, 0);
      for (int64_t i = 0; i < nr; ++i) cnt[lev[i] + 1]++;
      for (int32_t l = 0; l < depth; ++l) cnt[l + 1] += cnt[l];
      std::vector<int32_t> order(nr);
      {
        std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
        for (int64_t i = 0; i < nr; ++i) order[fill[lev[i]]++] = (int32_t)i;
      }
      for (int32_t l = 0; l < depth; ++l) {
        for (int32_t k = cnt[l]; k < cnt[l + 1]; ++k) {
          const int64_t i = order[k];
          pos_row.push_back((int32_t)(lo + i));
          for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
            const int64_t j = M.indices[e] - lo;
            if (j > i) {
              col.push_back((int32_t)(lo + j));
              val.push_back(M.data[e] * dinv[j]);  // scipy: U @ diags(1/diag)
            }
          }
          pos_ent.push_back((int32_t)col.size());
          sd.push_back(dg[i] * dinv[i]);
          invd.push_back(dinv[i]);
        }
        lvl_pos.push_back((int32_t)pos_row.size());
      }
      blk_lvl[b + 1] = blk_lvl[b] + depth;
    } else {
      for (int64_t i = 0; i < nr; ++i) {
        int32_t lv = 0;
        for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
          const int64_t jg = M.indices[e];
          if (jg < lo || jg >= hi) return fail(PSLR_EINVAL, std::string(name) + " is not block diagonal");
          const int64_t j = jg - lo;
          if (j > i) return fail(PSLR_EINVAL, std::string(name) + " is not lower triangular");
          if (j < i) lv = std::max(lv, lev[j] + 1);
        }
        lev[i] = lv;
      }
      int32_t depth = 0;
      for (int64_t i = 0; i < nr; ++i) depth = std::max(depth, lev[i] + 1);
      depth_max = std::max<int64_t>(depth_max, depth);
      std::vector<int32_t> cnt(depth + 1, 0);
      for (int64_t i = 0; i < nr; ++i) cnt[lev[i] + 1]++;
      for (int32_t l = 0; l < depth; ++l) cnt[l + 1] += cnt[l];
      std::vector<int32_t> order(nr);
      {
        std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
        for (int64_t i = 0; i < nr; ++i) order[fill[lev[i]]++] = (int32_t)i;
      }
      for (int32_t l = 0; l < depth; ++l) {
        for (int32_t k = cnt[l]; k < cnt[l + 1]; ++k) {
          const int64_t i = order[k];
          pos_row.push_back((int32_t)(lo + i));
          for (int64_t e = M.indptr[lo + i]; e < M.indptr[lo + i + 1]; ++e) {
            const int64_t j = M.indices[e] - lo;
            if (j < i) {  // unit diagonal: the stored diagonal is ignored (setdiag(1))
              col.push_back((int32_t)(lo + j));
              val.push_back(M.data[e]);
            }
          }
          pos_ent.push_back((int32_t)col.size());
        }
        lvl_pos.push_back((int32_t)pos_row.size());
      }
      blk_lvl[b + 1] = blk_lvl[b] + depth;
    }
  }
  out->nblocks = (int32_t)nb;
  out->nlevels = blk_lvl[nb];
  out->npos = (int32_t)pos_row.size();
  out->nnz = (int32_t)col.size();
  RET(upload(ctx, blk_lvl, &out->blk_lvl));
  RET(upload(ctx, lvl_pos, &out->lvl_pos));
  RET(upload(ctx, pos_row, &out->pos_row));
  RET(upload(ctx, pos_ent, &out->pos_ent));
  RET(upload(ctx, col, &out->col));
  RET(upload(ctx, val, &out->val));
  if (upper) {
    RET(upload(ctx, sd, &out->sd));
    RET(upload(ctx, invd, &out->invd));
  }
  *levels_total = blk_lvl[nb];
  *maxdepth = depth_max;
  return PSLR_OK;
}

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Launch-level profiling (pslr_apply_profiled): an event after every launch.
// kinds: 0 generic step, 1 correction core, 2 apply-first (B solve + F), 3 correction + C0,
// 4 Horner step (E, B solve, F, Cg, C0 solve), 5 apply-last (E, B solve)
enum LaunchKind : int32_t { LK_STEP = 0, LK_CORE = 1, LK_FIRST = 2, LK_CORR = 3, LK_HORNER = 4, LK_LAST = 5 };

static int mark(pslr_ctx* ctx, int32_t kind, cudaStream_t st) {
  if (!ctx->prof_on) return PSLR_OK;
  cudaEvent_t ev;
  CK(cudaEventCreate(&ev));
  CK(cudaEventRecord(ev, st));
  ctx->prof_events.push_back(ev);
  ctx->prof_kinds.push_back(kind);
  return PSLR_OK;
}

static int run_step(pslr_ctx* ctx, const StepArgs& a, cudaStream_t st) {
  CKL(launch_step(ctx, a, st));
  return mark(ctx, a.tag, st);
}

static int run_core(pslr_ctx* ctx, cudaStream_t st) {
  CKL(launch_correction_core(ctx, st));
  return mark(ctx, LK_CORE, st);
}

static int set_device(const pslr_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  return PSLR_OK;
}

// ---------------------------------------------------------------- composite operators
static int op_solve_B(pslr_ctx* ctx, const double* f, double* x, cudaStream_t st) {
  StepArgs a;
  a.b1 = BT_F;
  a.f = f;
  a.tb = ctx->tb;
  a.xb = x;
  RET(run_step(ctx, a, st));
  return PSLR_OK;
}

static int op_solve_C0(pslr_ctx* ctx, const double* g, double* y, cudaStream_t st) {
  StepArgs a;
  a.i1 = IT_G;
  a.g = g;
  a.do_c0 = 1;
  a.tw = ctx->tw;
  a.yout = y;
  RET(run_step(ctx, a, st));
  return PSLR_OK;
}

// out = [C0^{-1}] (F B^{-1} E v - Cg v) [+ cadd]
static int op_es_step(pslr_ctx* ctx, const double* v, double* out, int do_c0, const double* cadd,
                      cudaStream_t st) {
  StepArgs a;
  a.b1 = BT_EY;
  a.yE = v;
  a.tb = ctx->tb;
  a.xb = ctx->xb;
  a.i1 = IT_FX;
  a.i2 = IT_CGY;
  a.i2_sub = 1;
  a.yC = v;
  a.do_c0 = do_c0;
  a.tw = ctx->tw;
  a.cadd = cadd;
  a.yout = out;
  a.tag = (do_c0 && cadd) ? LK_HORNER : LK_STEP;
  RET(run_step(ctx, a, st));
  return PSLR_OK;
}

// Horner recurrence of schur.py:89-101 starting from c = C0^{-1} v already in `c`.
static int op_horner(pslr_ctx* ctx, int64_t m, const double* c, double* out, cudaStream_t st) {
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

// u = G V^T y (partials + core), y given on the device
static int op_correction_core_from(pslr_ctx* ctx, const double* y, cudaStream_t st) {
  StepArgs a;
  a.i1 = IT_G;
  a.g = y;
  a.yout = ctx->y0 == y ? ctx->y2 : ctx->y0;  // harmless copy target
  a.partials = ctx->partials;
  RET(run_step(ctx, a, st));
  RET(run_core(ctx, st));
  return PSLR_OK;
}

static int op_apply(pslr_ctx* ctx, int64_t m, const double* b, double* z, cudaStream_t st) {
  const int64_t p = ctx->p, q = ctx->q;
  if (q == 0) return op_solve_B(ctx, b, z, st);
  // (1) y0 = g - F B^{-1} f                                   preconditioner.py:89
  {
    StepArgs a;
    a.b1 = BT_F;
    a.f = b;
    a.tb = ctx->tb;
    a.xb = ctx->xb;
    a.i1 = IT_G;
    a.g = b + p;
    a.i2 = IT_FX;
    a.i2_sub = 1;
    a.yout = ctx->y0;
    a.partials = ctx->r > 0 ? ctx->partials : nullptr;
    a.tag = LK_FIRST;
    RET(run_step(ctx, a, st));
  }
  // (2) y1 = y0 + V G V^T y0 ; c = C0^{-1} y1                 preconditioner.py:90, schur.py:97
  double* c = (m == 0) ? z + p : ctx->c;
  {
    StepArgs a;
    a.i1 = IT_G;
    a.g = ctx->y0;
    if (ctx->r > 0) {
      RET(run_core(ctx, st));
      a.i2 = IT_VU;
      a.i2_sub = 0;
      a.u = ctx->u;
    }
    a.do_c0 = 1;
    a.tw = ctx->tw;
    a.yout = c;
    a.tag = LK_CORR;
    RET(run_step(ctx, a, st));
  }
  // (3) m Horner steps y = C0^{-1}(Es y) + c                  schur.py:99-100
  if (m > 0) RET(op_horner(ctx, m, c, z + p, st));
  // (4) x = B^{-1}(f - E y)                                   preconditioner.py:92
  {
    StepArgs a;
    a.b1 = BT_F;
    a.f = b;
    a.b2 = BT_EY;
    a.yE = z + p;
    a.tb = ctx->tb;
    a.xb = z;
    a.tag = LK_LAST;
    RET(run_step(ctx, a, st));
  }
  return PSLR_OK;
}

static int op_apply_err(pslr_ctx* ctx, int64_t m, const double* v, double* out, cudaStream_t st) {
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

static int dnorm(pslr_ctx* ctx, const double* x, int64_t n, double* out_host, cudaStream_t st) {
  RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)dot_grid(n, ctx->sm_count) * 1 + 8));
  RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 8));
  CKL(launch_multidot(ctx, x, n, 1, x, n, ctx->h_dev, st));
  double d = 0.0;
  CK(cudaMemcpyAsync(&d, ctx->h_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *out_host = std::sqrt(d);
  return PSLR_OK;
}

// Classical Gram-Schmidt with one reorthogonalisation on the first k columns of
// X (column-major, ld = n): krylov.py:75-80 / lowrank.py:62-67.  Returns h (host,
// h1 + h2) and the norm of the orthogonalised w.
static int cgs2(pslr_ctx* ctx, const double* X, int64_t n, int k, double* w, double* h_host,
                double* hnorm, cudaStream_t st) {
  RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)dot_grid(n, ctx->sm_count) * (k + 1) + 8));
  RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 2 * (int64_t)k + 8));
  double* h1 = ctx->h_dev;
  double* h2 = ctx->h_dev + k;
  double* nn = ctx->h_dev + 2 * k;
  CKL(launch_multidot(ctx, X, n, k, w, n, h1, st));
  CKL(launch_gemv_sub(X, n, k, h1, w, n, st));
  CKL(launch_multidot(ctx, X, n, k, w, n, h2, st));
  CKL(launch_gemv_sub(X, n, k, h2, w, n, st));
  CKL(launch_multidot(ctx, w, n, 1, w, n, nn, st));
  std::vector<double> tmp(2 * k + 1);
  CK(cudaMemcpyAsync(tmp.data(), ctx->h_dev, (2 * k + 1) * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int c = 0; c < k; ++c) h_host[c] = tmp[c] + tmp[k + c];
  *hnorm = std::sqrt(tmp[2 * k]);
  // keep the unsummed h1 for callers that need it (arnoldi stores h+h2 = same)
  return PSLR_OK;
}

}  // namespace pslr

using namespace pslr;

extern "C" {

const char* pslr_last_error(void) { return g_last_error.c_str(); }
int pslr_abi_version(void) { return 1; }

int pslr_ctx_create(pslr_ctx** out, int device, const pslr_system* sys) {
  *out = nullptr;
  if (!sys) return fail(PSLR_EINVAL, "null system");
  const int64_t n = sys->n, p = sys->p, q = sys->q, s = sys->s;
  if (p + q != n || s < 1) return fail(PSLR_EDIM, "inconsistent system dimensions");
  RET(check_csr(sys->LB, p, p, "L_B"));
  RET(check_csr(sys->UB, p, p, "U_B"));
  RET(check_csr(sys->LC, q, q, "L_C0"));
  RET(check_csr(sys->UC, q, q, "U_C0"));
  RET(check_csr(sys->E, p, q, "E"));
  RET(check_csr(sys->F, q, p, "F"));
  RET(check_csr(sys->C, q, q, "C"));
  RET(check_csr(sys->C0, q, q, "C0"));
  RET(check_csr(sys->Cg, q, q, "Cg"));
  RET(check_csr(sys->A, n, n, "A"));
  if (sys->interior_offsets[0] != 0 || sys->interior_offsets[s] != p ||
      sys->interface_offsets[0] != 0 || sys->interface_offsets[s] != q)
    return fail(PSLR_EDIM, "block offsets do not tile the system");
  auto* ctx = new pslr_ctx();
  ctx->device = device;
  ctx->n = n;
  ctx->p = p;
  ctx->q = q;
  ctx->s = s;
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
  pslr_ctx_info_t& I = ctx->info;
  if ((rc = pack_tri(ctx, sys->LB, ctx->interior_off, false, &ctx->LB, &I.levels_LB, &I.maxdepth_LB, "L_B"))) return bail(rc);
  if ((rc = pack_tri(ctx, sys->UB, ctx->interior_off, true, &ctx->UB, &I.levels_UB, &I.maxdepth_UB, "U_B"))) return bail(rc);
  if ((rc = pack_tri(ctx, sys->LC, ctx->interface_off, false, &ctx->LC, &I.levels_LC, &I.maxdepth_LC, "L_C0"))) return bail(rc);
  if ((rc = pack_tri(ctx, sys->UC, ctx->interface_off, true, &ctx->UC, &I.levels_UC, &I.maxdepth_UC, "U_C0"))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->E, &ctx->E))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->F, &ctx->F))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->C, &ctx->C))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->C0, &ctx->C0))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->Cg, &ctx->Cg))) return bail(rc);
  if ((rc = upload_csr(ctx, sys->A, &ctx->A))) return bail(rc);
  {
    std::vector<int32_t> io(s + 1), fo(s + 1);
    for (int64_t b = 0; b <= s; ++b) {
      io[b] = (int32_t)ctx->interior_off[b];
      fo[b] = (int32_t)ctx->interface_off[b];
    }
    const int32_t* d = nullptr;
    if ((rc = upload(ctx, io, &d))) return bail(rc);
    ctx->d_int_off = const_cast<int32_t*>(d);
    if ((rc = upload(ctx, fo, &d))) return bail(rc);
    ctx->d_ifc_off = const_cast<int32_t*>(d);
  }
  if ((rc = alloc_scratch(ctx, &ctx->tb, p))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->xb, p))) return bail(rc);
  if ((rc = alloc_scratch(ctx, &ctx->tw, q))) return bail(rc);
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
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(PSLR_ECUDA, "upload failed"));
  *out = ctx;
  return PSLR_OK;
}

void pslr_ctx_destroy(pslr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (void* p : ctx->allocations) cudaFree(p);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
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
  RET(set_device(ctx));
  free_ptr(ctx, ctx->V);
  free_ptr(ctx, ctx->G);
  free_ptr(ctx, ctx->partials);
  free_ptr(ctx, ctx->u);
  ctx->V = ctx->G = ctx->partials = ctx->u = nullptr;
  ctx->r = 0;
  if (r == 0 || ctx->q == 0) return PSLR_OK;
  RET(alloc_scratch(ctx, &ctx->V, ctx->q * r));
  RET(alloc_scratch(ctx, &ctx->G, r * r));
  RET(alloc_scratch(ctx, &ctx->partials, ctx->s * r));
  RET(alloc_scratch(ctx, &ctx->u, 2 * r));
  CK(cudaMemcpy(ctx->V, V, ctx->q * r * sizeof(double),
                V_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->G, G, r * r * sizeof(double), cudaMemcpyHostToDevice));
  ctx->r = r;
  return PSLR_OK;
}

int pslr_ctx_set_correction(pslr_ctx* ctx, int64_t r, const double* V, const double* G) {
  return set_correction_common(ctx, r, V, false, G);
}

int pslr_ctx_set_correction_device(pslr_ctx* ctx, int64_t r, const double* V_dev, const double* G) {
  return set_correction_common(ctx, r, V_dev, true, G);
}

int pslr_solve_B(pslr_ctx* ctx, const double* f, double* x, void* stream) {
  RET(set_device(ctx));
  return op_solve_B(ctx, f, x, S(stream));
}

int pslr_solve_C0(pslr_ctx* ctx, const double* g, double* y, void* stream) {
  RET(set_device(ctx));
  return op_solve_C0(ctx, g, y, S(stream));
}

int pslr_apply_Es(pslr_ctx* ctx, const double* v, double* out, void* stream) {
  RET(set_device(ctx));
  return op_es_step(ctx, v, out, 0, nullptr, S(stream));
}

int pslr_apply_S(pslr_ctx* ctx, const double* v, double* out, void* stream) {
  RET(set_device(ctx));
  StepArgs a;
  a.b1 = BT_EY;
  a.yE = v;
  a.tb = ctx->tb;
  a.xb = ctx->xb;
  a.i1 = IT_CY;
  a.yC = v;
  a.i2 = IT_FX;
  a.i2_sub = 1;
  a.yout = out;
  RET(run_step(ctx, a, S(stream)));
  return PSLR_OK;
}

int pslr_apply_neumann(pslr_ctx* ctx, int64_t m, const double* v, double* out, void* stream) {
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  RET(set_device(ctx));
  RET(op_solve_C0(ctx, v, ctx->c, S(stream)));
  return op_horner(ctx, m, ctx->c, out, S(stream));
}

int pslr_apply_Err(pslr_ctx* ctx, int64_t m, const double* v, double* out, void* stream) {
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
  RET(op_correction_core_from(ctx, y, st));
  StepArgs a;
  a.i1 = IT_G;
  a.g = y;
  a.i2 = IT_VU;
  a.i2_sub = 0;
  a.u = ctx->u;
  a.yout = out;
  RET(run_step(ctx, a, st));
  return PSLR_OK;
}

int pslr_apply(pslr_ctx* ctx, int64_t m, const double* b, double* z, void* stream) {
  if (m < 0) return fail(PSLR_EDIM, "series degree m must be >= 0");
  RET(set_device(ctx));
  return op_apply(ctx, m, b, z, S(stream));
}

int pslr_spmv(pslr_ctx* ctx, int which, const double* x, double* y, void* stream) {
  RET(set_device(ctx));
  const DevCsr* M = nullptr;
  switch (which) {
    case 0: M = &ctx->A; break;
    case 1: M = &ctx->E; break;
    case 2: M = &ctx->F; break;
    case 3: M = &ctx->C0; break;
    case 4: M = &ctx->Cg; break;
    case 5: M = &ctx->C; break;
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

int pslr_apply_host(pslr_ctx* ctx, int64_t m, const double* b_host, double* z_host, void* stream) {
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  CK(cudaMemcpyAsync(ctx->io_b, b_host, ctx->n * sizeof(double), cudaMemcpyHostToDevice, st));
  RET(op_apply(ctx, m, ctx->io_b, ctx->io_z, st));
  CK(cudaMemcpyAsync(z_host, ctx->io_z, ctx->n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return PSLR_OK;
}

int pslr_arnoldi(pslr_ctx* ctx, int64_t m, int64_t rank, const double* v0, double* V_dev, double* H,
                 int64_t* r_out, void* stream) {
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  const int64_t q = ctx->q;
  if (rank < 0) return fail(PSLR_EDIM, "rank must be >= 0");
  rank = std::min(rank, q);
  *r_out = 0;
  if (q == 0 || rank == 0) return PSLR_OK;
  RET(ensure(ctx, &ctx->kv, &ctx->kv_len, q * (rank + 1)));
  double* Vc = ctx->kv;  // column-major q x (rank+1)
  CK(cudaMemsetAsync(Vc, 0, q * (rank + 1) * sizeof(double), st));
  CK(cudaMemcpyAsync(Vc, v0, q * sizeof(double), cudaMemcpyHostToDevice, st));
  std::vector<double> Hb((rank + 1) * rank, 0.0);  // row-major (rank+1) x rank
  std::vector<double> h(rank + 1);
  int64_t r = rank;
  double* w = ctx->kw;
  for (int64_t j = 0; j < rank; ++j) {
    RET(op_apply_err(ctx, m, Vc + j * q, w, st));
    double hn = 0.0;
    RET(cgs2(ctx, Vc, q, (int)(j + 1), w, h.data(), &hn, st));
    for (int64_t i = 0; i <= j; ++i) Hb[i * rank + j] = h[i];
    Hb[(j + 1) * rank + j] = hn;
    if (hn <= 1e-14) {  // lowrank.py:69-71 (BREAKDOWN_RTOL, start vector has norm 1)
      r = j + 1;
      break;
    }
    CK(cudaMemcpyAsync(ctx->h_dev, &hn, sizeof(double), cudaMemcpyHostToDevice, st));
    CKL(launch_div_scalar(w, ctx->h_dev, Vc + (j + 1) * q, q, st));
  }
  CKL(launch_transpose_basis(Vc, q, (int)r, V_dev, st));
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < r; ++j) H[i * r + j] = Hb[i * rank + j];
  CK(cudaStreamSynchronize(st));
  *r_out = r;
  return PSLR_OK;
}

int pslr_gmres(pslr_ctx* ctx, int64_t m, const double* b, double* x, double tol, int64_t maxit,
               int64_t restart, int precond, int flexible, int64_t* iterations, int* converged,
               double* final_relres, double* history, int64_t* history_len, void* stream) {
  RET(set_device(ctx));
  cudaStream_t st = S(stream);
  const int64_t n = ctx->n;
  std::vector<double> hist;
  auto finish = [&](bool conv, int64_t its, double rel) {
    *iterations = its;
    *converged = conv ? 1 : 0;
    *final_relres = rel;
    for (size_t i = 0; i < hist.size() && (int64_t)i <= maxit; ++i) history[i] = hist[i];
    *history_len = (int64_t)std::min<size_t>(hist.size(), (size_t)maxit + 1);
  };
  double bnorm = 0.0;
  RET(dnorm(ctx, b, n, &bnorm, st));
  CK(cudaMemsetAsync(x, 0, n * sizeof(double), st));
  if (bnorm == 0.0) {
    hist.push_back(1.0);
    finish(true, 0, 0.0);
    CK(cudaStreamSynchronize(st));
    return PSLR_OK;
  }
  hist.push_back(1.0);
  int64_t total = 0;
  bool conv = false;
  double relres = 1.0;
  double* r = ctx->kr;
  double* w = ctx->kw;
  double* t = ctx->kt;
  auto apply_M = [&](const double* in, double* out) -> int {
    if (precond) return op_apply(ctx, m, in, out, st);
    if (out != in) CK(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return PSLR_OK;
  };
  while (total < maxit && !conv) {
    // r = b - A x                                            krylov.py:56
    CKL(launch_spmv(ctx->A, x, t, st));
    CKL(launch_sub(b, t, r, n, st));
    double beta = 0.0;
    RET(dnorm(ctx, r, n, &beta, st));
    relres = beta / bnorm;
    if (relres <= tol) {
      conv = true;
      break;
    }
    const int64_t cycle = restart <= 0 ? maxit - total : std::min(restart, maxit - total);
    RET(ensure(ctx, &ctx->kv, &ctx->kv_len, n * (cycle + 1)));
    if (flexible) RET(ensure(ctx, &ctx->kz, &ctx->kz_len, n * cycle));
    double* Vb = ctx->kv;
    std::vector<double> Hc((cycle + 1) * cycle, 0.0);  // row-major (cycle+1) x cycle
    auto Hat = [&](int64_t i, int64_t j) -> double& { return Hc[i * cycle + j]; };
    std::vector<double> cs(cycle, 0.0), sn(cycle, 0.0), g(cycle + 1, 0.0), h(cycle + 1);
    g[0] = beta;
    RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 2 * (cycle + 1) + 8));
    CK(cudaMemcpyAsync(ctx->h_dev, &beta, sizeof(double), cudaMemcpyHostToDevice, st));
    CKL(launch_div_scalar(r, ctx->h_dev, Vb, n, st));
    int64_t j = 0;
    bool breakdown = false;
    while (j < cycle) {
      // w = A M v_j                                          krylov.py:74
      double* mv = flexible ? ctx->kz + j * n : t;
      RET(apply_M(Vb + j * n, mv));
      CKL(launch_spmv(ctx->A, mv, w, st));
      double hnext = 0.0;
      RET(cgs2(ctx, Vb, n, (int)(j + 1), w, h.data(), &hnext, st));
      bool finite = std::isfinite(hnext);
      for (int64_t i = 0; i <= j; ++i) finite = finite && std::isfinite(h[i]);
      if (!finite) return fail(PSLR_ENONFINITE, "GMRES diverged: non-finite values in the recurrence");
      for (int64_t i = 0; i <= j; ++i) Hat(i, j) = h[i];
      Hat(j + 1, j) = hnext;
      for (int64_t i = 0; i < j; ++i) {  // krylov.py:86-97
        const double tmp = cs[i] * Hat(i, j) + sn[i] * Hat(i + 1, j);
        Hat(i + 1, j) = -sn[i] * Hat(i, j) + cs[i] * Hat(i + 1, j);
        Hat(i, j) = tmp;
      }
      const double denom = std::hypot(Hat(j, j), hnext);
      if (denom == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = Hat(j, j) / denom;
        sn[j] = hnext / denom;
      }
      Hat(j, j) = denom;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      ++j;
      const double est = std::fabs(g[j]) / bnorm;
      hist.push_back(est);
      if (hnext <= 1e-14 * beta) {
        breakdown = true;
        break;
      }
      if (est <= tol) break;
      if (j < cycle) {
        CK(cudaMemcpyAsync(ctx->h_dev, &hnext, sizeof(double), cudaMemcpyHostToDevice, st));
        CKL(launch_div_scalar(w, ctx->h_dev, Vb + j * n, n, st));
      }
    }
    if (j > 0) {  // krylov.py:110-114
      std::vector<double> y(j, 0.0);
      for (int64_t i = j - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int64_t k = i + 1; k < j; ++k) acc += Hat(i, k) * y[k];
        y[i] = (g[i] - acc) / Hat(i, i);
      }
      CK(cudaMemcpyAsync(ctx->h_dev, y.data(), j * sizeof(double), cudaMemcpyHostToDevice, st));
      if (flexible) {
        CKL(launch_gemv(ctx->kz, n, (int)j, ctx->h_dev, t, n, st));
        CKL(launch_add_inplace(x, t, n, st));
      } else {
        CKL(launch_gemv(Vb, n, (int)j, ctx->h_dev, r, n, st));
        RET(apply_M(r, t));
        CKL(launch_add_inplace(x, t, n, st));
      }
    }
    CKL(launch_spmv(ctx->A, x, t, st));
    CKL(launch_sub(b, t, r, n, st));
    double rn = 0.0;
    RET(dnorm(ctx, r, n, &rn, st));
    relres = rn / bnorm;
    hist.back() = relres;
    if (relres <= tol)
      conv = true;
    else if (breakdown)
      break;
  }
  if (!conv && total < maxit && !std::isfinite(relres))
    return fail(PSLR_ENONFINITE, "GMRES diverged: non-finite residual");
  const int64_t its = conv ? total : maxit;
  if (!conv)
    while ((int64_t)hist.size() < maxit + 1) hist.push_back(relres);
  finish(conv, its, relres);
  CK(cudaStreamSynchronize(st));
  return PSLR_OK;
}

}  // extern "C"
