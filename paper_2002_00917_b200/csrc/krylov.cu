// krylov.cu — device Krylov drivers of the C-ABI: Arnoldi on E_rr(m)
// (lowrank.py:39-73) and restarted right-preconditioned GMRES / FGMRES
// (krylov.py:35-129).  Vectors, the Krylov basis and every reduction live on the
// device (libpslr kernels); the (cycle+1)-sized Hessenberg/Givens bookkeeping is
// scalar host code with the reference's exact control flow.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <vector>

#include "pslr_ops.h"

namespace pslr {

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Leading dimension of a column-major Krylov basis: n rounded up to 32 doubles and made an
// odd multiple of 256 B, so the columns of one row tile do not share L1/L2 sets (a
// power-of-two n, e.g. 128^3, would put every column of a tile in the same set).
static int64_t basis_ld(int64_t n) {
  int64_t ld = (n + 31) / 32 * 32;
  if (((ld / 32) & 1) == 0) ld += 32;
  return ld;
}

static int dnorm(pslr_ctx* ctx, const double* x, int64_t n, double* out_host, cudaStream_t st) {
  RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)dot_grid(n, ctx->sm_count) * 1 + 8));
  RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 8));
  CKL(launch_multidot(ctx, x, n, 1, x, n, ctx->h_dev, st));
  RET(comm_allreduce(ctx, ctx->h_dev, 1, st));
  double d = 0.0;
  CK(cudaMemcpyAsync(&d, ctx->h_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *out_host = std::sqrt(d);
  return PSLR_OK;
}

// Classical Gram-Schmidt with one reorthogonalisation against the first k columns
// of X (column-major, ld = n): krylov.py:75-80 / lowrank.py:62-67.  h_host = h1 + h2,
// hnorm = ||w|| after both passes.  Three passes over X (each projection fused with the
// following dot / norm) and one host synchronisation.
static int cgs2(pslr_ctx* ctx, const double* X, int64_t ld, int64_t n, int k, double* w, double* h_host,
                double* hnorm, cudaStream_t st) {
  RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)dot_grid(n, ctx->sm_count) * (k + 1) + 8));
  RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 2 * (int64_t)k + 8));
  double* h1 = ctx->h_dev;
  double* h2 = ctx->h_dev + k;
  double* nn = ctx->h_dev + 2 * k;
  CKL(launch_multidot(ctx, X, ld, k, w, n, h1, st));      // h1 = X^T w
  RET(comm_allreduce(ctx, h1, k, st));                    // (sharded: over the ranks' rows)
  CKL(launch_sub_dot(ctx, X, ld, k, h1, w, n, h2, st));   // w -= X h1 ; h2 = X^T w
  RET(comm_allreduce(ctx, h2, k, st));
  CKL(launch_sub_norm(ctx, X, ld, k, h2, w, n, nn, st));  // w -= X h2 ; nn = w.w
  RET(comm_allreduce(ctx, nn, 1, st));
  std::vector<double> tmp(2 * k + 1);
  CK(cudaMemcpyAsync(tmp.data(), ctx->h_dev, (2 * k + 1) * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int c = 0; c < k; ++c) h_host[c] = tmp[c] + tmp[k + c];
  *hnorm = std::sqrt(tmp[2 * k]);
  return PSLR_OK;
}

// y = op(x) on device n-vectors, stream-ordered; returns a PSLR status
using VecOp = std::function<int(const double*, double*)>;

// A caller-supplied operator (C-ABI callback): PSLR_ECALLBACK when it reports failure
static VecOp callback_op(pslr_vec_fn fn, void* user, cudaStream_t st) {
  return [fn, user, st](const double* x, double* y) -> int {
    if (fn(user, x, y, static_cast<void*>(st)) != 0)
      return fail(PSLR_ECALLBACK, "operator callback reported an error");
    return PSLR_OK;
  };
}

// Krylov work vectors of length n (the context's own n, or a generic operator's)
static int krylov_vectors(pslr_ctx* ctx, int64_t n, double** r, double** w, double** t) {
  if (n <= ctx->n) {
    *r = ctx->kr;
    *w = ctx->kw;
    *t = ctx->kt;
    return PSLR_OK;
  }
  RET(ensure(ctx, &ctx->gr, &ctx->g_len, n));
  RET(ensure(ctx, &ctx->gw, &ctx->gw_len, n));
  RET(ensure(ctx, &ctx->gt, &ctx->gt_len, n));
  *r = ctx->gr;
  *w = ctx->gw;
  *t = ctx->gt;
  return PSLR_OK;
}

// lowrank.py:39-73: r-step CGS2 Arnoldi on op over `dim` rows (this rank's rows when
// sharded), V0 in Vc column 0 (unit norm).  V_dev: dim x r_out packed row-major.
static int arnoldi_core(pslr_ctx* ctx, int64_t dim, int64_t rank, const VecOp& op, const double* v0,
                        double* V_dev, double* H, int64_t* r_out, cudaStream_t st) {
  const int64_t ldq = basis_ld(dim);
  RET(ensure(ctx, &ctx->kv, &ctx->kv_len, ldq * (rank + 1)));
  double *wr = nullptr, *w = nullptr, *wt = nullptr;
  RET(krylov_vectors(ctx, dim, &wr, &w, &wt));
  double* Vc = ctx->kv;  // column-major dim x (rank+1), leading dimension ldq
  CK(cudaMemsetAsync(Vc, 0, ldq * (rank + 1) * sizeof(double), st));
  if (dim) CK(cudaMemcpyAsync(Vc, v0, dim * sizeof(double), cudaMemcpyHostToDevice, st));
  // lowrank.py:52-57 normalises the seeded draw.  A start vector that already has unit
  // norm (the Python wrapper normalises it with numpy, bit for bit as the reference) is
  // used as is; anything else is divided by its (allreduced) norm here.
  double v0n = 0.0;
  RET(dnorm(ctx, Vc, dim, &v0n, st));
  if (!(v0n > 0.0) || !std::isfinite(v0n)) return fail(PSLR_EDIM, "Arnoldi start vector has no direction");
  if (std::fabs(v0n - 1.0) > 1e-14) {
    CK(cudaMemcpyAsync(ctx->h_dev, &v0n, sizeof(double), cudaMemcpyHostToDevice, st));
    CKL(launch_div_scalar(Vc, ctx->h_dev, Vc, dim, st));
  }
  std::vector<double> Hb((rank + 1) * rank, 0.0);  // row-major (rank+1) x rank
  std::vector<double> h(rank + 1);
  int64_t r = rank;
  for (int64_t j = 0; j < rank; ++j) {
    RET(op(Vc + j * ldq, w));
    double hn = 0.0;
    RET(cgs2(ctx, Vc, ldq, dim, (int)(j + 1), w, h.data(), &hn, st));
    for (int64_t i = 0; i <= j; ++i) Hb[i * rank + j] = h[i];
    Hb[(j + 1) * rank + j] = hn;
    if (hn <= 1e-14) {  // lowrank.py:69-71 (BREAKDOWN_RTOL, start vector has norm 1)
      r = j + 1;
      break;
    }
    CK(cudaMemcpyAsync(ctx->h_dev, &hn, sizeof(double), cudaMemcpyHostToDevice, st));
    CKL(launch_div_scalar(w, ctx->h_dev, Vc + (j + 1) * ldq, dim, st));
  }
  // V_dev: dim rows x r columns, row-major with leading dimension r (packed)
  CKL(launch_transpose_basis(Vc, ldq, dim, (int)r, V_dev, st));
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < r; ++j) H[i * r + j] = Hb[i * rank + j];
  CK(cudaStreamSynchronize(st));
  *r_out = r;
  return PSLR_OK;
}

}  // namespace pslr

using namespace pslr;

extern "C" {

int pslr_arnoldi(pslr_ctx* ctx, int64_t m, int64_t rank, const double* v0, double* V_dev, double* H,
                 int64_t* r_out, void* stream) {
  pslr::NvtxRange nvtx_("pslr_arnoldi");
  RET(set_device(ctx));
  if (ctx->nghost && !ctx->comm)
    return fail(PSLR_EINVAL, "sharded context: pslr_comm_init + pslr_ctx_set_halo first (or shard.py)");
  cudaStream_t st = S(stream);
  const int64_t q = ctx->q;
  if (rank < 0) return fail(PSLR_EDIM, "rank must be >= 0");
  *r_out = 0;
  // the rank is capped by the GLOBAL interface dimension (lowrank.py:49): on a sharded
  // context every rank must take the same decision and run the same collectives, even a
  // rank that owns no interface row
  int64_t qg = q;
  if (ctx->comm) {
    RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 8));
    double qd = (double)q;
    CK(cudaMemcpyAsync(ctx->h_dev, &qd, sizeof(double), cudaMemcpyHostToDevice, st));
    RET(comm_allreduce(ctx, ctx->h_dev, 1, st));
    CK(cudaMemcpyAsync(&qd, ctx->h_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    qg = (int64_t)qd;
  }
  rank = std::min(rank, qg);
  if (qg == 0 || rank == 0) return PSLR_OK;
  RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 8));
  const VecOp op = [ctx, m, st](const double* x, double* y) { return op_apply_err(ctx, m, x, y, st); };
  return arnoldi_core(ctx, q, rank, op, v0, V_dev, H, r_out, st);
}

int pslr_arnoldi_op(pslr_ctx* ctx, int64_t dim, pslr_vec_fn op_fn, void* user, int64_t rank, const double* v0,
                    double* V_dev, double* H, int64_t* r_out, void* stream) {
  pslr::NvtxRange nvtx_("pslr_arnoldi_op");
  RET(set_device(ctx));
  if (!op_fn) return fail(PSLR_EINVAL, "operator callback missing");
  if (dim < 0 || rank < 0) return fail(PSLR_EDIM, "dim and rank must be >= 0");
  cudaStream_t st = S(stream);
  *r_out = 0;
  rank = std::min(rank, dim);
  if (dim == 0 || rank == 0) return PSLR_OK;
  RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 8));
  return arnoldi_core(ctx, dim, rank, callback_op(op_fn, user, st), v0, V_dev, H, r_out, st);
}

// krylov.py:35-129 for any operator pair on device n-vectors (A, M: stream-ordered)
static int gmres_core(pslr_ctx* ctx, int64_t n, const VecOp& A, const VecOp& apply_M, const double* b, double* x,
                      double tol, int64_t maxit, int64_t restart, int flexible, int64_t* iterations, int* converged,
                      double* final_relres, double* history, int64_t* history_len, cudaStream_t st) {
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
  hist.push_back(1.0);
  if (bnorm == 0.0) {
    finish(true, 0, 0.0);
    CK(cudaStreamSynchronize(st));
    return PSLR_OK;
  }
  int64_t total = 0;
  bool conv = false;
  double relres = 1.0;
  double *r = nullptr, *w = nullptr, *t = nullptr;
  RET(krylov_vectors(ctx, n, &r, &w, &t));
  while (total < maxit && !conv) {
    // r = b - A x                                            krylov.py:56
    RET(A(x, t));
    CKL(launch_sub(b, t, r, n, st));
    double beta = 0.0;
    RET(dnorm(ctx, r, n, &beta, st));
    relres = beta / bnorm;
    if (relres <= tol) {
      conv = true;
      break;
    }
    const int64_t cycle = restart <= 0 ? maxit - total : std::min(restart, maxit - total);
    const int64_t ld = basis_ld(n);
    RET(ensure(ctx, &ctx->kv, &ctx->kv_len, ld * (cycle + 1)));
    if (flexible) RET(ensure(ctx, &ctx->kz, &ctx->kz_len, n * cycle));
    double* Vb = ctx->kv;
    std::vector<double> Hc((cycle + 1) * cycle, 0.0);  // row-major (cycle+1) x cycle
    auto Hat = [&](int64_t i, int64_t j) -> double& { return Hc[i * cycle + j]; };
    std::vector<double> cs(cycle, 0.0), sn(cycle, 0.0), g(cycle + 1, 0.0), h(cycle + 1);
    g[0] = beta;
    // Iteration j's device work (apply, A-SpMV, the three CGS2 passes, hnext = ||w||,
    // v_{j+1} = w / hnext) and the copy of its coefficients to pinned host memory are
    // enqueued one iteration AHEAD of the host's scalar recurrence: while the host waits
    // for iteration j's coefficients the device already runs iteration j+1, so the
    // host round trip leaves the critical path.  A speculative iteration past a stop is
    // discarded (it only writes scratch and basis columns the cycle end does not read).
    const int64_t SL = 2 * (cycle + 1) + 8;  // one coefficient slot: h1 | h2 | nn | hnext
    RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 2 * SL));
    // reduction partials for the widest pass of the cycle (sized once: no reallocation
    // while iterations are in flight)
    RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)dot_grid(n, ctx->sm_count) * (cycle + 2) + 8));
    if (ctx->hpin_len < 2 * SL) {
      if (ctx->hpin) cudaFreeHost(ctx->hpin);
      ctx->hpin = nullptr;
      ctx->hpin_len = 0;
      CK(cudaMallocHost(&ctx->hpin, 2 * SL * sizeof(double)));
      ctx->hpin_len = 2 * SL;
    }
    for (auto& ev : ctx->kev)
      if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaMemcpyAsync(ctx->h_dev, &beta, sizeof(double), cudaMemcpyHostToDevice, st));
    CKL(launch_div_scalar(r, ctx->h_dev, Vb, n, st));
    auto enqueue = [&](int64_t jj) -> int {
      const int k = (int)(jj + 1);
      double* mv = flexible ? ctx->kz + jj * n : t;  // w = A M v_j   krylov.py:74
      RET(apply_M(Vb + jj * ld, mv));
      RET(A(mv, w));
      double* hs = ctx->h_dev + (jj & 1) * SL;
      CKL(launch_multidot(ctx, Vb, ld, k, w, n, hs, st));           // h1 = V^T w
      RET(comm_allreduce(ctx, hs, k, st));                           // (sharded: all ranks' rows)
      CKL(launch_sub_dot(ctx, Vb, ld, k, hs, w, n, hs + k, st));      // w -= V h1 ; h2 = V^T w
      RET(comm_allreduce(ctx, hs + k, k, st));
      CKL(launch_sub_norm(ctx, Vb, ld, k, hs + k, w, n, hs + 2 * k, st));  // w -= V h2 ; ||w||^2
      RET(comm_allreduce(ctx, hs + 2 * k, 1, st));
      CKL(launch_sqrt(hs + 2 * k, hs + 2 * k + 1, st));
      CK(cudaMemcpyAsync(ctx->hpin + (jj & 1) * SL, hs, (2 * k + 2) * sizeof(double),
                         cudaMemcpyDeviceToHost, st));
      CK(cudaEventRecord(ctx->kev[jj & 1], st));
      if (jj + 1 < cycle) CKL(launch_div_scalar(w, hs + 2 * k + 1, Vb + (jj + 1) * ld, n, st));
      return PSLR_OK;
    };
    int64_t j = 0;
    bool breakdown = false;
    RET(enqueue(0));
    while (j < cycle) {
      if (j + 1 < cycle) RET(enqueue(j + 1));
      CK(cudaEventSynchronize(ctx->kev[j & 1]));
      const double* hp = ctx->hpin + (j & 1) * SL;
      const int64_t k = j + 1;
      for (int64_t i = 0; i < k; ++i) h[i] = hp[i] + hp[k + i];  // h = h1 + h2
      const double hnext = hp[2 * k + 1];
      bool finite = std::isfinite(hnext);
      for (int64_t i = 0; i <= j; ++i) finite = finite && std::isfinite(h[i]);
      if (!finite) {
        CK(cudaStreamSynchronize(st));
        return fail(PSLR_ENONFINITE, "GMRES diverged: non-finite values in the recurrence");
      }
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
        CKL(launch_gemv(Vb, ld, (int)j, ctx->h_dev, r, n, st));
        RET(apply_M(r, t));
        CKL(launch_add_inplace(x, t, n, st));
      }
    }
    RET(A(x, t));
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

int pslr_gmres(pslr_ctx* ctx, int64_t m, const double* b, double* x, double tol, int64_t maxit,
               int64_t restart, int precond, int flexible, int64_t* iterations, int* converged,
               double* final_relres, double* history, int64_t* history_len, void* stream) {
  pslr::NvtxRange nvtx_("pslr_gmres");
  RET(set_device(ctx));
  if (ctx->nghost && !ctx->comm)
    return fail(PSLR_EINVAL, "sharded context: pslr_comm_init + pslr_ctx_set_halo first (or shard.py)");
  cudaStream_t st = S(stream);
  const int64_t n = ctx->n;
  const VecOp A = [ctx, st](const double* in, double* out) { return op_spmv_A_sharded(ctx, in, out, st); };
  const VecOp M = [ctx, m, precond, n, st](const double* in, double* out) -> int {
    if (precond) return op_apply(ctx, m, in, out, st);
    if (out != in) CK(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return PSLR_OK;
  };
  return gmres_core(ctx, n, A, M, b, x, tol, maxit, restart, flexible, iterations, converged, final_relres,
                    history, history_len, st);
}

// A / M: NULL -> the context's reordered matrix / its PSLR apply (precond != 0) or the
// identity (precond == 0); otherwise the callback (any operator on device n-vectors)
static int ctx_ops(pslr_ctx* ctx, int64_t m, int64_t n, pslr_vec_fn A_fn, void* A_user, pslr_vec_fn M_fn,
                   void* M_user, int precond, cudaStream_t st, VecOp* A, VecOp* M) {
  if (!A_fn && n != ctx->n) return fail(PSLR_EDIM, "the context's matrix has another dimension");
  if (!M_fn && precond && n != ctx->n) return fail(PSLR_EDIM, "the context's preconditioner has another dimension");
  if (A_fn)
    *A = callback_op(A_fn, A_user, st);
  else
    *A = [ctx, st](const double* in, double* out) { return op_spmv_A_sharded(ctx, in, out, st); };
  if (M_fn)
    *M = callback_op(M_fn, M_user, st);
  else
    *M = [ctx, m, precond, n, st](const double* in, double* out) -> int {
      if (precond) return op_apply(ctx, m, in, out, st);
      if (out != in) CK(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      return PSLR_OK;
    };
  return PSLR_OK;
}

int pslr_gmres_op(pslr_ctx* ctx, int64_t m, int64_t n, pslr_vec_fn A_fn, void* A_user, pslr_vec_fn M_fn,
                  void* M_user, int precond, const double* b, double* x, double tol, int64_t maxit,
                  int64_t restart, int flexible, int64_t* iterations, int* converged, double* final_relres,
                  double* history, int64_t* history_len, void* stream) {
  pslr::NvtxRange nvtx_("pslr_gmres_op");
  RET(set_device(ctx));
  if (n < 0) return fail(PSLR_EDIM, "negative dimension");
  cudaStream_t st = S(stream);
  VecOp A, M;
  RET(ctx_ops(ctx, m, n, A_fn, A_user, M_fn, M_user, precond, st, &A, &M));
  return gmres_core(ctx, n, A, M, b, x, tol, maxit, restart, flexible, iterations, converged, final_relres,
                    history, history_len, st);
}

int pslr_cgs_pass(pslr_ctx* ctx, int mode, const double* X, int64_t ld, int64_t n, int64_t k, double* w,
                  const double* h0, double* out, void* stream) {
  RET(set_device(ctx));
  if (mode < 0 || mode > 2) return fail(PSLR_EINVAL, "cgs pass mode must be 0, 1 or 2");
  if (n < 0 || k < 1 || ld < n) return fail(PSLR_EDIM, "cgs pass: need k >= 1, n >= 0, ld >= n");
  if (mode != 0 && !h0) return fail(PSLR_EINVAL, "cgs pass: projection coefficients missing");
  cudaStream_t st = S(stream);
  RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)dot_grid(n, ctx->sm_count) * (k + 1) + 8));
  if (mode == 0) CKL(launch_multidot(ctx, X, ld, (int)k, w, n, out, st));
  if (mode == 1) CKL(launch_sub_dot(ctx, X, ld, (int)k, h0, w, n, out, st));
  if (mode == 2) CKL(launch_sub_norm(ctx, X, ld, (int)k, h0, w, n, out, st));
  return PSLR_OK;
}

// krylov.py:132-174.  Device vectors; the scalar recurrence (alpha, beta, the SPD check,
// the residual test) is host code with the reference's exact control flow.
static int cg_core(pslr_ctx* ctx, int64_t n, const VecOp& A, const VecOp& apply_M, const double* b, double* x,
                   double tol, int64_t maxit, int64_t* iterations, int* converged, double* final_relres,
                   double* history, int64_t* history_len, cudaStream_t st) {
  if (maxit < 0) return fail(PSLR_EDIM, "maxit must be >= 0");
  std::vector<double> hist;
  auto finish = [&](bool conv, int64_t its, double rel) {
    *iterations = its;
    *converged = conv ? 1 : 0;
    *final_relres = rel;
    const size_t cnt = std::min<size_t>(hist.size(), (size_t)maxit + 1);
    for (size_t i = 0; i < cnt; ++i) history[i] = hist[i];
    *history_len = (int64_t)cnt;
  };
  double bnorm = 0.0;
  RET(dnorm(ctx, b, n, &bnorm, st));
  CK(cudaMemsetAsync(x, 0, n * sizeof(double), st));
  if (bnorm == 0.0) {  // krylov.py:138-139
    hist.push_back(1.0);
    finish(true, 0, 0.0);
    CK(cudaStreamSynchronize(st));
    return PSLR_OK;
  }
  RET(ensure(ctx, &ctx->kv, &ctx->kv_len, n));
  RET(ensure(ctx, &ctx->red, &ctx->red_len, (int64_t)dot_grid(n, ctx->sm_count) + 8));
  RET(ensure(ctx, &ctx->h_dev, &ctx->h_len, 8));
  double *r = nullptr, *z = nullptr, *Ap = nullptr;
  RET(krylov_vectors(ctx, n, &r, &Ap, &z));
  double* p = ctx->kv;
  auto dot = [&](const double* u, const double* v, double* out) -> int {
    CKL(launch_multidot(ctx, u, n, 1, v, n, ctx->h_dev, st));
    RET(comm_allreduce(ctx, ctx->h_dev, 1, st));
    CK(cudaMemcpyAsync(out, ctx->h_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PSLR_OK;
  };
  CK(cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));  // r = b
  RET(apply_M(r, z));                                                          // z = M r
  CK(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, st));  // p = z
  double rz = 0.0;
  RET(dot(r, z, &rz));
  hist.push_back(1.0);
  bool conv = false;
  double relres = 1.0;
  int64_t it = 0;
  for (it = 1; it <= maxit; ++it) {
    RET(A(p, Ap));  // krylov.py:152
    double pAp = 0.0;
    RET(dot(p, Ap, &pAp));
    if (pAp <= 0.0) {  // krylov.py:153-154
      CK(cudaStreamSynchronize(st));
      return fail(PSLR_ENOTSPD, "matrix not SPD: non-positive curvature encountered");
    }
    const double alpha = rz / pAp;
    CKL(launch_cg_update(ctx, x, r, p, Ap, alpha, n, ctx->h_dev, st));  // x, r, r.r
    RET(comm_allreduce(ctx, ctx->h_dev, 1, st));
    double rr = 0.0;
    CK(cudaMemcpyAsync(&rr, ctx->h_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    relres = std::sqrt(rr) / bnorm;
    hist.push_back(relres);
    if (relres <= tol) {
      conv = true;
      break;
    }
    RET(apply_M(r, z));
    double rz_new = 0.0;
    RET(dot(r, z, &rz_new));
    CKL(launch_xpby(z, rz_new / rz, p, n, st));  // krylov.py:163
    rz = rz_new;
  }
  const int64_t its = conv ? it : maxit;
  if (!conv)
    while ((int64_t)hist.size() < maxit + 1) hist.push_back(relres);
  finish(conv, its, relres);
  CK(cudaStreamSynchronize(st));
  return PSLR_OK;
}

int pslr_cg(pslr_ctx* ctx, int64_t m, const double* b, double* x, double tol, int64_t maxit, int precond,
            int64_t* iterations, int* converged, double* final_relres, double* history,
            int64_t* history_len, void* stream) {
  pslr::NvtxRange nvtx_("pslr_cg");
  RET(set_device(ctx));
  if (ctx->nghost && !ctx->comm)
    return fail(PSLR_EINVAL, "sharded context: pslr_comm_init + pslr_ctx_set_halo first (or shard.py)");
  cudaStream_t st = S(stream);
  VecOp A, M;
  RET(ctx_ops(ctx, m, ctx->n, nullptr, nullptr, nullptr, nullptr, precond, st, &A, &M));
  return cg_core(ctx, ctx->n, A, M, b, x, tol, maxit, iterations, converged, final_relres, history, history_len,
                 st);
}

int pslr_cg_op(pslr_ctx* ctx, int64_t m, int64_t n, pslr_vec_fn A_fn, void* A_user, pslr_vec_fn M_fn,
               void* M_user, int precond, const double* b, double* x, double tol, int64_t maxit,
               int64_t* iterations, int* converged, double* final_relres, double* history, int64_t* history_len,
               void* stream) {
  pslr::NvtxRange nvtx_("pslr_cg_op");
  RET(set_device(ctx));
  if (n < 0) return fail(PSLR_EDIM, "negative dimension");
  cudaStream_t st = S(stream);
  VecOp A, M;
  RET(ctx_ops(ctx, m, n, A_fn, A_user, M_fn, M_user, precond, st, &A, &M));
  return cg_core(ctx, n, A, M, b, x, tol, maxit, iterations, converged, final_relres, history, history_len, st);
}

int pslr_csr_spmv(int64_t nrows, int64_t ncols, const int32_t* indptr, const int32_t* indices, const double* data,
                  const double* x, double* y, void* stream) {
  if (nrows < 0 || ncols < 0 || nrows > 0x7fffffffLL) return fail(PSLR_EDIM, "bad CSR dimensions");
  DevCsr M;
  M.nrows = (int32_t)nrows;
  M.ncols = (int32_t)ncols;
  M.ptr = indptr;
  M.col = indices;
  M.val = data;
  CKL(launch_spmv(M, x, y, S(stream)));
  return PSLR_OK;
}

}  // extern "C"
