// pslr_ops.h — internal operator/launcher declarations shared by capi.cu and krylov.cu.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "pslr_internal.h"

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
#define RET(expr)                 \
  do {                            \
    int _r = (expr);              \
    if (_r != PSLR_OK) return _r; \
  } while (0)

namespace pslr {

// Launch kinds recorded by pslr_apply_profiled: 0 generic step, 1 correction core,
// 2 apply-first (B solve + F), 3 correction + C0, 4 Horner step (E, B solve, F, Cg,
// C0 solve), 5 apply-last (E, B solve).
enum LaunchKind : int32_t {
  LK_STEP = 0, LK_CORE = 1, LK_FIRST = 2, LK_CORR = 3, LK_HORNER = 4, LK_LAST = 5, LK_PERMUTE = 6
};

// kernels.cu
int configure_step_kernel(int nv, int smem_bytes);
int launch_step(const pslr_ctx* ctx, const StepArgs& a, cudaStream_t st, int nv = 1);
int launch_correction_core(const pslr_ctx* ctx, cudaStream_t st);
int launch_spmv(const DevCsr& M, const double* x, double* y, cudaStream_t st);
int launch_multidot(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* y, int64_t n,
                    double* out, cudaStream_t st);
// CGS2 passes (k <= 128 columns): w -= X h0 then h = X^T w  /  w -= X h0 then out[0] = w.w
int launch_sub_dot(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* h0, double* w,
                   int64_t n, double* out, cudaStream_t st);
int launch_sub_norm(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* h0, double* w,
                    int64_t n, double* out, cudaStream_t st);
int launch_gemv(const double* X, int64_t ld, int k, const double* h, double* y, int64_t n,
                cudaStream_t st);
// CG (krylov.py:156-163): x += alpha p ; r -= alpha Ap ; out[0] = r.r   /   p = z + beta p
int launch_cg_update(pslr_ctx* ctx, double* x, double* r, const double* p, const double* Ap, double alpha,
                     int64_t n, double* out, cudaStream_t st);
int launch_xpby(const double* z, double beta, double* p, int64_t n, cudaStream_t st);
int launch_sqrt(const double* in, double* out, cudaStream_t st);
int launch_sub(const double* a, const double* b, double* y, int64_t n, cudaStream_t st);
int launch_add_inplace(double* y, const double* a, int64_t n, cudaStream_t st);
int launch_div_scalar(const double* x, const double* s, double* y, int64_t n, cudaStream_t st);
int launch_transpose_basis(const double* X, int64_t ld, int64_t q, int r, double* Y, cudaStream_t st);
int dot_grid(int64_t n, int sm_count);
int vt_grid(int64_t q, int sm_count);
int launch_vt_dot(pslr_ctx* ctx, const double* y, cudaStream_t st);
int launch_vt_local(pslr_ctx* ctx, const double* y, double* s, cudaStream_t st);
int launch_gs(pslr_ctx* ctx, const double* s, cudaStream_t st);
int launch_permute_f(const pslr_ctx* ctx, const double* f, cudaStream_t st);
int launch_vu_add(const pslr_ctx* ctx, const double* y, double* out, cudaStream_t st);
// two interleaved right-hand sides ([row][2]): strided correction, (de)interleaving
int launch_vt_dot_strided(pslr_ctx* ctx, const double* y, int64_t ys, cudaStream_t st);
int launch_vu_add_strided(const pslr_ctx* ctx, const double* y, int64_t ys, double* out, int64_t os,
                          cudaStream_t st);
int launch_permute2(const pslr_ctx* ctx, const double* b, cudaStream_t st);
int launch_deinterleave2(const pslr_ctx* ctx, const double* y2, double* z, cudaStream_t st);
int launch_vt_local_strided(pslr_ctx* ctx, const double* y, int64_t ys, double* s, cudaStream_t st);

// comm.cu (multi-GPU contexts; no-ops without a communicator)
int comm_allreduce(pslr_ctx* ctx, double* x, int64_t n, cudaStream_t st);
int comm_halo(pslr_ctx* ctx, double* v_ext, cudaStream_t st);
int comm_destroy(pslr_ctx* ctx);
int op_apply_sharded(pslr_ctx* ctx, int64_t m, const double* b, double* z, cudaStream_t st);
int op_apply2_sharded(pslr_ctx* ctx, int64_t m, const double* b2, double* z2, cudaStream_t st);
int comm_halo2(pslr_ctx* ctx, double* v2_ext, cudaStream_t st);
// the exchange on the communication stream, consumed by the next launch_step (comm.cu)
int comm_halo_async(pslr_ctx* ctx, double* v_ext, int nv, cudaStream_t st);
int comm_halo_join(pslr_ctx* ctx, cudaStream_t st);
int op_apply_err_sharded(pslr_ctx* ctx, int64_t m, const double* v, double* out, cudaStream_t st);
int op_spmv_A_sharded(pslr_ctx* ctx, const double* x, double* w, cudaStream_t st);

// capi.cu
int alloc_scratch(pslr_ctx* ctx, double** p, int64_t count);
void free_ptr(pslr_ctx* ctx, void* p);
int ensure(pslr_ctx* ctx, double** p, int64_t* len, int64_t need);
int set_device(const pslr_ctx* ctx);
int op_solve_B(pslr_ctx* ctx, const double* f, double* x, cudaStream_t st);
int op_solve_C0(pslr_ctx* ctx, const double* g, double* y, cudaStream_t st);
int op_es_step(pslr_ctx* ctx, const double* v, double* out, int do_c0, const double* cadd,
               cudaStream_t st);
int op_horner(pslr_ctx* ctx, int64_t m, const double* c, double* out, cudaStream_t st);
int op_apply(pslr_ctx* ctx, int64_t m, const double* b, double* z, cudaStream_t st);
int op_apply_err(pslr_ctx* ctx, int64_t m, const double* v, double* out, cudaStream_t st);

}  // namespace pslr
