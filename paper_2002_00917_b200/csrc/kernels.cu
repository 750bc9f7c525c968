// kernels.cu — sm_100a kernels of the PSLR hot path.
//
// Arithmetic contract (bit-exact parity with the reference's scipy calls):
//  * the library is compiled with -fmad=false: every multiply and add rounds
//    separately, as numpy/scipy (no FMA on their x86-64 baseline builds) do;
//  * SpMV rows are summed sequentially from 0 in CSR order (scipy csr_matvec);
//  * the unit-lower solve is  z_i = b_i - L_ij z_j ... in ascending j  and the
//    upper solve is the scaled form scipy's spsolve_triangular hands to SuperLU
//    gstrs:  z_i = b_i/sd_i - U'_ij z_j ...,  x_i = z_i * invd_i  (ilu.py:194-195);
//  * any dependency-respecting schedule yields the same per-row operation
//    sequence, so the level-scheduled solves equal the sequential ones bit for bit.
#include <cuda_runtime.h>

#include "pslr_internal.h"

namespace pslr {

constexpr int kStepThreads = 512;

__device__ __forceinline__ double spmv_row(const DevCsr& M, int row, const double* __restrict__ x) {
  double s = 0.0;
  const int e1 = M.ptr[row + 1];
  for (int e = M.ptr[row]; e < e1; ++e) s = s + M.val[e] * x[M.col[e]];
  return s;
}

// Unit-lower solve of block b, in place on z (z holds the right-hand side).
__device__ void cta_trsv_lower(const DevTri& T, int b, double* z) {
  const int l0 = T.blk_lvl[b], l1 = T.blk_lvl[b + 1];
  for (int lv = l0; lv < l1; ++lv) {
    const int p0 = T.lvl_pos[lv], p1 = T.lvl_pos[lv + 1];
    for (int pos = p0 + (int)threadIdx.x; pos < p1; pos += blockDim.x) {
      const int row = T.pos_row[pos];
      const int e1 = T.pos_ent[pos + 1];
      double t = z[row];
      for (int e = T.pos_ent[pos]; e < e1; ++e) t = t - T.val[e] * z[T.col[e]];
      z[row] = t;
    }
    __syncthreads();
  }
}

// Upper solve of block b: z holds the right-hand side and receives the scaled
// intermediate; x receives z*invd (+ cadd when given).
__device__ void cta_trsv_upper(const DevTri& T, int b, double* z, double* x,
                               const double* __restrict__ cadd) {
  const int l0 = T.blk_lvl[b], l1 = T.blk_lvl[b + 1];
  for (int lv = l0; lv < l1; ++lv) {
    const int p0 = T.lvl_pos[lv], p1 = T.lvl_pos[lv + 1];
    for (int pos = p0 + (int)threadIdx.x; pos < p1; pos += blockDim.x) {
      const int row = T.pos_row[pos];
      const int e1 = T.pos_ent[pos + 1];
      double t = z[row] / T.sd[pos];
      for (int e = T.pos_ent[pos]; e < e1; ++e) t = t - T.val[e] * z[T.col[e]];
      z[row] = t;
      double out = t * T.invd[pos];
      if (cadd) out = out + cadd[row];
      x[row] = out;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double iface_term(int kind, int row, const StepArgs& a, const DevCsr& F,
                                             const DevCsr& C, const DevCsr& Cg,
                                             const double* __restrict__ V, int r) {
  switch (kind) {
    case IT_G: return a.g[row];
    case IT_FX: return spmv_row(F, row, a.xb);
    case IT_CY: return spmv_row(C, row, a.yC);
    case IT_CGY: return spmv_row(Cg, row, a.yC);
    case IT_VU: {
      double s = 0.0;
      const double* vr = V + (int64_t)row * r;
      for (int c = 0; c < r; ++c) s = s + vr[c] * a.u[c];
      return s;
    }
    default: return 0.0;
  }
}

// One CTA per subdomain: the whole per-subdomain chain of one PSLR step.
//   interior phase:  xb = B_b^{-1} (b1 (-) b2)            (B solve, E folded into the rhs)
//   interface phase: w = i1 (+|-) i2 ; y = [C0_b^{-1}] w [+ cadd] ; [partials = V_b^T y]
// Only Cg couples subdomains, and it reads a vector produced by a previous launch,
// so one launch per Horner step is the only grid-wide synchronisation needed.
__global__ void __launch_bounds__(kStepThreads)
subdomain_step_kernel(StepArgs a, DevTri LB, DevTri UB, DevTri LC, DevTri UC, DevCsr E, DevCsr F,
                      DevCsr C, DevCsr Cg, const int32_t* __restrict__ int_off,
                      const int32_t* __restrict__ ifc_off, const double* __restrict__ V, int r) {
  const int b = blockIdx.x;
  if (a.b1 != BT_NONE) {
    const int r0 = int_off[b], r1 = int_off[b + 1];
    for (int row = r0 + (int)threadIdx.x; row < r1; row += blockDim.x) {
      double v = (a.b1 == BT_F) ? a.f[row] : spmv_row(E, row, a.yE);
      if (a.b2 == BT_EY) v = v - spmv_row(E, row, a.yE);
      a.tb[row] = v;
    }
    __syncthreads();
    cta_trsv_lower(LB, b, a.tb);
    cta_trsv_upper(UB, b, a.tb, a.xb, nullptr);
  }
  if (a.i1 != IT_NONE) {
    const int r0 = ifc_off[b], r1 = ifc_off[b + 1];
    for (int row = r0 + (int)threadIdx.x; row < r1; row += blockDim.x) {
      double w = iface_term(a.i1, row, a, F, C, Cg, V, r);
      if (a.i2 != IT_NONE) {
        const double t2 = iface_term(a.i2, row, a, F, C, Cg, V, r);
        w = a.i2_sub ? (w - t2) : (w + t2);
      }
      if (a.do_c0) {
        a.tw[row] = w;
      } else {
        if (a.cadd) w = w + a.cadd[row];
        a.yout[row] = w;
      }
    }
    __syncthreads();
    if (a.do_c0) {
      cta_trsv_lower(LC, b, a.tw);
      cta_trsv_upper(UC, b, a.tw, a.yout, a.cadd);
    }
    if (a.partials) {
      // partials[b][c] = sum_{rows of b} V[row][c] * yout[row]; deterministic order
      __shared__ double red[kStepThreads / 32][128];
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int c0 = 0; c0 < r; c0 += 128) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int row = r0 + warp; row < r1; row += nw) {
          const double y = a.yout[row];
          const double* vr = V + (int64_t)row * r;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int c = c0 + lane + 32 * k;
            if (c < r) acc[k] = acc[k] + vr[c] * y;
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) red[warp][lane + 32 * k] = acc[k];
        __syncthreads();
        for (int c = threadIdx.x; c < 128; c += blockDim.x) {
          double s = 0.0;
          for (int w2 = 0; w2 < nw; ++w2) s = s + red[w2][c];
          if (c0 + c < r) a.partials[(int64_t)b * r + c0 + c] = s;
        }
        __syncthreads();
      }
    }
  }
}

// u = G (sum_b partials[b]) ; one CTA. h lives in u[r..2r).
__global__ void correction_core_kernel(const double* __restrict__ partials, int s, int r,
                                       const double* __restrict__ G, double* u) {
  double* h = u + r;
  for (int c = threadIdx.x; c < r; c += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < s; ++b) acc = acc + partials[(int64_t)b * r + c];
    h[c] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    double acc = 0.0;
    const double* gi = G + (int64_t)i * r;
    for (int c = 0; c < r; ++c) acc = acc + gi[c] * h[c];
    u[i] = acc;
  }
}

// y = M x, one thread per row (scipy csr_matvec order).
__global__ void spmv_kernel(DevCsr M, const double* __restrict__ x, double* __restrict__ y) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < M.nrows) y[row] = spmv_row(M, row, x);
}

// ---------------------------------------------------------------- Krylov building blocks
// out[c] = sum_i X[c*ld + i] * y[i], c < k.  Grid-stride partials + last-block
// reduction in a fixed order (deterministic, no atomics on values).
constexpr int kDotThreads = 256;
constexpr int kDotCols = 4;

__global__ void __launch_bounds__(kDotThreads)
multidot_kernel(const double* __restrict__ X, int64_t ld, int k, const double* __restrict__ y,
                int64_t n, double* __restrict__ partials, double* __restrict__ out,
                unsigned int* counter) {
  __shared__ double sh[kDotCols][kDotThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int c0 = 0; c0 < k; c0 += kDotCols) {
    double acc[kDotCols] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const double yi = y[i];
#pragma unroll
      for (int t = 0; t < kDotCols; ++t)
        if (c0 + t < k) acc[t] = acc[t] + X[(int64_t)(c0 + t) * ld + i] * yi;
    }
#pragma unroll
    for (int t = 0; t < kDotCols; ++t) {
      double v = acc[t];
      for (int o = 16; o > 0; o >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) sh[t][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < kDotCols && c0 + (int)threadIdx.x < k) {
      double v = 0.0;
      for (int w = 0; w < kDotThreads / 32; ++w) v = v + sh[threadIdx.x][w];
      partials[(int64_t)blockIdx.x * k + c0 + threadIdx.x] = v;
    }
    __syncthreads();
  }
  __threadfence();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (last) {
    __threadfence();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      double v = 0.0;
      for (int g = 0; g < (int)gridDim.x; ++g) v = v + ((volatile double*)partials)[(int64_t)g * k + c];
      out[c] = v;
    }
    if (threadIdx.x == 0) *counter = 0u;
  }
}

// w[i] = w[i] - sum_c X[c*ld + i] * h[c]   (w - V h, numpy order: V@h first)
__global__ void gemv_sub_kernel(const double* __restrict__ X, int64_t ld, int k,
                                const double* __restrict__ h, double* __restrict__ w, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int c = 0; c < k; ++c) s = s + X[(int64_t)c * ld + i] * h[c];
  w[i] = w[i] - s;
}

// y[i] = sum_c X[c*ld + i] * h[c]   (V y)
__global__ void gemv_kernel(const double* __restrict__ X, int64_t ld, int k,
                            const double* __restrict__ h, double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int c = 0; c < k; ++c) s = s + X[(int64_t)c * ld + i] * h[c];
  y[i] = s;
}

// y = a - b
__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] - b[i];
}

// y = y + a
__global__ void add_inplace_kernel(double* __restrict__ y, const double* __restrict__ a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = y[i] + a[i];
}

// y = x * (1/s) computed as x / s (numpy: w / hnext)
__global__ void div_scalar_kernel(const double* __restrict__ x, const double* __restrict__ s,
                                  double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / *s;
}

// row-major (q x r) <- column-major (ld = q) transpose for the Arnoldi basis
__global__ void colmajor_to_rowmajor_kernel(const double* __restrict__ X, int64_t q, int r,
                                            double* __restrict__ Y) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= q * r) return;
  const int64_t i = idx / r;
  const int c = (int)(idx % r);
  Y[idx] = X[(int64_t)c * q + i];
}

// ---------------------------------------------------------------- host-side launchers
int launch_step(const pslr_ctx* ctx, const StepArgs& a, cudaStream_t st) {
  if (ctx->s == 0) return 0;
  subdomain_step_kernel<<<(unsigned)ctx->s, kStepThreads, 0, st>>>(
      a, ctx->LB, ctx->UB, ctx->LC, ctx->UC, ctx->E, ctx->F, ctx->C, ctx->Cg, ctx->d_int_off,
      ctx->d_ifc_off, ctx->V, (int)ctx->r);
  return (int)cudaGetLastError();
}

int launch_correction_core(const pslr_ctx* ctx, cudaStream_t st) {
  correction_core_kernel<<<1, 256, 0, st>>>(ctx->partials, (int)ctx->s, (int)ctx->r, ctx->G, ctx->u);
  return (int)cudaGetLastError();
}

int launch_spmv(const DevCsr& M, const double* x, double* y, cudaStream_t st) {
  if (M.nrows == 0) return 0;
  spmv_kernel<<<(M.nrows + 255) / 256, 256, 0, st>>>(M, x, y);
  return (int)cudaGetLastError();
}

int dot_grid(int64_t n, int sm_count) {
  int64_t g = (n + kDotThreads * 4 - 1) / (kDotThreads * 4);
  const int64_t cap = 2 * (int64_t)sm_count;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

int launch_multidot(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* y, int64_t n,
                    double* out, cudaStream_t st) {
  if (k <= 0) return 0;
  const int g = dot_grid(n, ctx->sm_count);
  multidot_kernel<<<g, kDotThreads, 0, st>>>(X, ld, k, y, n, ctx->red, out, ctx->counter);
  return (int)cudaGetLastError();
}

int launch_gemv_sub(const double* X, int64_t ld, int k, const double* h, double* w, int64_t n,
                    cudaStream_t st) {
  if (n == 0) return 0;
  gemv_sub_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(X, ld, k, h, w, n);
  return (int)cudaGetLastError();
}

int launch_gemv(const double* X, int64_t ld, int k, const double* h, double* y, int64_t n,
                cudaStream_t st) {
  if (n == 0) return 0;
  gemv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(X, ld, k, h, y, n);
  return (int)cudaGetLastError();
}

int launch_sub(const double* a, const double* b, double* y, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  sub_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, b, y, n);
  return (int)cudaGetLastError();
}

int launch_add_inplace(double* y, const double* a, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  add_inplace_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, a, n);
  return (int)cudaGetLastError();
}

int launch_div_scalar(const double* x, const double* s, double* y, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  div_scalar_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, s, y, n);
  return (int)cudaGetLastError();
}

int launch_transpose_basis(const double* X, int64_t q, int r, double* Y, cudaStream_t st) {
  if (q * r == 0) return 0;
  colmajor_to_rowmajor_kernel<<<(unsigned)((q * r + 255) / 256), 256, 0, st>>>(X, q, r, Y);
  return (int)cudaGetLastError();
}

}  // namespace pslr
