// kernels.cu — the non-solve sm_100a kernels of the PSLR hot path: the
// correction core, CSR SpMV (the A operator of GMRES) and the Krylov building
// blocks (multi-dot, GEMV updates, scaling).  The fused solve kernel is in
// step_kernel.cu.
//
// Arithmetic contract: compiled with -fmad=false (every multiply and add rounds
// separately, as numpy/scipy on x86-64 baseline do); SpMV rows are summed
// sequentially from 0 in CSR order (scipy csr_matvec), so A @ v is bit-exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <utility>

#include "pslr_internal.h"

namespace pslr {

// Programmatic dependent launch for the vector kernels (Krylov passes, correction, SpMV,
// permutes): a kernel may be launched while the previous kernel of its stream drains;
// pdl_wait() at the top of every kernel orders all its memory accesses after that kernel
// (a no-op for an ordinary launch).  PSLR_PDL=0 turns the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

static bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PSLR_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

template <class... KArgs, class... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ double csr_row(const DevCsr& M, int row, const double* __restrict__ x) {
  double s = 0.0;
  const int e1 = M.ptr[row + 1];
  for (int e = M.ptr[row]; e < e1; ++e) s = s + M.val[e] * x[M.col[e]];
  return s;
}

// u = G (sum_b partials[b]) ; one CTA. h lives in u[r..2r).
__global__ void correction_core_kernel(const double* __restrict__ partials, int s, int r,
                                       const double* __restrict__ G, double* u) {
  pdl_wait();
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

// ---------------------------------------------------------------- rank-r correction
// u = G (V^T y) for row-major V (q x r), all SMs: each warp accumulates rows with lanes on
// columns, a block reduction writes per-CTA partials, the last CTA sums them in a fixed
// order (deterministic) and applies G.  h = V^T y lives in hu[r..2r), u in hu[0..r).
constexpr int kVtThreads = 256;

__global__ void __launch_bounds__(kVtThreads)
vt_dot_kernel(const double* __restrict__ V, const double* __restrict__ y, int64_t ys, int64_t q, int r,
              const double* __restrict__ G, double* __restrict__ partials, double* hu,
              unsigned int* counter) {
  pdl_wait();
  __shared__ double red[kVtThreads / 32][128];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kVtThreads / 32;
  const int64_t stride = (int64_t)gridDim.x * nw;
  if (r <= 64) {
    // two columns per lane, eight rows in flight per warp (V rows are 512 B at r = 64)
    double a0 = 0.0, a1 = 0.0;
    const bool v0 = lane < r, v1 = lane + 32 < r;
    int64_t row = (int64_t)blockIdx.x * nw + warp;
    for (; row < q; row += 8 * stride) {  // predicated batches: the tail is one batch too
      double yv[8], x0[8], x1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t ru = row + u * stride;
        const bool ok = ru < q;
        const double* vr = V + ru * r;
        yv[u] = ok ? __ldg(y + ru * ys) : 0.0;
        x0[u] = (ok && v0) ? __ldg(vr + lane) : 0.0;
        x1[u] = (ok && v1) ? __ldg(vr + lane + 32) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 = a0 + x0[u] * yv[u];
        a1 = a1 + x1[u] * yv[u];
      }
    }
    red[warp][lane] = a0;
    red[warp][lane + 32] = a1;
    __syncthreads();
    for (int c = threadIdx.x; c < r; c += kVtThreads) {
      double sum = 0.0;
      for (int w = 0; w < nw; ++w) sum = sum + red[w][c];
      partials[(int64_t)blockIdx.x * r + c] = sum;
    }
  }
  for (int c0 = 0; c0 < r && r > 64; c0 += 128) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t row = (int64_t)blockIdx.x * nw + warp;
    // four rows per iteration: their loads are independent and in flight together
    for (; row + 3 * stride < q; row += 4 * stride) {
      double yv[4], vv[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        yv[u] = __ldg(y + (row + u * stride) * ys);
        const double* vr = V + (row + u * stride) * r;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = c0 + lane + 32 * k;
          vv[u][k] = (c < r) ? __ldg(vr + c) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (c0 + lane + 32 * k < r) acc[k] = acc[k] + vv[u][k] * yv[u];
    }
    for (; row < q; row += stride) {
      const double yv = __ldg(y + row * ys);
      const double* vr = V + row * r;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = c0 + lane + 32 * k;
        if (c < r) acc[k] = acc[k] + __ldg(vr + c) * yv;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) red[warp][lane + 32 * k] = acc[k];
    __syncthreads();
    for (int c = threadIdx.x; c < 128 && c0 + c < r; c += kVtThreads) {
      double sum = 0.0;
      for (int w = 0; w < nw; ++w) sum = sum + red[w][c];
      partials[(int64_t)blockIdx.x * r + c0 + c] = sum;
    }
    __syncthreads();
  }
  __threadfence();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double* h = hu + r;
  for (int c = threadIdx.x; c < r; c += kVtThreads) {
    double s = 0.0;
    for (int g = 0; g < (int)gridDim.x; ++g) s = s + ((volatile double*)partials)[(int64_t)g * r + c];
    h[c] = s;
  }
  __syncthreads();
  if (G)  // sharded contexts stop at h: the ranks sum it before G is applied
    for (int i = threadIdx.x; i < r; i += kVtThreads) {
      double s = 0.0;
      const double* gi = G + (int64_t)i * r;
      for (int c = 0; c < r; ++c) s = s + gi[c] * ((volatile double*)h)[c];
      hu[i] = s;
    }
  if (threadIdx.x == 0) *counter = 0u;
}

// u = G s (one CTA): the correction core after the ranks' V^T y partial sums are reduced
__global__ void gs_kernel(const double* __restrict__ G, const double* __restrict__ s, double* u, int r) {
  pdl_wait();
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    double acc = 0.0;
    const double* gi = G + (int64_t)i * r;
    for (int c = 0; c < r; ++c) acc = acc + gi[c] * s[c];
    u[i] = acc;
  }
}

// out = y + V u (one warp per row, lanes on columns, fixed shuffle-tree reduction)
__global__ void vu_add_kernel(const double* __restrict__ V, const double* __restrict__ u,
                              const double* __restrict__ y, int64_t ys, double* __restrict__ out,
                              int64_t os, int64_t q, int r) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r <= 64) {  // two columns per lane, four rows in flight per warp
    const double u0 = lane < r ? __ldg(u + lane) : 0.0, u1 = lane + 32 < r ? __ldg(u + lane + 32) : 0.0;
    for (; row < q; row += 4 * nwarps) {  // predicated batches: the tail is one batch too
      double s[4], yv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        yv[k] = (lane == 0 && row + k * nwarps < q) ? __ldg(y + (row + k * nwarps) * ys) : 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ok = row + k * nwarps < q;
        const double* vr = V + (row + k * nwarps) * r;
        const double a = (ok && lane < r) ? __ldg(vr + lane) : 0.0;
        const double b = (ok && lane + 32 < r) ? __ldg(vr + lane + 32) : 0.0;
        s[k] = (lane < r ? a * u0 : 0.0);
        s[k] = s[k] + (lane + 32 < r ? b * u1 : 0.0);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < 4; ++k) s[k] = s[k] + __shfl_xor_sync(0xffffffffu, s[k], o);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (row + k * nwarps < q) out[(row + k * nwarps) * os] = yv[k] + s[k];
    }
    return;
  }
  for (; row < q; row += nwarps) {
    const double* vr = V + row * r;
    double s = 0.0;
    for (int c = lane; c < r; c += 32) s = s + __ldg(vr + c) * __ldg(u + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[row * os] = __ldg(y + row * ys) + s;
  }
}

// fL[pos] = f[row at pos]: the L solve's right-hand side in position order, on all SMs
__global__ void permute_f_kernel(const int32_t* __restrict__ lrow, const double* __restrict__ f,
                                 double* __restrict__ fL, int64_t p) {
  pdl_wait();
  // gather form: coalesced stores, the random reads of f (15 MB at cfg5) hit L2
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x)
    fL[i] = __ldg(f + __ldg(lrow + i));
}

// Level-merged L_B (pack.cpp merge_levels): a merged row's right-hand side is
// f_i - (c0 f_j0 + c1 f_j1 + c2 f_j2); lrowx holds -(record + 1) at its position.
template <int NV>
__device__ __forceinline__ void permute_x_one(const int32_t* __restrict__ lrowx, const int4* __restrict__ xrows,
                                              const double2* __restrict__ xval, const double* __restrict__ b,
                                              int64_t n, double* __restrict__ fL, int64_t i) {
  auto ld = [&](int64_t row) -> double2 {
    return make_double2(__ldg(b + row), NV == 2 ? __ldg(b + n + row) : 0.0);
  };
  const int r = __ldg(lrowx + i);
  double2 v;
  if (r >= 0) {
    v = ld(r);
  } else {
    const int k = -r - 1;
    const int4 id = __ldg(xrows + k);
    const double2 c01 = __ldg(xval + 2 * k), c2 = __ldg(xval + 2 * k + 1);
    const double2 fi = ld(id.x), f0 = ld(id.y), f1 = ld(id.z), f2 = ld(id.w);
    double tx = f0.x * c01.x;
    tx = tx + c01.y * f1.x;
    tx = tx + c2.x * f2.x;
    double ty = f0.y * c01.x;
    ty = ty + c01.y * f1.y;
    ty = ty + c2.x * f2.y;
    v = make_double2(fi.x - tx, fi.y - ty);
  }
  if (NV == 2)
    reinterpret_cast<double2*>(fL)[i] = v;
  else
    fL[i] = v.x;
}

__global__ void permute_fx_kernel(const int32_t* __restrict__ lrowx, const int4* __restrict__ xrows,
                                  const double2* __restrict__ xval, const double* __restrict__ f,
                                  double* __restrict__ fL, int64_t p) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x)
    permute_x_one<1>(lrowx, xrows, xval, f, 0, fL, i);
}

int launch_permute_f(const pslr_ctx* ctx, const double* f, cudaStream_t st) {
  if (ctx->p == 0) return 0;
  const int blocks = 4 * ctx->sm_count;
  if (ctx->K.lrowx)
    launch_pdl(permute_fx_kernel, dim3(blocks), dim3(512), 0, st, ctx->K.lrowx,
               reinterpret_cast<const int4*>(ctx->K.xlb_rows), reinterpret_cast<const double2*>(ctx->K.XLB.val), f,
               ctx->fL, ctx->p);
  else
    launch_pdl(permute_f_kernel, dim3(blocks), dim3(512), 0, st, ctx->K.LB.lrow, f, ctx->fL, ctx->p);
  return (int)cudaGetLastError();
}

// Two right-hand sides ([row][2] interleaved inside the step kernels): b and z are the
// caller's two vectors of n, vector-major.  fL2[pos][v] = f_v[row at pos], g2[i][v] = g_v[i].
__global__ void permute2_kernel(const int32_t* __restrict__ lrow, const double* __restrict__ b, int64_t n,
                                int64_t p, int64_t q, double* __restrict__ fL2, double* __restrict__ g2) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p + q; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < p) {
      const int64_t row = __ldg(lrow + i);
      reinterpret_cast<double2*>(fL2)[i] = make_double2(__ldg(b + row), __ldg(b + n + row));
    } else {
      const int64_t k = i - p;
      reinterpret_cast<double2*>(g2)[k] = make_double2(__ldg(b + p + k), __ldg(b + n + p + k));
    }
  }
}

__global__ void permute2x_kernel(const int32_t* __restrict__ lrowx, const int4* __restrict__ xrows,
                                 const double2* __restrict__ xval, const double* __restrict__ b, int64_t n,
                                 int64_t p, int64_t q, double* __restrict__ fL2, double* __restrict__ g2) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p + q; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < p) {
      permute_x_one<2>(lrowx, xrows, xval, b, n, fL2, i);
    } else {
      const int64_t k = i - p;
      reinterpret_cast<double2*>(g2)[k] = make_double2(__ldg(b + p + k), __ldg(b + n + p + k));
    }
  }
}

__global__ void deinterleave2_kernel(const double* __restrict__ x2, const double* __restrict__ y2, int64_t n,
                                     int64_t p, double* __restrict__ z) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = (i < p) ? reinterpret_cast<const double2*>(x2)[i] : reinterpret_cast<const double2*>(y2)[i - p];
    z[i] = v.x;
    z[n + i] = v.y;
  }
}

int vt_grid(int64_t q, int sm_count);

int launch_permute2(const pslr_ctx* ctx, const double* b, cudaStream_t st) {
  if (ctx->K.lrowx)
    launch_pdl(permute2x_kernel, dim3(4 * ctx->sm_count), dim3(512), 0, st, ctx->K.lrowx,
               reinterpret_cast<const int4*>(ctx->K.xlb_rows), reinterpret_cast<const double2*>(ctx->K.XLB.val), b,
               ctx->n, ctx->p, ctx->q, ctx->fL2, ctx->g2);
  else
    launch_pdl(permute2_kernel, dim3(4 * ctx->sm_count), dim3(512), 0, st, ctx->K.LB.lrow, b, ctx->n, ctx->p,
               ctx->q, ctx->fL2, ctx->g2);
  return (int)cudaGetLastError();
}

int launch_deinterleave2(const pslr_ctx* ctx, const double* y2, double* z, cudaStream_t st) {
  launch_pdl(deinterleave2_kernel, dim3(4 * ctx->sm_count), dim3(512), 0, st, ctx->xF2, y2, ctx->n, ctx->p, z);
  return (int)cudaGetLastError();
}

int launch_vt_dot_strided(pslr_ctx* ctx, const double* y, int64_t ys, cudaStream_t st) {
  const int g = vt_grid(ctx->q, ctx->sm_count);
  launch_pdl(vt_dot_kernel, dim3(g), dim3(kVtThreads), 0, st, ctx->V, y, ys, ctx->q, (int)ctx->r, ctx->G, ctx->red, ctx->u,
                                          ctx->counter);
  return (int)cudaGetLastError();
}

int launch_vu_add_strided(const pslr_ctx* ctx, const double* y, int64_t ys, double* out, int64_t os,
                          cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>((ctx->q + 7) / 8, 8 * (int64_t)ctx->sm_count);
  launch_pdl(vu_add_kernel, dim3((unsigned)std::max<int64_t>(blocks, 1)), dim3(256), 0, st, ctx->V, ctx->u, y, ys, out, os, ctx->q,
                                                                        (int)ctx->r);
  return (int)cudaGetLastError();
}

// y = M x, one thread per row (scipy csr_matvec order).
__global__ void spmv_kernel(DevCsr M, const double* __restrict__ x, double* __restrict__ y) {
  pdl_wait();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < M.nrows) y[row] = csr_row(M, row, x);
}

// ---------------------------------------------------------------- Krylov building blocks
// Column-major Krylov basis passes (X: k columns, ld = n), the blocks of CGS2
// (krylov.py:75-80, lowrank.py:62-67).  One kernel, three modes, each ONE pass over X:
//   kDot:     h = X^T w
//   kSubDot:  w = w - X h0 ; h = X^T w        (first projection fused with the second dot)
//   kSubNorm: w = w - X h0 ; h[0] = w . w     (second projection fused with the norm)
// so CGS2 + norm reads the basis three times instead of four plus one.  A CTA walks
// 256-row tiles (grid-stride): phase A (thread = row) forms w_i - sum_c X[c,i] h0[c]
// in column order (numpy's w - V@h); phase B (warp = column set c = warp + 8j, lanes on
// rows) accumulates X[c, tile] . w_tile lane-locally, re-reading the tile phase A just
// brought into L1.  Per-CTA partials are summed by the last CTA in a fixed order
// (deterministic, no atomics on values).
constexpr int kCgsThreads = 256;
constexpr int kCgsWarps = kCgsThreads / 32;
constexpr int kCgsMaxCols = 128;
enum CgsMode : int { kDot = 0, kSubDot = 1, kSubNorm = 2 };

// resident CTAs per SM the register budget is set for: the fused mode-1 pass (two dependent
// phases per tile) gains from occupancy (3 CTAs at 80 registers: k = 10 / 25 / 50 columns
// 69 -> 56 / 116 -> 99 / 203 -> 190 us), the one-phase passes from registers (2 CTAs at 128)
#ifndef PSLR_CGS_MINB1
#define PSLR_CGS_MINB1 3
#endif
template <int MODE, int CPW>  // CPW: columns per warp (k <= 8 * CPW)
__global__ void __launch_bounds__(kCgsThreads, MODE == 1 ? PSLR_CGS_MINB1 : 2)
cgs_pass_kernel(const double* __restrict__ X, int64_t ld, int k, double* __restrict__ w, int64_t n,
                const double* __restrict__ h0, double* __restrict__ partials, double* __restrict__ out,
                unsigned int* counter) {
  pdl_wait();
  __shared__ double hs[kCgsMaxCols];
  __shared__ double ws[kCgsThreads];
  __shared__ double nred[kCgsWarps];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (MODE != kDot)
    for (int c = tid; c < k; c += kCgsThreads) hs[c] = h0[c];
  __syncthreads();
  double acc[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) acc[j] = 0.0;
  double nacc = 0.0;
  const int64_t ntiles = (n + kCgsThreads - 1) / kCgsThreads;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * kCgsThreads;
    const int64_t i = base + tid;
    double wi = (i < n) ? w[i] : 0.0;
    if (MODE != kDot) {
      double s = 0.0;
      if (i < n) {
        // w_i - sum_c X[c,i] h0[c] in column order, the next 8 columns' loads in flight
        // while the current 8 fold (two register buffers: a batch's load latency hides
        // behind the previous batch's dependent DADD chain)
        const double* xi = X + i;
        double va[8], vb[8];
        auto load8 = [&](double (&v)[8], int c0) {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = (c0 + u < k) ? xi[(int64_t)(c0 + u) * ld] : 0.0;
        };
        auto fold8 = [&](const double (&v)[8], int c0) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c0 + u < k) s = s + v[u] * hs[c0 + u];
        };
        load8(va, 0);
        for (int c = 0; c < k; c += 16) {
          if (c + 8 < k) load8(vb, c + 8);
          fold8(va, c);
          if (c + 16 < k) load8(va, c + 16);
          if (c + 8 < k) fold8(vb, c + 8);
        }
        wi = wi - s;
        w[i] = wi;
      }
    }
    if (MODE == kSubNorm) {
      nacc = nacc + wi * wi;
      continue;
    }
    ws[tid] = wi;
    __syncthreads();
    // Branch-free so every load of the tile can be in flight at once: rows past n read
    // row rows-1 against ws = 0 (adds +0), columns past k re-read column k-1 into
    // accumulators that are never stored.
    const int rlast = ((n - base < kCgsThreads) ? (int)(n - base) : kCgsThreads) - 1;
    const double* xt = X + base;
#pragma unroll
    for (int rr = 0; rr < kCgsThreads / 32; ++rr) {  // rows outer: the column chains interleave
      const int r = lane + 32 * rr;
      const int rc = r < rlast ? r : rlast;
      const double wr = ws[r];
#pragma unroll
      for (int j = 0; j < CPW; ++j) {
        const int c = min(warp + kCgsWarps * j, k - 1);
        acc[j] = acc[j] + xt[(int64_t)c * ld + rc] * wr;
      }
    }
    __syncthreads();
  }
  const int kk = (MODE == kSubNorm) ? 1 : k;
  if (MODE == kSubNorm) {
    double v = nacc;
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) nred[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int q = 0; q < kCgsWarps; ++q) s = s + nred[q];
      partials[blockIdx.x] = s;
    }
  } else {
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      const int c = warp + kCgsWarps * j;
      if (c < k) {  // warp-uniform
        double v = acc[j];
        for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) partials[(int64_t)blockIdx.x * k + c] = v;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int g = (int)gridDim.x;
  for (int c = warp; c < kk; c += kCgsWarps) {  // warp per column, lanes over CTAs
    double v = 0.0;
    for (int b = lane; b < g; b += 32) v = v + __ldcg(partials + (int64_t)b * kk + c);
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[c] = v;
  }
  if (tid == 0) *counter = 0u;
}

// ---------------------------------------------------------------- CG vector updates
// krylov.py:156-158 fused with the residual norm: x += alpha p ; r -= alpha Ap ; out = r.r
// (numpy order: alpha * p first, then the add), deterministic two-level reduction.
__global__ void __launch_bounds__(256)
cg_update_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                 const double* __restrict__ Ap, double alpha, int64_t n, double* __restrict__ partials,
                 double* __restrict__ out, unsigned int* counter) {
  pdl_wait();
  __shared__ double red[8];
  __shared__ bool last;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    double pv[4], av[4], xv[4], rv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = i + u * stride;
      const bool ok = j < n;
      pv[u] = ok ? p[j] : 0.0;
      av[u] = ok ? Ap[j] : 0.0;
      xv[u] = ok ? x[j] : 0.0;
      rv[u] = ok ? r[j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = i + u * stride;
      const double xn = xv[u] + alpha * pv[u];
      const double rn = rv[u] - alpha * av[u];
      if (j < n) {
        x[j] = xn;
        r[j] = rn;
        acc = acc + rn * rn;
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) acc = acc + __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = s + red[w];
    partials[blockIdx.x] = s;
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (warp == 0) {
    double v = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) v = v + __ldcg(partials + b);
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) {
      out[0] = v;
      *counter = 0u;
    }
  }
}

// out = sqrt(in) (the GMRES hnext = ||w||, krylov.py:80, kept on the device for w / hnext)
__global__ void sqrt_kernel(const double* __restrict__ in, double* __restrict__ out) { *out = sqrt(*in); }

// p = z + beta p (krylov.py:163)
__global__ void xpby_kernel(const double* __restrict__ z, double beta, double* __restrict__ p, int64_t n) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// w[i] = w[i] - sum_c X[c*ld + i] * h[c]   (w - V h, numpy order: V@h first; k > 128 passes)
__global__ void gemv_sub_kernel(const double* __restrict__ X, int64_t ld, int k,
                                const double* __restrict__ h, double* __restrict__ w, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int c = 0; c < k; ++c) s = s + X[(int64_t)c * ld + i] * h[c];
  w[i] = w[i] - s;
}

// y[i] = sum_c X[c*ld + i] * h[c]   (V y)
__global__ void gemv_kernel(const double* __restrict__ X, int64_t ld, int k,
                            const double* __restrict__ h, double* __restrict__ y, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int c = 0; c < k; ++c) s = s + X[(int64_t)c * ld + i] * h[c];
  y[i] = s;
}

// y = a - b
__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ y, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] - b[i];
}

// y = y + a
__global__ void add_inplace_kernel(double* __restrict__ y, const double* __restrict__ a, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = y[i] + a[i];
}

// y = x / s (numpy: w / hnext)
__global__ void div_scalar_kernel(const double* __restrict__ x, const double* __restrict__ s,
                                  double* __restrict__ y, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / *s;
}

// row-major (q x r) <- column-major (ld = q) transpose for the Arnoldi basis
__global__ void colmajor_to_rowmajor_kernel(const double* __restrict__ X, int64_t ld, int64_t q, int r,
                                            double* __restrict__ Y) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= q * r) return;
  const int64_t i = idx / r;
  const int c = (int)(idx % r);
  Y[idx] = X[(int64_t)c * ld + i];
}

// ---------------------------------------------------------------- host-side launchers
int launch_correction_core(const pslr_ctx* ctx, cudaStream_t st) {
  launch_pdl(correction_core_kernel, dim3(1), dim3(256), 0, st, ctx->partials, (int)ctx->s, (int)ctx->r, ctx->G, ctx->u);
  return (int)cudaGetLastError();
}

int vt_grid(int64_t q, int sm_count) {
  int64_t g = (q + 8 * 16 - 1) / (8 * 16);
  const int64_t cap = 4 * (int64_t)sm_count;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// s = V^T y over this context's rows (sharded contexts; h lands in ctx->u[r..2r) first)
int launch_vt_local(pslr_ctx* ctx, const double* y, double* s, cudaStream_t st) {
  const int g = vt_grid(ctx->q, ctx->sm_count);
  launch_pdl(vt_dot_kernel, dim3(g), dim3(kVtThreads), 0, st, ctx->V, y, 1, ctx->q, (int)ctx->r, nullptr, ctx->red, ctx->u,
                                          ctx->counter);
  if (cudaGetLastError() != cudaSuccess) return 1;
  return (int)cudaMemcpyAsync(s, ctx->u + ctx->r, ctx->r * sizeof(double), cudaMemcpyDeviceToDevice, st);
}

// s = V^T y for a strided y (rank-local partial sums; no G)
int launch_vt_local_strided(pslr_ctx* ctx, const double* y, int64_t ys, double* s, cudaStream_t st) {
  const int g = vt_grid(ctx->q, ctx->sm_count);
  launch_pdl(vt_dot_kernel, dim3(g), dim3(kVtThreads), 0, st, ctx->V, y, ys, ctx->q, (int)ctx->r, nullptr, ctx->red, ctx->u,
                                          ctx->counter);
  if (cudaGetLastError() != cudaSuccess) return 1;
  return (int)cudaMemcpyAsync(s, ctx->u + ctx->r, ctx->r * sizeof(double), cudaMemcpyDeviceToDevice, st);
}

int launch_gs(pslr_ctx* ctx, const double* s, cudaStream_t st) {
  launch_pdl(gs_kernel, dim3(1), dim3(128), 0, st, ctx->G, s, ctx->u, (int)ctx->r);
  return (int)cudaGetLastError();
}

// u = G V^T y  (writes ctx->u[0..r), h in ctx->u[r..2r))
int launch_vt_dot(pslr_ctx* ctx, const double* y, cudaStream_t st) {
  const int g = vt_grid(ctx->q, ctx->sm_count);
  launch_pdl(vt_dot_kernel, dim3(g), dim3(kVtThreads), 0, st, ctx->V, y, 1, ctx->q, (int)ctx->r, ctx->G, ctx->red,
                                          ctx->u, ctx->counter);
  return (int)cudaGetLastError();
}

// out = y + V u
int launch_vu_add(const pslr_ctx* ctx, const double* y, double* out, cudaStream_t st) {
  int64_t blocks = (ctx->q + 7) / 8;
  const int64_t cap = 8 * (int64_t)ctx->sm_count;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  launch_pdl(vu_add_kernel, dim3((unsigned)blocks), dim3(256), 0, st, ctx->V, ctx->u, y, 1, out, 1, ctx->q, (int)ctx->r);
  return (int)cudaGetLastError();
}

int launch_spmv(const DevCsr& M, const double* x, double* y, cudaStream_t st) {
  if (M.nrows == 0) return 0;
  launch_pdl(spmv_kernel, dim3((M.nrows + 255) / 256), dim3(256), 0, st, M, x, y);
  return (int)cudaGetLastError();
}

int dot_grid(int64_t n, int sm_count) {
  // small k passes have few loads in flight per thread: more CTAs per SM
  int64_t g = (n + kCgsThreads - 1) / kCgsThreads;
  const int64_t cap = 4 * (int64_t)sm_count;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

template <int MODE, int CPW>
static int launch_cgs_w(pslr_ctx* ctx, const double* X, int64_t ld, int k, double* w, int64_t n,
                        const double* h0, double* out, cudaStream_t st) {
  static int resident = 0;  // CTAs per SM at this instance's register count (one full wave)
  if (!resident) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, cgs_pass_kernel<MODE, CPW>, kCgsThreads, 0) !=
            cudaSuccess || b < 1)
      b = 2;
    resident = std::min(b, 4);
  }
  const int g = (int)std::min<int64_t>(dot_grid(n, ctx->sm_count), (int64_t)resident * ctx->sm_count);
  launch_pdl(cgs_pass_kernel<MODE, CPW>, dim3(g), dim3(kCgsThreads), 0, st, X, ld, k, w, n, h0, ctx->red, out, ctx->counter);
  return (int)cudaGetLastError();
}

template <int MODE>
static int launch_cgs(pslr_ctx* ctx, const double* X, int64_t ld, int k, double* w, int64_t n,
                      const double* h0, double* out, cudaStream_t st) {
  if (MODE == kSubNorm || k <= kCgsWarps) return launch_cgs_w<MODE, 1>(ctx, X, ld, k, w, n, h0, out, st);
  if (k <= 2 * kCgsWarps) return launch_cgs_w<MODE, 2>(ctx, X, ld, k, w, n, h0, out, st);
  if (k <= 4 * kCgsWarps) return launch_cgs_w<MODE, 4>(ctx, X, ld, k, w, n, h0, out, st);
  if (k <= 8 * kCgsWarps) return launch_cgs_w<MODE, 8>(ctx, X, ld, k, w, n, h0, out, st);
  return launch_cgs_w<MODE, 16>(ctx, X, ld, k, w, n, h0, out, st);
}

// (bases wider than kCgsMaxCols: the projection as its own pass, dots 128 columns at a time)
static int launch_gemv_sub(const double* X, int64_t ld, int k, const double* h, double* w, int64_t n,
                           cudaStream_t st) {
  if (n == 0) return 0;
  launch_pdl(gemv_sub_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, X, ld, k, h, w, n);
  return (int)cudaGetLastError();
}

int launch_multidot(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* y, int64_t n,
                    double* out, cudaStream_t st) {
  for (int c0 = 0; c0 < k; c0 += kCgsMaxCols) {
    const int e = launch_cgs<kDot>(ctx, X + (int64_t)c0 * ld, ld, std::min(kCgsMaxCols, k - c0),
                                   const_cast<double*>(y), n, nullptr, out + c0, st);
    if (e) return e;
  }
  return 0;
}

int launch_sub_dot(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* h0, double* w,
                   int64_t n, double* out, cudaStream_t st) {
  if (k <= kCgsMaxCols) return launch_cgs<kSubDot>(ctx, X, ld, k, w, n, h0, out, st);
  const int e = launch_gemv_sub(X, ld, k, h0, w, n, st);
  return e ? e : launch_multidot(ctx, X, ld, k, w, n, out, st);
}

int launch_sub_norm(pslr_ctx* ctx, const double* X, int64_t ld, int k, const double* h0, double* w,
                    int64_t n, double* out, cudaStream_t st) {
  if (k <= kCgsMaxCols) return launch_cgs<kSubNorm>(ctx, X, ld, k, w, n, h0, out, st);
  const int e = launch_gemv_sub(X, ld, k, h0, w, n, st);
  return e ? e : launch_multidot(ctx, w, n, 1, w, n, out, st);
}

int launch_cg_update(pslr_ctx* ctx, double* x, double* r, const double* p, const double* Ap, double alpha,
                     int64_t n, double* out, cudaStream_t st) {
  const int g = dot_grid(n, ctx->sm_count);
  launch_pdl(cg_update_kernel, dim3(g), dim3(256), 0, st, x, r, p, Ap, alpha, n, ctx->red, out, ctx->counter);
  return (int)cudaGetLastError();
}

int launch_sqrt(const double* in, double* out, cudaStream_t st) {
  launch_pdl(sqrt_kernel, dim3(1), dim3(1), 0, st, in, out);
  return (int)cudaGetLastError();
}

int launch_xpby(const double* z, double beta, double* p, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  launch_pdl(xpby_kernel, dim3((unsigned)std::min<int64_t>((n + 255) / 256, 4096)), dim3(256), 0, st, z, beta, p, n);
  return (int)cudaGetLastError();
}

int launch_gemv(const double* X, int64_t ld, int k, const double* h, double* y, int64_t n,
                cudaStream_t st) {
  if (n == 0) return 0;
  launch_pdl(gemv_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, X, ld, k, h, y, n);
  return (int)cudaGetLastError();
}

int launch_sub(const double* a, const double* b, double* y, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  launch_pdl(sub_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, a, b, y, n);
  return (int)cudaGetLastError();
}

int launch_add_inplace(double* y, const double* a, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  launch_pdl(add_inplace_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, y, a, n);
  return (int)cudaGetLastError();
}

int launch_div_scalar(const double* x, const double* s, double* y, int64_t n, cudaStream_t st) {
  if (n == 0) return 0;
  launch_pdl(div_scalar_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, x, s, y, n);
  return (int)cudaGetLastError();
}

int launch_transpose_basis(const double* X, int64_t ld, int64_t q, int r, double* Y, cudaStream_t st) {
  if (q * r == 0) return 0;
  launch_pdl(colmajor_to_rowmajor_kernel, dim3((unsigned)((q * r + 255) / 256)), dim3(256), 0, st, X, ld, q, r, Y);
  return (int)cudaGetLastError();
}

}  // namespace pslr
