// pslr_internal.h — shared definitions of libpslr.so (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/pslr.h"

#ifndef __CUDACC__
typedef struct CUevent_st* cudaEvent_t;
#else
#include <cuda_runtime.h>
#endif

namespace pslr {

int fail(int code, const std::string& msg);  // records the thread-local message, returns code
double numpy_sum(const double* a, int64_t n);

#ifdef __CUDACC__
#define PSLR_HD __host__ __device__
#else
#define PSLR_HD
#endif

// CSR on the device, int32 row pointers (every matrix here has < 2^31 entries).
struct DevCsr {
  int32_t nrows = 0, ncols = 0, nnz = 0;
  const int32_t* ptr = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
};

// A block-diagonal triangular factor, level-scheduled per block and packed in
// level order ("position" = index in that order).  Off-diagonal entries only;
// for U the values are pre-scaled by 1/diag of their column, exactly as scipy's
// spsolve_triangular does before calling SuperLU (so the device solve reproduces
// the reference bit for bit):  z_i = (b_i / sd_i) - sum_j U'_ij z_j ,  x_i = z_i * invd_i.
struct DevTri {
  int32_t nblocks = 0;
  int32_t nlevels = 0, npos = 0, nnz = 0;
  const int32_t* blk_lvl = nullptr;  // nblocks+1: level range of each block
  const int32_t* lvl_pos = nullptr;  // nlevels+1: position range of each level
  const int32_t* pos_row = nullptr;  // npos: absolute row (index into the p- or q-vector)
  const int32_t* pos_ent = nullptr;  // npos+1: entry range of each position
  const int32_t* col = nullptr;      // nnz: absolute column
  const double* val = nullptr;       // nnz
  const double* sd = nullptr;        // U only, per position: U_ii * (1/U_ii)
  const double* invd = nullptr;      // U only, per position: 1/U_ii
};

// Terms of the per-subdomain fused step (see kernels.cu: subdomain_step_kernel).
enum BTerm : int { BT_NONE = 0, BT_F = 1, BT_EY = 2 };
enum ITerm : int { IT_NONE = 0, IT_G = 1, IT_FX = 2, IT_CY = 3, IT_CGY = 4, IT_VU = 5 };

struct StepArgs {
  // ---- interior (B) phase:  rhs = b1 [(-) b2];  xb = B^{-1} rhs
  int b1 = BT_NONE, b2 = BT_NONE;
  const double* f = nullptr;   // p-vector used by BT_F
  const double* yE = nullptr;  // q-vector multiplied by E for BT_EY
  double* tb = nullptr;        // p scratch (L output / scaled U intermediate)
  double* xb = nullptr;        // p output of the B solve
  // ---- interface phase:  w = i1 (+|-) i2 ;  [y = C0^{-1} w] ; [y += cadd]
  int i1 = IT_NONE, i2 = IT_NONE;
  int i2_sub = 1;              // 1: w = i1 - i2 ; 0: w = i1 + i2
  const double* g = nullptr;   // q-vector for IT_G
  const double* yC = nullptr;  // q-vector for IT_CY / IT_CGY
  const double* u = nullptr;   // r-vector for IT_VU
  int do_c0 = 0;
  double* tw = nullptr;        // q scratch for the C0 solve
  const double* cadd = nullptr;
  double* yout = nullptr;      // q output
  double* partials = nullptr;  // [s][r] V^T yout partial sums (nullable)
  int tag = 0;                 // launch kind, for pslr_apply_profiled
};

}  // namespace pslr

// The context behind the opaque C handle.
struct pslr_ctx {
  int device = 0;
  int64_t n = 0, p = 0, q = 0, s = 0, r = 0;
  int sm_count = 0;
  std::vector<int64_t> interior_off, interface_off;
  // device-resident state
  pslr::DevTri LB, UB, LC, UC;
  pslr::DevCsr E, F, C, C0, Cg, A;
  int32_t* d_int_off = nullptr;  // s+1
  int32_t* d_ifc_off = nullptr;  // s+1
  double* V = nullptr;           // q x r row-major
  double* G = nullptr;           // r x r row-major
  // scratch
  double* tb = nullptr;          // p
  double* xb = nullptr;          // p
  double* tw = nullptr;          // q
  double* y0 = nullptr;          // q
  double* y1 = nullptr;          // q
  double* y2 = nullptr;          // q
  double* c = nullptr;           // q
  double* partials = nullptr;    // s x r
  double* u = nullptr;           // r
  double* red = nullptr;         // reduction scratch (multi-dot partials)
  int64_t red_len = 0;
  unsigned int* counter = nullptr;  // last-block reduction ticket
  double* h_dev = nullptr;       // small vector results (dots)
  int64_t h_len = 0;
  // krylov work
  double* kv = nullptr;          // Krylov basis
  int64_t kv_len = 0;
  double* kz = nullptr;          // FGMRES Z basis
  int64_t kz_len = 0;
  double* kw = nullptr;          // n
  double* kt = nullptr;          // n
  double* kr = nullptr;          // n
  double* pinned = nullptr;      // host staging
  int64_t pinned_len = 0;
  double* io_b = nullptr;        // n device staging for host apply
  double* io_z = nullptr;        // n
  std::vector<void*> allocations;
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_events;
  std::vector<int32_t> prof_kinds;
  int64_t device_bytes = 0;
  pslr_ctx_info_t info{};
};
