// pslr_internal.h — shared definitions of libpslr.so (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pslr.h"
#ifdef __CUDACC__
#include <nvtx3/nvToolsExt.h>
#endif

#ifndef __CUDACC__
typedef struct CUevent_st* cudaEvent_t;
typedef struct CUstream_st* cudaStream_t;
#else
#include <cuda_runtime.h>
#endif

namespace pslr {

int fail(int code, const std::string& msg);  // records the thread-local message, returns code

// NVTX range over one C-ABI call (ranges per apply / solve for nsys/ncu
// --nvtx filtering; header-only NVTX3, a no-op without an attached tool)
#ifdef __CUDACC__
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#endif
double numpy_sum(const double* a, int64_t n);

// CSR on the device, int32 row pointers (every matrix here has < 2^31 entries).
struct DevCsr {
  int32_t nrows = 0, ncols = 0, nnz = 0;
  const int32_t* ptr = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
};

// One TMA-streamed chunk of a packed triangular factor (pack.cpp): the two bulk copies
// the producer issues for it, precomputed so the producer loop does no arithmetic.
struct alignas(16) ChunkDesc {
  uint32_t off16;   // byte offset in the factor's data / 16
  uint32_t bytes;   // packed bytes (multiple of 16)
  int32_t rpos;     // first position of the chunk's rhs slice (even: 16-B aligned)
  uint32_t rbytes;  // rhs slice bytes (multiple of 16)
};

// max rows per chunk: bounds the per-stage right-hand-side buffer
#ifndef PSLR_CHUNK_ROWS
#define PSLR_CHUNK_ROWS 1024
#endif
constexpr int kChunkRows = PSLR_CHUNK_ROWS;
// bytes of the step kernel's shared-memory control block (mbarriers, descriptor queue)
constexpr int kCtlBytes = 1024;

// Segment layout inside a chunk (all parts 16-byte aligned; pack.cpp emit_factor):
//   int32 hdr[12] = {nrows | w << 16, flags | tb << 8, pos0, bytes, S, far_off,
//                    rbase (first segment of a chunk), 0, 0, 0, 0, 0}
//                    flags: bit0 ends a level, bit1 has far deps, bit2 explicit sd/rcp,
//                    bit3 last segment of its chunk; tb = first consumer thread
//                    (the first 16 bytes are all a consumer warp needs to follow the stream)
//   S = nrows rounded up to 4; G = max(1, ceil(w/4)) groups of 4 entries (no-op padding)
//   int32 info[S]   L: U-position of the row ; U: row id | bit 31: sd = 1 - 2^-53
//                   | bit 30: the row is a far dependency (its value also goes to global z)
//   U only: double invd[S] [, sd[S], rcp[S] if flags bit2]
//   uint16 slot[G][S][4]    near: ring slot (<= W, W = zero slot) ; far: 0x8000 | far index
//   double val[G][2][S][2]  (U values pre-scaled by 1/diag of their column)
//   int32 far[a4(nfar)]     U-positions of the far dependencies
struct DevTri {
  int32_t nblocks = 0, nchunks = 0;
  const uint8_t* data = nullptr;
  const ChunkDesc* chunks = nullptr;
  const int32_t* blk_chunk = nullptr;  // nblocks+1
  const int32_t* lpos = nullptr;       // L only: row -> global L-position (rhs placement)
  const int32_t* lrow = nullptr;       // L only: global L-position -> row
};

// host-side analysis + packed output (pack.cpp)
struct TriAnalysis {
  bool upper = false;
  std::vector<int32_t> pos_of_row, row_at_pos, level_end, level_of_row, len;
  std::vector<int32_t> blk_depth;  // dependency levels of each block
  std::vector<double> diag;
  int64_t depth_max = 0, levels = 0, reach = 0;
};

struct TriHost {
  std::vector<uint8_t> data;
  std::vector<ChunkDesc> chunks;
  std::vector<int32_t> blk_chunk;
  int64_t far = 0, nnz_offdiag = 0, segments = 0;
  int64_t far_slots = 0;  // far-ring slots used (shared memory beside the ring)
};

int analyze_factor(const pslr_csr& M, const std::vector<int64_t>& off, bool upper, TriAnalysis& A,
                   const char* name, int64_t sched_cap = 0, int64_t sched_delay = 0);
// Level-merged factors (pack.cpp merge_levels): an owned host CSR and the right-hand-side
// transform of the merged rows, one record per row: rows[4] = {i, j0, j1, j2} (padding
// j = i), c[4] = {c0, c1, c2, 0};  rhs'_i = rhs_i - (c0 rhs_j0 + c1 rhs_j1 + c2 rhs_j2).
constexpr int kXfWidth = 3;   // substituted dependencies per row
constexpr int kXfWidth1 = 4;  // ints per record
struct HostCsr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
  std::vector<double> data;
  pslr_csr view() const { return pslr_csr{nrows, ncols, nnz, indptr.data(), indices.data(), data.data()}; }
};
struct MergeXf {
  std::vector<int32_t> rows;  // 4 per record, row space
  std::vector<double> c;      // 4 per record
  std::vector<int32_t> blk;   // nblocks + 1 record offsets
};
int merge_levels(const pslr_csr& M, const std::vector<int64_t>& off, bool upper, int64_t wmax, HostCsr& out,
                 MergeXf& X, const char* name);

// The transform on the device, in the position space of the array it rewrites in place
// (L: the L-position-ordered rhs, U: the U-position-ordered L output): idx = {pos_i,
// pos_j0, pos_j1, pos_j2}, val = {c0, c1}, {c2, 0}; blk: records of block b are
// [blk[b], blk[b+1]).  nrec == 0: the factor is not merged.
struct DevXform {
  int32_t nrec = 0;
  const int32_t* idx = nullptr;  // 4 per record (read as int4)
  const double* val = nullptr;   // 4 per record (read as two double2)
  const int32_t* blk = nullptr;
};

// consumer threads per CTA of the fused step kernel = max rows per packed segment
// (PSLR_STEP_THREADS: timing-experiment builds under lib_variants/ only)
#ifndef PSLR_STEP_THREADS
#define PSLR_STEP_THREADS 480
#endif
constexpr int kStepThreads = PSLR_STEP_THREADS;
// consumer threads of the step kernel's second instantiation (systems of narrow levels)
constexpr int kNarrowThreads = kStepThreads < 128 ? kStepThreads : 128;
// consumer threads of the two-vector launches of a wide system: a row's two interleaved
// chains need ~167 registers per thread; under the 512-thread launch bound the compiler
// caps them at 128 and spills, under 352 + 32 threads it does not, and the two-vector sweep
// gains 6 % (cfg5: 0.315 -> 0.295 ms per apply; 224-352 consumer threads measure alike).
// The one-vector kernel fits 128 registers and keeps 480 threads (1.63 vs 1.67 ms at 352).
constexpr int kWide2Threads = kStepThreads < 352 ? kStepThreads : 352;

int emit_factor(const pslr_csr& M, const std::vector<int64_t>& off, const TriAnalysis& A, int64_t W,
                int64_t stage_bytes, int64_t seg_rows, const std::vector<int32_t>& far_index,
                const std::vector<int32_t>& info_of_row, int64_t far_slots_max, int64_t rhs_row_bytes,
                TriHost& out, const char* name, bool alt_groups = false);

// Terms of the per-subdomain fused step (see kernels.cu: subdomain_step_kernel).
enum BTerm : int { BT_NONE = 0, BT_F = 1, BT_EY = 2 };
enum ITerm : int { IT_NONE = 0, IT_G = 1, IT_FX = 2, IT_CY = 3, IT_CGY = 4, IT_VU = 5, IT_PRE = 6 };

struct StepArgs {
  // ---- interior (B) phase:  rhs = b1 [(-) b2];  xb = B^{-1} rhs
  int b1 = BT_NONE, b2 = BT_NONE;
  const double* f = nullptr;   // p-vector used by BT_F
  double* fL = nullptr;        // f already in L-position order (permute_f): the L phase reads
                               // it as its right-hand side; E y rows are folded into it
  const double* yE = nullptr;  // q-vector multiplied by E for BT_EY
  double* xb = nullptr;        // p output of the B solve
  // ---- interface phase:  w = i1 (+|-) i2 ;  [y = C0^{-1} w] ; [y += cadd]
  int i1 = IT_NONE, i2 = IT_NONE;
  int i2_sub = 1;              // 1: w = i1 - i2 ; 0: w = i1 + i2
  const double* g = nullptr;   // q-vector for IT_G
  const double* yC = nullptr;  // q-vector for IT_CY / IT_CGY
  const double* u = nullptr;   // r-vector for IT_VU
  const double* pre = nullptr; // q-vector for IT_PRE (C_g y by the all-SM pre-kernel)
  int do_c0 = 0;
  const double* cadd = nullptr;
  double* yout = nullptr;      // q output
  double* partials = nullptr;  // [s][r] V^T yout partial sums (nullable)
  int tag = 0;                 // launch kind, for pslr_apply_profiled
  int ifc_done = 0;            // set by launch_step: the interface phase's result (rhsC) was
                               // written by the all-SM iface_kernel (split launch)
  int ey_done = 0;             // set by launch_step: the E y rows of the L right-hand side were
                               // written by the all-SM ey_rhs_kernel (no in-kernel prepass)
  int xpos = 0;                // set by launch_step: xb in U-position order (F read via Fpos)
};

// Everything the fused kernel reads besides StepArgs (constant per context).
struct StepConst {
  DevTri LB, UB, LC, UC;
  DevXform XLB, XUB, XLC, XUC;  // level-merged factors: their in-place rhs transforms
  const int32_t* lrowx = nullptr;   // merged L_B: L-position -> row, or -(record + 1) for a
  const int32_t* xlb_rows = nullptr;  //   merged row whose f gets the transform (permute_f):
                                    //   {row_i, row_j0, row_j1, row_j2} of the record
  DevCsr E, F, C, Cg;
  DevCsr Fpos;  // F with its columns mapped to the interior rows' U-positions
  const int32_t* int_off = nullptr;
  const int32_t* ifc_off = nullptr;
  const int32_t* erows = nullptr;     // int4 per interior row with E entries, grouped by block:
                                      // {L-position, row, E.ptr[row], E.ptr[row+1]}
  const int32_t* erow_off = nullptr;  // s+1
  int nerows = 0;                     // erow_off[s]
  const double* V = nullptr;
  int r = 0;
  double* rhsB = nullptr;  // p: L_B right-hand side in L-position order
  double* rhsE = nullptr;  // p: right-hand side E y alone: only the E rows are ever written,
                           //    every other position stays 0 from the allocation
  double* zB = nullptr;    // p: L_B output / U_B intermediate in U-position order
  double* rhsC = nullptr;  // q
  double* zC = nullptr;    // q
  double* cgy = nullptr;   // q: C_g y of the step, by the all-SM pre-kernel (launch_step)
  int ring_mask = 0;       // W - 1
  int far_slots = 0;       // far-ring slots after the ring's zero slot (ring index W + 1 + slot)
  int nst = 0;             // pipeline stages
  int stage_bytes = 0;
  int rhs_stride = 0;      // doubles per stage right-hand-side buffer
  int smem_bytes = 0;
  long long* trace = nullptr;  // PSLR_TRACE: [count, pad, (code, ns)...] of CTA 0
  long long trace_cap = 0;
  int trace_block = 0;       // the CTA whose timeline trace builds record (PSLR_TRACE_CTA)
  int dbg = 0;               // PSLR_DBG timing experiments (wrong results): bit0 skip rows,
                             // bit1 skip next-row loads, bit3 no producer back-off
  long long l2ahead = 0;     // bytes of the factor stream prefetched into L2 ahead (0: default)
  int nthr = kStepThreads;  // consumer threads per step CTA (the packing's segment rows)
  const int8_t* l2keep = nullptr;  // per block: 1 = its factor chunks are copied with an L2
                                   // evict_last policy (the deepest blocks, whose streams
                                   // bound every step, stay L2-resident across the steps)
};

}  // namespace pslr

// The context behind the opaque C handle.
struct pslr_ctx {
  int device = 0;
  int64_t n = 0, p = 0, q = 0, s = 0, r = 0;
  int64_t nghost = 0;  // sharded contexts: ghost interface columns of C, Cg and A
  bool pdl = true;     // programmatic dependent launch of the step kernel (PSLR_PDL=0: off)
  bool ey_all_sm = true;  // E y rows of the L right-hand side by the all-SM kernel (PSLR_EY_ALLSM=0: prepass)
  bool split_iface = true;  // interface phase by the all-SM iface_kernel between a B-phase and a
                            // C0-phase launch (PSLR_SPLIT_IFACE=0: inside the step kernel)
  const pslr_ctx* parent = nullptr;  // clones: the context whose read-only data they share
  // shared by a context and its clones: use_count() - 1 = live clones of the parent
  std::shared_ptr<int> family = std::make_shared<int>(0);
  int smem_optin = 0;
  // two right-hand sides per launch (pslr_apply_multi): step constants with the doubled
  // ring / rhs slices and interleaved ([row][2]) scratch, set up on first use
  bool nv2_ready = false;
  pslr::StepConst K2;
  pslr::DevTri tri2[4];  // the factor streams packed at the two-vector chunk size (LB, UB, LC, UC)
  int64_t sb2 = 0;       // that chunk size
  int64_t far2 = 0;      // far-ring slots of the two-vector packing
  double *fL2 = nullptr, *g2 = nullptr, *xb2 = nullptr, *y0_2 = nullptr, *y1_2 = nullptr;
  double *c2 = nullptr, *yA2 = nullptr, *yB2 = nullptr, *yF2 = nullptr, *xF2 = nullptr;
  double *io_b2 = nullptr, *io_z2 = nullptr;  // host-buffer two-vector apply staging
  int sm_count = 0;
  std::vector<int64_t> interior_off, interface_off;
  // device-resident state
  pslr::StepConst K;
  pslr::DevCsr A, C0;
  double* V = nullptr;           // q x r row-major
  double* G = nullptr;           // r x r row-major
  // scratch
  double* xb = nullptr;          // p
  double* fL = nullptr;          // p+2: f in L-position order, per apply
  double* y0 = nullptr;          // q
  double* y1 = nullptr;          // q
  double* y2 = nullptr;          // q
  double* c = nullptr;           // q
  double* partials = nullptr;    // s x r
  double* u = nullptr;           // 2r
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
  double *gr = nullptr, *gw = nullptr, *gt = nullptr;  // Krylov vectors of a generic operator
  int64_t g_len = 0, gw_len = 0, gt_len = 0;            //   longer than n (pslr_*_op)
  double* io_b = nullptr;        // n device staging for host apply
  double* io_z = nullptr;        // n
  // multi-GPU (comm.cu): NCCL communicator and halo plan of a rank-local context
  void* comm = nullptr;          // ncclComm_t
  int world = 1, rank = 0;
  std::vector<int64_t> halo_send_cnt, halo_send_off, halo_recv_cnt, halo_recv_off;  // per peer rank
  int32_t* halo_idx = nullptr;   // local interface indices to send, peers in rank order
  double* halo_buf = nullptr;    // their gathered values
  int64_t halo_nsend = 0;
  // halo overlapped with the interior phase (comm.cu comm_halo_async; PSLR_HALO_OVERLAP=0: off):
  // the exchange runs on comm_stream after ev_y (the sent vector is final on the caller's
  // stream) and records ev_halo; the next launch_step runs its E y rows and B phases first and
  // waits for pending_halo only before the C_g y term of its interface phase
  bool halo_overlap = true;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_y = nullptr, ev_halo = nullptr;
  mutable cudaEvent_t pending_halo = nullptr;
  double *sh_a = nullptr, *sh_b = nullptr, *sh_c = nullptr, *sh_s = nullptr, *sh_x = nullptr;
  int64_t sh_a_len = 0, sh_b_len = 0, sh_c_len = 0, sh_s_len = 0, sh_x_len = 0;
  double *sh2_y0 = nullptr, *sh2_a = nullptr, *sh2_b = nullptr, *sh2_c = nullptr, *halo_buf2 = nullptr;
  int64_t sh2_y0_len = 0, sh2_a_len = 0, sh2_b_len = 0, sh2_c_len = 0, halo_buf2_len = 0;
  double* hpin = nullptr;        // pinned host: the GMRES coefficients of two iterations
  int64_t hpin_len = 0;
  cudaEvent_t kev[2] = {nullptr, nullptr};  // their device-to-host copies landed
  std::vector<void*> allocations;
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_events;
  std::vector<int32_t> prof_kinds;
  int64_t device_bytes = 0;
  pslr_ctx_info_t info{};
};
