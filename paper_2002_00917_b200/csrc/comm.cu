// comm.cu — the multi-GPU part of the C-ABI (SURVEY §8b `pslr_comm_init`, §8e): an NCCL
// communicator and a halo plan held by a rank-local (sharded) context, so that the same
// pslr_apply / pslr_apply_Err / pslr_arnoldi / pslr_gmres calls run the coupled N-GPU
// problem from inside libpslr (one process per GPU, any host language).
//
// Per apply: one allreduce of the r partial V^T y sums and m halo exchanges of the
// interface ghosts C_g reads (batched ncclSend/ncclRecv, stream-ordered); per Krylov
// iteration one more halo for the A-SpMV and one allreduce per CGS2 pass.  The plan is
// the one shard.py derives from the replicated global system (plan_shard): per peer, the
// local interface indices this rank sends (peer order = ascending rank) and the number of
// ghosts it receives (stored after the q local interface rows, in ascending peer rank).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch process that is
// the NCCL torch already loaded, elsewhere the system's.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pslr_ops.h"

namespace pslr {

namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.getUniqueId, "ncclGetUniqueId");
    sym(api.commInitRank, "ncclCommInitRank");
    sym(api.commDestroy, "ncclCommDestroy");
    sym(api.allReduce, "ncclAllReduce");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.groupStart, "ncclGroupStart");
    sym(api.groupEnd, "ncclGroupEnd");
    sym(api.errorString, "ncclGetErrorString");
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PSLR_OK;
  const char* msg = nccl().errorString ? nccl().errorString(r) : "?";
  return fail(PSLR_ENCCL, std::string(what) + ": " + msg);
}

int nccl_ready() {
  const NcclApi& A = nccl();
  if (!A.error.empty()) return fail(PSLR_ENCCL, A.error);
  return PSLR_OK;
}
}  // namespace

#define NCK(call, what) RET(nccl_check((call), what))

__global__ void halo_gather_kernel(const double* __restrict__ v, const int32_t* __restrict__ idx,
                                   double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v[idx[i]];
}
// two interleaved right-hand sides ([i][2]): one 16-byte pair per sent index
__global__ void halo_gather2_kernel(const double2* __restrict__ v, const int32_t* __restrict__ idx,
                                    double2* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v[idx[i]];
}

bool sharded_comm(const pslr_ctx* ctx) { return ctx->comm != nullptr; }

int comm_allreduce(pslr_ctx* ctx, double* x, int64_t n, cudaStream_t st) {
  if (!ctx->comm || n == 0) return PSLR_OK;  // (a one-rank communicator still runs NCCL)
  NCK(nccl().allReduce(x, x, (size_t)n, ncclDouble, ncclSum, static_cast<ncclComm_t>(ctx->comm), st),
      "ncclAllReduce");
  return PSLR_OK;
}

// v_ext = [q local interface values | nghost ghosts]: fill the ghosts from their owners
int comm_halo(pslr_ctx* ctx, double* v_ext, cudaStream_t st) {
  if (!ctx->comm) return PSLR_OK;
  const int64_t ns = ctx->halo_nsend;
  if (ns > 0) {
    const int64_t blocks = std::min<int64_t>((ns + 255) / 256, 4 * (int64_t)ctx->sm_count);
    halo_gather_kernel<<<(unsigned)blocks, 256, 0, st>>>(v_ext, ctx->halo_idx, ctx->halo_buf, ns);
    CK(cudaGetLastError());
  }
  auto comm = static_cast<ncclComm_t>(ctx->comm);
  NCK(nccl().groupStart(), "ncclGroupStart");
  for (int r = 0; r < ctx->world; ++r) {
    if (ctx->halo_send_cnt[r])
      NCK(nccl().send(ctx->halo_buf + ctx->halo_send_off[r], (size_t)ctx->halo_send_cnt[r], ncclDouble, r, comm, st),
          "ncclSend");
    if (ctx->halo_recv_cnt[r])
      NCK(nccl().recv(v_ext + ctx->q + ctx->halo_recv_off[r], (size_t)ctx->halo_recv_cnt[r], ncclDouble, r, comm,
                      st),
          "ncclRecv");
  }
  NCK(nccl().groupEnd(), "ncclGroupEnd");
  return PSLR_OK;
}

// the same exchange for an interleaved two-vector interface array v2 ([i][2]): ghosts after
// the 2q local values, every count doubled
int comm_halo2(pslr_ctx* ctx, double* v2_ext, cudaStream_t st) {
  if (!ctx->comm) return PSLR_OK;
  const int64_t ns = ctx->halo_nsend;
  if (ns > 0) {
    RET(ensure(ctx, &ctx->halo_buf2, &ctx->halo_buf2_len, 2 * ns));
    const int64_t blocks = std::min<int64_t>((ns + 255) / 256, 4 * (int64_t)ctx->sm_count);
    halo_gather2_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(v2_ext), ctx->halo_idx,
                                                         reinterpret_cast<double2*>(ctx->halo_buf2), ns);
    CK(cudaGetLastError());
  }
  auto comm = static_cast<ncclComm_t>(ctx->comm);
  NCK(nccl().groupStart(), "ncclGroupStart");
  for (int r = 0; r < ctx->world; ++r) {
    if (ctx->halo_send_cnt[r])
      NCK(nccl().send(ctx->halo_buf2 + 2 * ctx->halo_send_off[r], (size_t)(2 * ctx->halo_send_cnt[r]), ncclDouble,
                      r, comm, st),
          "ncclSend");
    if (ctx->halo_recv_cnt[r])
      NCK(nccl().recv(v2_ext + 2 * (ctx->q + ctx->halo_recv_off[r]), (size_t)(2 * ctx->halo_recv_cnt[r]),
                      ncclDouble, r, comm, st),
          "ncclRecv");
  }
  NCK(nccl().groupEnd(), "ncclGroupEnd");
  return PSLR_OK;
}

// The halo of v_ext (nv = 1) or of an interleaved pair (nv = 2) overlapped with the next
// step's interior phase: the exchange is ordered after the caller's stream (ev_y: v is
// final), runs on the context's communication stream and leaves ev_halo in
// ctx->pending_halo; launch_step (step_kernel.cu) makes the caller's stream wait for it only
// before the C_g y term, the one reader of ghost columns (E y and the B solves of the step
// run meanwhile).  PSLR_HALO_OVERLAP=0, or a context without a communicator: the plain
// stream-ordered exchange.
int comm_halo_async(pslr_ctx* ctx, double* v_ext, int nv, cudaStream_t st) {
  if (!ctx->comm) return PSLR_OK;
  if (!ctx->halo_overlap || !ctx->comm_stream) return nv == 2 ? comm_halo2(ctx, v_ext, st) : comm_halo(ctx, v_ext, st);
  CK(cudaEventRecord(ctx->ev_y, st));
  CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_y, 0));
  RET(nv == 2 ? comm_halo2(ctx, v_ext, ctx->comm_stream) : comm_halo(ctx, v_ext, ctx->comm_stream));
  CK(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
  ctx->pending_halo = ctx->ev_halo;
  return PSLR_OK;
}

// a pending halo nobody consumed (no launch_step followed): order the stream after it
int comm_halo_join(pslr_ctx* ctx, cudaStream_t st) {
  if (ctx->pending_halo) {
    CK(cudaStreamWaitEvent(st, ctx->pending_halo, 0));
    ctx->pending_halo = nullptr;
  }
  return PSLR_OK;
}

int comm_destroy(pslr_ctx* ctx) {
  if (ctx->comm && nccl().commDestroy) nccl().commDestroy(static_cast<ncclComm_t>(ctx->comm));
  ctx->comm = nullptr;
  ctx->pending_halo = nullptr;
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev_y) cudaEventDestroy(ctx->ev_y);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  ctx->comm_stream = nullptr;
  ctx->ev_y = ctx->ev_halo = nullptr;
  return PSLR_OK;
}

// interface vectors with room for the ghosts
static int ifc_scratch(pslr_ctx* ctx, double** p, int64_t* len) {
  return ensure(ctx, p, len, ctx->q + ctx->nghost + 2);
}

// The sharded apply (preconditioner.py:79-93 on the rank's rows): shard.py's
// ShardedPreconditioner.apply through the split entry points, collectives inside.
int op_apply_sharded(pslr_ctx* ctx, int64_t m, const double* b, double* z, cudaStream_t st) {
  void* sv = static_cast<void*>(st);
  const int64_t q = ctx->q;
  if (q == 0 && ctx->world == 1) return op_solve_B(ctx, b, z, st);
  RET(ifc_scratch(ctx, &ctx->sh_c, &ctx->sh_c_len));
  RET(ifc_scratch(ctx, &ctx->sh_a, &ctx->sh_a_len));
  RET(ifc_scratch(ctx, &ctx->sh_b, &ctx->sh_b_len));
  RET(ensure(ctx, &ctx->sh_s, &ctx->sh_s_len, std::max<int64_t>(ctx->r, 1) + 2));
  CK(cudaMemsetAsync(ctx->sh_s, 0, (std::max<int64_t>(ctx->r, 1) + 2) * sizeof(double), st));
  // y0 = g - F B^{-1} f and the local V^T y0 partial sums, summed over the ranks
  RET(pslr_apply_first(ctx, b, ctx->y0, ctx->sh_s, sv));
  if (ctx->r > 0) RET(comm_allreduce(ctx, ctx->sh_s, ctx->r, st));
  CK(cudaMemsetAsync(ctx->sh_c, 0, (q + ctx->nghost) * sizeof(double), st));
  RET(pslr_apply_mid(ctx, ctx->y0, ctx->sh_s, ctx->sh_c, sv));  // c = C0^{-1}(y0 + V G s)
  const double* y = ctx->sh_c;
  if (m > 0) {
    // each halo overlaps the E y rows and the B solves of the step that consumes it
    RET(comm_halo_async(ctx, ctx->sh_c, 1, st));
    double* outs[2] = {ctx->sh_a, ctx->sh_b};
    for (int64_t k = 0; k < m; ++k) {
      double* out = outs[k & 1];
      RET(pslr_apply_horner(ctx, y, ctx->sh_c, out, sv));
      if (k < m - 1) RET(comm_halo_async(ctx, out, 1, st));
      y = out;
    }
    RET(comm_halo_join(ctx, st));  // (q == 0 ranks launch no step)
  }
  return pslr_apply_last(ctx, b, y, z, sv);
}

// Two right-hand sides (b2, z2: two vector-major local n-vectors) through one launch
// sequence and one set of collectives: the split two-vector entry points (each vector's
// arithmetic is the single-vector one bit for bit), halos of interleaved pairs, one
// allreduce of 2r.  Ranks without interior or interface rows run the vectors one by one
// between the SAME collectives (shard.py ShardedPreconditioner.apply2's contract).
int op_apply2_sharded(pslr_ctx* ctx, int64_t m, const double* b2, double* z2, cudaStream_t st) {
  void* sv = static_cast<void*>(st);
  const int64_t n = ctx->n, q = ctx->q, ng = ctx->nghost, r = ctx->r;
  if (ctx->p == 0 || q == 0) {  // no two-vector kernels here: per vector, same collectives
    for (int v = 0; v < 2; ++v) RET(op_apply_sharded(ctx, m, b2 + v * n, z2 + v * n, st));
    return PSLR_OK;
  }
  RET(ensure(ctx, &ctx->sh2_y0, &ctx->sh2_y0_len, 2 * q + 2));
  RET(ensure(ctx, &ctx->sh2_c, &ctx->sh2_c_len, 2 * (q + ng) + 2));
  RET(ensure(ctx, &ctx->sh2_a, &ctx->sh2_a_len, 2 * (q + ng) + 2));
  RET(ensure(ctx, &ctx->sh2_b, &ctx->sh2_b_len, 2 * (q + ng) + 2));
  RET(ensure(ctx, &ctx->sh_s, &ctx->sh_s_len, 2 * std::max<int64_t>(r, 1) + 2));
  CK(cudaMemsetAsync(ctx->sh_s, 0, (2 * std::max<int64_t>(r, 1) + 2) * sizeof(double), st));
  RET(pslr_apply2_first(ctx, b2, ctx->sh2_y0, ctx->sh_s, sv));
  if (r > 0) RET(comm_allreduce(ctx, ctx->sh_s, 2 * r, st));
  CK(cudaMemsetAsync(ctx->sh2_c, 0, 2 * (q + ng) * sizeof(double), st));
  RET(pslr_apply2_mid(ctx, ctx->sh2_y0, ctx->sh_s, ctx->sh2_c, sv));
  const double* y = ctx->sh2_c;
  if (m > 0) {
    RET(comm_halo_async(ctx, ctx->sh2_c, 2, st));
    double* outs[2] = {ctx->sh2_a, ctx->sh2_b};
    for (int64_t k = 0; k < m; ++k) {
      double* out = outs[k & 1];
      RET(pslr_apply2_horner(ctx, y, ctx->sh2_c, out, sv));
      if (k < m - 1) RET(comm_halo_async(ctx, out, 2, st));
      y = out;
    }
    RET(comm_halo_join(ctx, st));
  }
  return pslr_apply2_last(ctx, b2, y, z2, sv);
}

// E_rr(m) v on the rank's rows (schur.py:104-112; shard.py sharded_arnoldi's operator)
int op_apply_err_sharded(pslr_ctx* ctx, int64_t m, const double* v, double* out, cudaStream_t st) {
  void* sv = static_cast<void*>(st);
  const int64_t q = ctx->q;
  RET(ifc_scratch(ctx, &ctx->sh_a, &ctx->sh_a_len));
  RET(ifc_scratch(ctx, &ctx->sh_b, &ctx->sh_b_len));
  CK(cudaMemsetAsync(ctx->sh_a, 0, (q + ctx->nghost) * sizeof(double), st));
  CK(cudaMemsetAsync(ctx->sh_b, 0, (q + ctx->nghost) * sizeof(double), st));
  RET(pslr_solve_C0(ctx, v, ctx->sh_a, sv));
  double* src = ctx->sh_a;
  double* dst = ctx->sh_b;
  for (int64_t k = 1; k <= m + 1; ++k) {
    RET(comm_halo_async(ctx, src, 1, st));
    RET(pslr_apply_es_step(ctx, src, dst, k != m + 1 ? 1 : 0, sv));
    RET(comm_halo_join(ctx, st));
    std::swap(src, dst);
  }
  if (q) CK(cudaMemcpyAsync(out, src, q * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return PSLR_OK;
}

// w = A x on the rank's rows: x's interface part refreshed with the owners' ghosts first
int op_spmv_A_sharded(pslr_ctx* ctx, const double* x, double* w, cudaStream_t st) {
  const int64_t n = ctx->n, p = ctx->p;
  if (!ctx->comm) {
    CKL(launch_spmv(ctx->A, x, w, st));
    return PSLR_OK;
  }
  RET(ensure(ctx, &ctx->sh_x, &ctx->sh_x_len, n + ctx->nghost + 2));
  CK(cudaMemcpyAsync(ctx->sh_x, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  RET(comm_halo(ctx, ctx->sh_x + p, st));
  CKL(launch_spmv(ctx->A, ctx->sh_x, w, st));
  return PSLR_OK;
}

}  // namespace pslr

using namespace pslr;

extern "C" {

int pslr_comm_unique_id(void* out) {
  RET(nccl_ready());
  NCK(nccl().getUniqueId(static_cast<ncclUniqueId*>(out)), "ncclGetUniqueId");
  return PSLR_OK;
}

int pslr_comm_init(pslr_ctx* ctx, const void* nccl_unique_id, int nranks, int rank) {
  if (!ctx) return fail(PSLR_EINVAL, "null context");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PSLR_EINVAL, "bad rank / nranks");
  // a clone may own a communicator of its own: an independent pipeline of the same
  // sharded problem (its collectives are ordered on its communicator alone)
  RET(nccl_ready());
  RET(set_device(ctx));
  RET(comm_destroy(ctx));
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  NCK(nccl().commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  ctx->comm = comm;
  ctx->world = nranks;
  ctx->rank = rank;
  const char* ov = std::getenv("PSLR_HALO_OVERLAP");
  ctx->halo_overlap = !(ov && ov[0] == '0');
  if (ctx->halo_overlap) {
    CK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_y, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
  }
  ctx->halo_send_cnt.assign(nranks, 0);
  ctx->halo_send_off.assign(nranks, 0);
  ctx->halo_recv_cnt.assign(nranks, 0);
  ctx->halo_recv_off.assign(nranks, 0);
  return PSLR_OK;
}

int pslr_ctx_set_halo(pslr_ctx* ctx, int world, const int64_t* send_counts, const int32_t* send_idx,
                      const int64_t* recv_counts) {
  if (!ctx) return fail(PSLR_EINVAL, "null context");
  if (!ctx->comm) return fail(PSLR_EINVAL, "pslr_comm_init first");
  if (world != ctx->world) return fail(PSLR_EDIM, "halo plan size differs from the communicator's");
  RET(set_device(ctx));
  int64_t ns = 0, nr = 0;
  for (int r = 0; r < world; ++r) {
    if (send_counts[r] < 0 || recv_counts[r] < 0) return fail(PSLR_EDIM, "negative halo count");
    if (r == ctx->rank && (send_counts[r] || recv_counts[r])) return fail(PSLR_EDIM, "halo with oneself");
    ctx->halo_send_off[r] = ns;
    ctx->halo_send_cnt[r] = send_counts[r];
    ctx->halo_recv_off[r] = nr;
    ctx->halo_recv_cnt[r] = recv_counts[r];
    ns += send_counts[r];
    nr += recv_counts[r];
  }
  if (nr != ctx->nghost) return fail(PSLR_EDIM, "received ghosts differ from the context's ghost columns");
  for (int64_t i = 0; i < ns; ++i)
    if (send_idx[i] < 0 || send_idx[i] >= ctx->q) return fail(PSLR_EDIM, "halo send index out of range");
  free_ptr(ctx, ctx->halo_idx);
  free_ptr(ctx, ctx->halo_buf);
  ctx->halo_idx = nullptr;
  ctx->halo_buf = nullptr;
  ctx->halo_nsend = ns;
  if (ns > 0) {
    double* idx = nullptr;  // int32 indices in a double-sized scratch allocation
    RET(alloc_scratch(ctx, &idx, (ns + 1) / 2 + 1));
    ctx->halo_idx = reinterpret_cast<int32_t*>(idx);
    CK(cudaMemcpy(ctx->halo_idx, send_idx, ns * sizeof(int32_t), cudaMemcpyHostToDevice));
    RET(alloc_scratch(ctx, &ctx->halo_buf, ns));
  }
  return PSLR_OK;
}

}  // extern "C"
