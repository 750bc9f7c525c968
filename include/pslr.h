/*
 * pslr.h — C-ABI of libpslr.so, the B200-native (sm_100a) hot path of the
 * PSLR preconditioner (arXiv 2002.00917).
 *
 * The reference (pslr 0.1.0, pure Python) has no FFI layer: its seam is the
 * Python API.  Each entry point below replaces one reference function, cited
 * as file:line under /root/reference/pkg/src/pslr/.  Plain pointers and sizes
 * only; no torch types.  Device-side entry points take DEVICE pointers and a
 * cudaStream_t passed as void*; `_host` variants take host pointers and do the
 * host<->device copies inside the call.
 *
 * Status codes map to the reference's exceptions in the Python binding:
 *   PSLR_EDIM / PSLR_EINVAL -> ValueError            (schur.py:62-66, preconditioner.py:82-84,
 *                                                     lowrank.py:101-102, ilu.py:189-191)
 *   PSLR_ENONFINITE         -> ArithmeticError       (krylov.py:81-82, 122-123)
 *   PSLR_ESINGULAR          -> CorrectionSingularError (lowrank.py:88-93)
 *   PSLR_ECUDA / PSLR_ENOMEM-> RuntimeError
 *   PSLR_ENOTSPD            -> NotSpdError           (krylov.py:18-19, 153-154)
 * pslr_last_error() returns a thread-local message for the last failure.
 *
 * Threading: one context per GPU per process; calls on one context are
 * stream-ordered and must not run concurrently (the context owns its scratch).
 */
#ifndef PSLR_H_
#define PSLR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSLR_OK 0
#define PSLR_EDIM 1
#define PSLR_ENONFINITE 2
#define PSLR_ESINGULAR 3
#define PSLR_ECUDA 4
#define PSLR_EINVAL 5
#define PSLR_ENOMEM 6
#define PSLR_ENCCL 7
#define PSLR_ENOTSPD 8
#define PSLR_ECALLBACK 9  /* a caller-supplied operator callback failed (its own error stands) */

typedef struct pslr_ctx pslr_ctx;
/* A caller-supplied linear operator for the *_op Krylov drivers: y = op(x) on device
 * vectors of the driver's dimension, enqueued on (or synchronised with) `stream`;
 * returns 0 on success.  It is called from the thread that called the driver. */
typedef int (*pslr_vec_fn)(void* user, const double* x_dev, double* y_dev, void* stream);
typedef struct pslr_factors pslr_factors;

/* A CSR matrix in host memory (sorted column indices, no duplicates). */
typedef struct {
  int64_t nrows, ncols, nnz;
  const int64_t* indptr;  /* nrows+1 */
  const int32_t* indices; /* nnz */
  const double* data;     /* nnz */
} pslr_csr;

/* The reordered system and its block factors — the state the reference keeps in
 * PartitionedSystem (partition.py:33-56) and SchurContext (schur.py:26-38). */
typedef struct {
  int64_t n, p, q, s;
  const int64_t* interior_offsets;  /* s+1: block offsets of B (cumsum of interior_sizes) */
  const int64_t* interface_offsets; /* s+1: block offsets of C0 (cumsum of interface_sizes) */
  pslr_csr LB, UB;                  /* BlockILU of B: unit-lower L (diag stored), upper U (ilu.py:141-164) */
  pslr_csr LC, UC;                  /* BlockILU of C0 */
  pslr_csr E, F;                    /* p x q, q x p (partition.py:522-525) */
  pslr_csr C, C0, Cg;               /* q x q: C, its block-diagonal part C0, and C - C0 (schur.py:52-59) */
  pslr_csr A;                       /* n x n reordered matrix (PartitionedSystem.matrix; cli.py:135) */
} pslr_system;

typedef struct {
  int64_t n, p, q, s, rank;
  int64_t levels_LB, levels_UB, levels_LC, levels_UC;      /* summed over blocks */
  int64_t maxdepth_LB, maxdepth_UB, maxdepth_LC, maxdepth_UC;
  int64_t nnz_LB, nnz_UB, nnz_LC, nnz_UC, nnz_E, nnz_F, nnz_C, nnz_C0, nnz_Cg, nnz_A;
  int64_t device_bytes;                                    /* resident device footprint */
  int64_t sm_count;
  int64_t ring_slots;  /* W: shared-memory solution ring (doubles) of the streamed solve */
  int64_t stages;      /* TMA pipeline stages per CTA */
  int64_t far_deps;    /* dependencies read from global memory (beyond the ring) */
  int64_t reach;       /* max level-order distance of a dependency */
  int64_t nghost;      /* sharded contexts: ghost interface values after the local q (see below) */
} pslr_ctx_info_t;

/* ---------------------------------------------------------------- misc */
const char* pslr_last_error(void);
int pslr_abi_version(void);

/* ---------------------------------------------------------------- host setup (C++)
 * Bit-identical restatements of the reference's pure-Python setup loops. */

/* partition.py:72-132 (_bfs_order/_bisect/partition_graph) on the symmetrised
 * off-diagonal adjacency pattern (partition.py:59-69). assignment: n int64. */
int pslr_partition_bisect(int64_t n, const int64_t* adj_indptr, const int64_t* adj_indices,
                          int64_t parts, int64_t* assignment);

/* ilu.py:35-138 (ilut) for every diagonal block, ilu.py:167-184 (factor_blocks).
 * Input: the block-diagonal matrix (CSR) and nblocks+1 offsets; fill_cap < 0 = None.
 * Blocks run in parallel on nthreads host threads (<=0: all cores). */
int pslr_ilut_blocks(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data,
                     int64_t nblocks, const int64_t* offsets, double droptol, int64_t fill_cap,
                     int nthreads, pslr_factors** out, int64_t* nnz_L, int64_t* nnz_U,
                     int64_t* pivot_repairs);
/* Assembled block-diagonal CSR factors (global indices), as sp.block_diag builds them. */
int pslr_factors_fetch(const pslr_factors* f, int64_t* Lp, int32_t* Li, double* Lx, int64_t* Up,
                       int32_t* Ui, double* Ux, int64_t* block_nnz /* 2*nblocks or NULL */,
                       int64_t* block_repairs /* nblocks or NULL */);
void pslr_factors_free(pslr_factors* f);
/* ilu.py:52 row norms (np.sqrt(A.multiply(A).sum(axis=1))), exposed for bit-exact tests. */
int pslr_row_norms(int64_t n, const int64_t* indptr, const double* data, double* out);

/* ---------------------------------------------------------------- device context */
/* Uploads the system, level-schedules every triangular factor per block, packs the
 * device formats. Replaces the state build() hands to the apply (preconditioner.py:120-141). */
int pslr_ctx_create(pslr_ctx** out, int device, const pslr_system* sys);
/* pslr_ctx_create with the packed device format as a reusable artefact:
 * the level schedules and streamed factor chunks are host work (pack.cpp).  blob_in (may be
 * NULL): a blob from an earlier call for the same system; it is used when it matches the
 * system, this library build and the device's shared-memory plan (*reused = 1), else the
 * system is packed again (*reused = 0).  blob_out (may be NULL): receives a malloc'd blob of
 * the packed format in use, to store next to a setup cache; free it with pslr_blob_free. */
int pslr_ctx_create_packed(pslr_ctx** out, int device, const pslr_system* sys, const void* blob_in,
                           int64_t blob_len, void** blob_out, int64_t* blob_out_len, int* reused);
void pslr_blob_free(void* blob);
void pslr_ctx_destroy(pslr_ctx* ctx);
int pslr_ctx_info(const pslr_ctx* ctx, pslr_ctx_info_t* info);
/* LowRankCorrection (lowrank.py:26-36): V q x r row-major, G r x r row-major, host pointers. */
int pslr_ctx_set_correction(pslr_ctx* ctx, int64_t r, const double* V, const double* G);
/* same, V already on the device (q x r row-major), G on the host */
int pslr_ctx_set_correction_device(pslr_ctx* ctx, int64_t r, const double* V_dev, const double* G);

/* ---------------------------------------------------------------- hot-path operators (device ptrs) */
int pslr_solve_B(pslr_ctx* ctx, const double* f, double* x, void* stream);        /* schur.py:69-70 */
int pslr_solve_C0(pslr_ctx* ctx, const double* g, double* y, void* stream);       /* schur.py:73-74 */
int pslr_apply_S(pslr_ctx* ctx, const double* v, double* out, void* stream);      /* schur.py:77-80 */
int pslr_apply_Es(pslr_ctx* ctx, const double* v, double* out, void* stream);     /* schur.py:83-86 */
int pslr_apply_neumann(pslr_ctx* ctx, int64_t m, const double* v, double* out, void* stream); /* schur.py:89-101 */
int pslr_apply_Err(pslr_ctx* ctx, int64_t m, const double* v, double* out, void* stream);     /* schur.py:104-112 */
int pslr_apply_correction(pslr_ctx* ctx, const double* y, double* out, void* stream);         /* lowrank.py:98-105 */
int pslr_apply(pslr_ctx* ctx, int64_t m, const double* b, double* z, void* stream);          /* preconditioner.py:79-93 */
/* which: 0=A 1=E 2=F 3=C0 4=Cg 5=C ; y = M x  (sparse.py:60-65 / scipy csr @) */
int pslr_spmv(pslr_ctx* ctx, int which, const double* x, double* y, void* stream);
/* pslr_apply with a CUDA event after every kernel launch (measurement only): per-launch
 * milliseconds and kinds (1 correction core, 2 first step, 3 correction+C0, 4 Horner step,
 * 5 last step, 6 permute of f); nlaunch = launches issued (up to cap reported). */
int pslr_apply_profiled(pslr_ctx* ctx, int64_t m, const double* b, double* z, void* stream,
                        double* launch_ms, int32_t* launch_kind, int64_t cap, int64_t* nlaunch);
/* Diagnostics (contexts created with PSLR_TRACE=1): timeline of CTA 0 since the last call,
 * as (code<<32 | arg, globaltimer ns) pairs; count = pairs returned. */
int pslr_debug_trace(pslr_ctx* ctx, int64_t* out, int64_t cap, int64_t* count);
/* Alg. 3.2 with HOST buffers (copies inside): the call a CPU user of P.apply makes. */
int pslr_apply_host(pslr_ctx* ctx, int64_t m, const double* b_host, double* z_host, void* stream);
/* The same without the final stream synchronisation (pinned host buffers; the caller
 * synchronises the stream before reading z_host). */
int pslr_apply_host_async(pslr_ctx* ctx, int64_t m, const double* b_host, double* z_host, void* stream);

/* Alg. 3.2 for nv vectors (b, z: nv n-vectors, vector-major, device pointers): pairs of
 * vectors share one launch sequence (each launch streams the factors once for both and
 * interleaves their two dependency chains); every vector's result is the single-vector
 * pslr_apply bit for bit. */
int pslr_apply_multi(pslr_ctx* ctx, int64_t m, int64_t nv, const double* b, double* z, void* stream);
/* pslr_apply_multi with HOST buffers (pinned for asynchrony), enqueued on `stream` without
 * synchronising: nv vector-major n-vectors copied in, applied, copied back. */
int pslr_apply_multi_host_async(pslr_ctx* ctx, int64_t m, int64_t nv, const double* b_host,
                                double* z_host, void* stream);

/* ---------------------------------------------------------------- concurrent applies
 * A step launch occupies one SM per subdomain (s of the 148); independent applies (the
 * apply sweep, several right-hand sides) run concurrently on separate streams, one
 * context each.  A clone shares every read-only device array of its source (factors,
 * matrices, the low-rank correction) and owns only its scratch: it must be destroyed
 * before the source, and the correction cannot be reset while clones exist. */
int pslr_ctx_clone(const pslr_ctx* src, pslr_ctx** out);

/* ---------------------------------------------------------------- sharded apply (multi-GPU)
 * rank g owns a contiguous range of subdomains; B, C0, E, F are local.
 * A context is SHARDED when its C, Cg (q rows) and A (n rows) carry nghost extra
 * columns: interface values owned by other ranks ("ghosts"), which every interface
 * vector the Horner steps read stores after its q local values ("extended" vectors,
 * q + nghost).  The apply (preconditioner.py:79-93) is split where ranks exchange data;
 * the caller (paper_2002_00917_b200/shard.py) runs the exchanges between the calls:
 *   first  : y0 = g - F B^{-1} f ; s = V^T y0 over the local rows   -> allreduce(s)
 *   mid    : y1 = y0 + V G s ; c = C0^{-1} y1  (c extended)         -> halo(c)
 *   horner : out = C0^{-1}(E_s y) + c  (y extended), m times        -> halo(out) between
 *   last   : z = [B^{-1}(f - E y) ; y]   (same b as the preceding first: f is kept permuted)
 * The fused single-context calls above require nghost == 0. */
int pslr_apply_first(pslr_ctx* ctx, const double* b, double* y0, double* s, void* stream);
int pslr_apply_mid(pslr_ctx* ctx, const double* y0, const double* s, double* c, void* stream);
int pslr_apply_horner(pslr_ctx* ctx, const double* y, const double* c, double* out, void* stream);
int pslr_apply_last(pslr_ctx* ctx, const double* b, const double* y, double* z, void* stream);
/* The same split for TWO right-hand sides sharing every launch (pslr_apply_multi's path;
 * needs p > 0 and q > 0): b, z two vector-major local n-vectors; y0, c, y, out
 * interleaved interface vectors (value of vector v at interface row i at [2 i + v],
 * ghosts after the q local rows); s two vector-major r-vectors.  Each vector's result is
 * the single-vector split apply's bit for bit. */
int pslr_apply2_first(pslr_ctx* ctx, const double* b, double* y0, double* s, void* stream);
int pslr_apply2_mid(pslr_ctx* ctx, const double* y0, const double* s, double* c, void* stream);
int pslr_apply2_horner(pslr_ctx* ctx, const double* y, const double* c, double* out, void* stream);
int pslr_apply2_last(pslr_ctx* ctx, const double* b, const double* y, double* z, void* stream);
/* out = C0^{-1}? (F B^{-1} E v - Cg v) with v extended: one E_rr / Arnoldi operator step
 * (schur.py:83-86, 104-112); do_c0 selects the C0 solve. */
int pslr_apply_es_step(pslr_ctx* ctx, const double* v, double* out, int do_c0, void* stream);
/* Halo overlapped with the interior phase.  Of a horner / es_step call only the C_g y term
 * of the interface phase reads ghost columns; the E y rows and the B solves (most of the
 * step) read local values.  A caller whose ghost refresh of y runs on ANOTHER stream
 * registers the cudaEvent_t that completes it: the next horner / es_step (one- or
 * two-vector) on this context launches the E y kernel and the B phases at once and makes
 * its stream wait for the event only before the C_g y kernel.  The exchange itself must be
 * ordered after the producer of y by the caller (an event on the compute stream).  The
 * registration is consumed by that one call; event NULL clears it.  The in-library NCCL
 * route (pslr_comm_init) does the same internally on a communication stream of its own. */
int pslr_halo_pending(pslr_ctx* ctx, void* event);

/* ---------------------------------------------------------------- multi-GPU (NCCL) */
/* One process per GPU; each rank holds a rank-local context (pslr_ctx_create on its
 * subdomains' rows; C, Cg and A carry nghost ghost interface columns).  With a
 * communicator and a halo plan, pslr_apply / pslr_apply_Err / pslr_arnoldi / pslr_gmres /
 * pslr_cg on that context run the coupled problem: m halo exchanges + 1 allreduce(r) per
 * apply, a halo per A-SpMV, an allreduce per CGS2 pass.  NCCL is loaded
 * at run time (libnccl.so.2).
 * pslr_comm_unique_id: rank 0 creates the 128-byte ncclUniqueId; the caller broadcasts it.
 * pslr_ctx_set_halo: per peer rank (world entries), the number of local interface values
 * sent (send_idx: their local interface indices, peers in ascending rank) and of ghosts
 * received (stored after the q local interface rows, peers in ascending rank). */
int pslr_comm_unique_id(void* out_128_bytes);
int pslr_comm_init(pslr_ctx* ctx, const void* nccl_unique_id, int nranks, int rank);
int pslr_ctx_set_halo(pslr_ctx* ctx, int world, const int64_t* send_counts, const int32_t* send_idx,
                      const int64_t* recv_counts);

/* ---------------------------------------------------------------- Krylov (device) */
/* lowrank.py:39-73 on op = E_rr(m) (schur.py:104-112), preconditioner.py:133-136.
 * v0: host start vector (this rank's q rows of the global seeded draw).  It is used as is
 * when its (global) 2-norm is 1 to within 1e-14 — the Python wrapper normalises it with
 * numpy, as the reference — and divided by its norm otherwise.
 * V_dev: q x r_out row-major output, PACKED (leading dimension r_out, the achieved rank;
 * room for q x rank doubles); H: host r_out x r_out row-major (room for rank x rank);
 * r_out: achieved rank (< rank on happy breakdown).  On a sharded context the rank is
 * capped by the global interface dimension and every rank runs the same collectives. */
int pslr_arnoldi(pslr_ctx* ctx, int64_t m, int64_t rank, const double* v0, double* V_dev,
                 double* H, int64_t* r_out, void* stream);
/* lowrank.py:39-73 for any operator (the reference's `op` callable): the same device CGS2
 * Arnoldi, V_dev dim x r_out packed; ctx only provides device scratch (a
 * pslr_workspace_create context will do). */
int pslr_arnoldi_op(pslr_ctx* ctx, int64_t dim, pslr_vec_fn op, void* user, int64_t rank, const double* v0,
                    double* V_dev, double* H, int64_t* r_out, void* stream);
/* A context without a system: device scratch for the *_op drivers on generic operators
 * (krylov.py's gmres / cg with arbitrary apply_A / apply_M).  Destroy with pslr_ctx_destroy. */
int pslr_workspace_create(pslr_ctx** out, int device);
/* y = M x for a device CSR matrix (int32 indptr / indices, fp64 data), scipy csr_matvec
 * order (bit-identical to A @ x): the generic drivers' operator for a scipy matrix. */
int pslr_csr_spmv(int64_t nrows, int64_t ncols, const int32_t* indptr, const int32_t* indices, const double* data,
                  const double* x, double* y, void* stream);
/* krylov.py:35-129 for any operator pair on device n-vectors: A_fn NULL -> the context's
 * reordered matrix; M_fn NULL -> the context's PSLR apply (precond != 0) or the identity. */
int pslr_gmres_op(pslr_ctx* ctx, int64_t m, int64_t n, pslr_vec_fn A_fn, void* A_user, pslr_vec_fn M_fn,
                  void* M_user, int precond, const double* b, double* x, double tol, int64_t maxit,
                  int64_t restart, int flexible, int64_t* iterations, int* converged, double* final_relres,
                  double* history, int64_t* history_len, void* stream);
/* krylov.py:35-129 on (A = reordered matrix, M = PSLR apply (precond!=0) or identity).
 * flexible!=0: FGMRES (Z_j = M v_j stored, x += Z y) — config 3's accelerator.
 * b, x: device n-vectors. history: host buffer of maxit+1 doubles. */
int pslr_gmres(pslr_ctx* ctx, int64_t m, const double* b, double* x, double tol, int64_t maxit,
               int64_t restart, int precond, int flexible, int64_t* iterations, int* converged,
               double* final_relres, double* history, int64_t* history_len, void* stream);
/* One CGS2 pass over a column-major basis X (k columns of n rows, leading dimension ld)
 * and a vector w, all device pointers (krylov.py:75-80, lowrank.py:62-67):
 *   mode 0: out[0..k) = X^T w ;  mode 1: w -= X h0, then out[0..k) = X^T w ;
 *   mode 2: w -= X h0, then out[0] = w.w .
 * The sharded Krylov loops (shard.py) run the three passes with an allreduce of `out`
 * between them; the single-GPU drivers use the same kernels inside pslr_gmres/pslr_arnoldi. */
int pslr_cgs_pass(pslr_ctx* ctx, int mode, const double* X, int64_t ld, int64_t n, int64_t k, double* w,
                  const double* h0, double* out, void* stream);
/* krylov.py:132-174: preconditioned CG (zero initial guess) on the same operators,
 * the CLI's `--krylov cg` path (cli.py:138-139).  PSLR_ENOTSPD when p.Ap <= 0
 * (krylov.py:153-154).  b, x: device n-vectors; history: host, maxit+1 doubles. */
int pslr_cg(pslr_ctx* ctx, int64_t m, const double* b, double* x, double tol, int64_t maxit, int precond,
            int64_t* iterations, int* converged, double* final_relres, double* history,
            int64_t* history_len, void* stream);
/* krylov.py:132-174 for any operator pair (same conventions as pslr_gmres_op). */
int pslr_cg_op(pslr_ctx* ctx, int64_t m, int64_t n, pslr_vec_fn A_fn, void* A_user, pslr_vec_fn M_fn,
               void* M_user, int precond, const double* b, double* x, double tol, int64_t maxit,
               int64_t* iterations, int* converged, double* final_relres, double* history, int64_t* history_len,
               void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PSLR_H_ */
