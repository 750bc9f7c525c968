"""Multi-GPU sharding of the PSLR apply: one process per GPU, each rank owns a
contiguous range of subdomains.

The reference is single-process (pslr/preconditioner.py); this module is the sharded form
of its apply (preconditioner.py:79-93), Arnoldi (lowrank.py:39-73) and GMRES
(krylov.py:35-129).  Everything block-diagonal in Eq. 2.2 - the B and C0 solves, E, F - is
rank-local.  Ranks exchange data at exactly three kinds of points:

  * halo   - C_g couples interface values of different subdomains.  Each rank stores the
             remote interface values its C_g rows read as *ghosts* after its q local values
             ("extended" interface vectors); `Halo.exchange` refreshes them with one batch of
             point-to-point sends/receives before every operator step that reads C_g
             (m per apply, m+1 per Arnoldi operator, one per GMRES A-SpMV).
  * allreduce(r) - the low-rank correction's V^T y.
  * allreduce(k) - inner products of Arnoldi / GMRES (CGS2 projections, norms).

Subdomain ids from the depth-first bisection are contiguous subtrees (partition.py:103-116),
so a contiguous id range is a compact region of the mesh and the halo is small.

The orchestration is backend-agnostic: `ShardedPreconditioner` drives a local-operator
backend (`DeviceShardOps`: the split C-ABI apply pslr_apply_first/mid/horner/last on the
rank's GPU) through `torch.distributed` collectives (NCCL on GPUs; gloo in the CPU tests,
which plug in an oracle backend).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .ilu import factor_blocks
from .lowrank import BREAKDOWN_RTOL, LowRankCorrection, _start_vector, build_correction
from .partition import PartitionedSystem
from .sparse import canonical


# ---------------------------------------------------------------------------- plan
def subdomain_range(s: int, world: int, rank: int) -> tuple[int, int]:
    """Rank `rank` owns subdomain ids [lo, hi): contiguous, balanced by count."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    if s < world:
        raise ValueError(f"{s} subdomains cannot be sharded over {world} ranks")
    return rank * s // world, (rank + 1) * s // world


@dataclass
class ShardPlan:
    rank: int
    world: int
    sub_lo: int
    sub_hi: int
    int_lo: int            # global interior rows [int_lo, int_hi) of [0, p)
    int_hi: int
    ifc_lo: int            # global interface indices [ifc_lo, ifc_hi) of [0, q)
    ifc_hi: int
    ghosts: np.ndarray     # global interface indices of the ghosts, grouped by owner rank
    recv_counts: np.ndarray  # ghosts received from each rank (contiguous, in rank order)
    send_idx: list         # per rank: local interface indices this rank sends to it
    local: PartitionedSystem = field(repr=False)  # C and matrix carry the ghost columns
    C0: sp.csr_matrix = field(repr=False, default=None)
    Cg: sp.csr_matrix = field(repr=False, default=None)

    @property
    def q_loc(self) -> int:
        return self.ifc_hi - self.ifc_lo

    @property
    def nghost(self) -> int:
        return int(self.ghosts.size)

    @property
    def n_loc(self) -> int:
        return self.local.n


def _ranges(ps: PartitionedSystem, world: int):
    io = np.concatenate([[0], np.cumsum(ps.interior_sizes)]).astype(np.int64)
    fo = np.concatenate([[0], np.cumsum(ps.interface_sizes)]).astype(np.int64)
    out = []
    for r in range(world):
        lo, hi = subdomain_range(ps.num_parts, world, r)
        out.append((lo, hi, int(io[lo]), int(io[hi]), int(fo[lo]), int(fo[hi])))
    return out


def _remote_cols(C: sp.csr_matrix, f0: int, f1: int) -> np.ndarray:
    """Interface columns outside [f0, f1) read by interface rows [f0, f1) of C (sorted)."""
    blk = C[f0:f1]
    cols = np.unique(blk.indices)
    return cols[(cols < f0) | (cols >= f1)].astype(np.int64)


def plan_shard(ps: PartitionedSystem, world: int, rank: int) -> ShardPlan:
    """Local system of `rank` and its halo pattern.  Every rank derives every rank's ghost
    set from the (replicated) global system, so no collective is needed to set up."""
    if not hasattr(ps, "num_parts"):  # the oracle's System names it `s`
        ps = PartitionedSystem(matrix=ps.matrix, perm=ps.perm, num_parts=ps.s, p=ps.p, q=ps.q,
                               interior_sizes=ps.interior_sizes, interface_sizes=ps.interface_sizes,
                               B=ps.B, E=ps.E, F=ps.F, C=ps.C)
    rg = _ranges(ps, world)
    sub_lo, sub_hi, i0, i1, f0, f1 = rg[rank]
    owner_of_ifc = np.empty(ps.q, dtype=np.int64)
    for r, (_, _, _, _, a, b) in enumerate(rg):
        owner_of_ifc[a:b] = r
    C = canonical(ps.C)
    ghosts = _remote_cols(C, f0, f1)
    ghosts = ghosts[np.lexsort((ghosts, owner_of_ifc[ghosts]))]  # by owner, then index
    recv_counts = np.bincount(owner_of_ifc[ghosts], minlength=world).astype(np.int64)
    send_idx = []
    for r, (_, _, _, _, a, b) in enumerate(rg):
        if r == rank:
            send_idx.append(np.zeros(0, dtype=np.int64))
            continue
        theirs = _remote_cols(C, a, b)
        mine = theirs[(theirs >= f0) & (theirs < f1)]  # sorted = their ghost order for me
        send_idx.append((mine - f0).astype(np.int64))
    p_loc, q_loc = i1 - i0, f1 - f0
    # local column map of the reordered matrix: interiors, interfaces, ghosts
    ncol = np.full(ps.n, -1, dtype=np.int64)
    ncol[i0:i1] = np.arange(p_loc)
    ncol[ps.p + f0:ps.p + f1] = p_loc + np.arange(q_loc)
    ncol[ps.p + ghosts] = p_loc + q_loc + np.arange(ghosts.size)
    A = canonical(ps.matrix)
    rows = np.concatenate([np.arange(i0, i1), ps.p + np.arange(f0, f1)])
    Ar = canonical(A[rows])
    if np.any(ncol[Ar.indices] < 0):
        raise ValueError("the reordered matrix couples rows outside the subdomain + halo pattern")
    n_loc = p_loc + q_loc
    # Entries keep the global column order inside every row (ghost indices are not sorted
    # against local ones): it is the reference's summation order (scipy csr_matvec), so the
    # rank-local SpMVs of the ghost-carrying matrices stay bit-identical to the global ones.
    A_loc = _ordered_csr(Ar.data, ncol[Ar.indices], Ar.indptr, (n_loc, n_loc + ghosts.size))
    local = PartitionedSystem(
        matrix=A_loc, perm=None, num_parts=sub_hi - sub_lo, p=p_loc, q=q_loc,
        interior_sizes=np.asarray(ps.interior_sizes[sub_lo:sub_hi], dtype=np.int64),
        interface_sizes=np.asarray(ps.interface_sizes[sub_lo:sub_hi], dtype=np.int64),
        B=_block(A_loc, 0, p_loc, 0, p_loc),
        E=_block(A_loc, 0, p_loc, p_loc, n_loc),
        F=_block(A_loc, p_loc, n_loc, 0, p_loc),
        C=_block(A_loc, p_loc, n_loc, p_loc, n_loc + ghosts.size),  # q_loc x (q_loc + nghost)
    )
    C0, Cg = split_interface(local.C, local.interface_sizes)
    return ShardPlan(rank=rank, world=world, sub_lo=sub_lo, sub_hi=sub_hi, int_lo=i0, int_hi=i1,
                     ifc_lo=f0, ifc_hi=f1, ghosts=ghosts, recv_counts=recv_counts, send_idx=send_idx,
                     local=local, C0=C0, Cg=Cg)


def _ordered_csr(data, indices, indptr, shape) -> sp.csr_matrix:
    """CSR taken as given: entries stay in their order within each row (no sorting)."""
    M = sp.csr_matrix((np.asarray(data, dtype=np.float64), np.asarray(indices, dtype=np.int32),
                       np.asarray(indptr, dtype=np.int64)), shape=shape)
    M.has_sorted_indices = False  # never let scipy reorder the summation order
    return M


def _select(M: sp.csr_matrix, r0: int, r1: int, keep_fn, col_fn, ncols: int) -> sp.csr_matrix:
    """Rows [r0, r1) of M, the entries keep_fn(cols) selects, columns mapped by col_fn,
    in their original order."""
    ip = M.indptr
    lo, hi = ip[r0], ip[r1]
    cols = M.indices[lo:hi]
    rows = np.repeat(np.arange(r1 - r0), np.diff(ip[r0:r1 + 1]))
    k = keep_fn(cols, rows)
    counts = np.bincount(rows[k], minlength=r1 - r0)
    indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return _ordered_csr(M.data[lo:hi][k], col_fn(cols[k]), indptr, (r1 - r0, ncols))


def _block(M, r0, r1, c0, c1):
    return _select(M, r0, r1, lambda c, r: (c >= c0) & (c < c1), lambda c: c - c0, c1 - c0)


def split_interface(C: sp.csr_matrix, sizes) -> tuple[sp.csr_matrix, sp.csr_matrix]:
    """C0 = block-diagonal part over the local interface blocks (q x q), Cg = C - C0 keeping
    the ghost columns (schur.py:41-59 on the extended column space), entry order kept."""
    q = C.shape[0]
    block_of = np.repeat(np.arange(len(sizes)), sizes)

    def same(cols, rows):
        inb = cols < q
        out = np.zeros(cols.size, dtype=bool)
        out[inb] = block_of[rows[inb]] == block_of[cols[inb]]
        return out

    C0 = _select(C, 0, q, same, lambda c: c, q)
    Cg = _select(C, 0, q, lambda c, r: ~same(c, r), lambda c: c, C.shape[1])
    return C0, Cg


# ---------------------------------------------------------------------------- communication
class Halo:
    """Ghost exchange + reductions over a torch.distributed process group."""

    def __init__(self, plan: ShardPlan, device, group=None):
        import torch
        import torch.distributed as dist
        self.t, self.dist, self.group = torch, dist, group
        self.plan = plan
        self.q = plan.q_loc
        self.peers_send = [(r, torch.as_tensor(ix, device=device)) for r, ix in enumerate(plan.send_idx)
                           if ix.size]
        off = np.concatenate([[0], np.cumsum(plan.recv_counts)])
        self.peers_recv = [(r, int(off[r]), int(plan.recv_counts[r])) for r in range(plan.world)
                           if plan.recv_counts[r]]

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def exchange(self, v_ext):
        """Fill v_ext[q:] (the ghosts) with the owners' current values of v_ext[:q]."""
        if not self.peers_send and not self.peers_recv:
            return v_ext
        ops, bufs = [], []
        for r, ix in self.peers_send:
            buf = v_ext[:self.q].index_select(0, ix)
            bufs.append(buf)
            ops.append(self.dist.P2POp(self.dist.isend, buf, self._peer(r), self.group))
        for r, off, cnt in self.peers_recv:
            ops.append(self.dist.P2POp(self.dist.irecv, v_ext[self.q + off:self.q + off + cnt],
                                       self._peer(r), self.group))
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()
        return v_ext

    def exchange_for_step(self, v_ext, ops):
        """exchange(v_ext) for the horner / es_step call that follows on `ops`, overlapped
        with that step's interior phase when the rank-local operators are the device ones:
        the exchange runs on a side stream ordered after v_ext's producer and its completion
        event is registered with the context (pslr_halo_pending), so the step's E y kernel
        and B solves start at once and only the C_g y term waits for the ghosts.  Any other
        backend (or PSLR_HALO_OVERLAP=0): the plain exchange."""
        t = self.t
        if (not (self.peers_send or self.peers_recv) or not getattr(v_ext, "is_cuda", False)
                or not hasattr(ops, "halo_pending") or os.environ.get("PSLR_HALO_OVERLAP", "1") == "0"):
            return self.exchange(v_ext)
        if getattr(self, "_side", None) is None:
            self._side = t.cuda.Stream(device=v_ext.device)
            self._event = t.cuda.Event()
        main = t.cuda.current_stream(v_ext.device)
        self._side.wait_stream(main)
        v_ext.record_stream(self._side)
        with t.cuda.stream(self._side):
            self.exchange(v_ext)
            self._event.record(self._side)
        ops.halo_pending(self._event)
        return v_ext

    def allreduce(self, x):
        if self.plan.world > 1:
            self.dist.all_reduce(x, group=self.group)
        return x

    def dot(self, a, b):
        d = (a * b).sum().reshape(1)
        return self.allreduce(d)


# ---------------------------------------------------------------------------- device backend
class DeviceShardOps:
    """Rank-local operators of the split apply on this rank's GPU (libpslr.so)."""

    def __init__(self, plan: ShardPlan, droptol=1e-2, fill_cap=None, device=None):
        from .device import DeviceContext, require_cuda
        t = require_cuda()
        ps = plan.local
        self.plan = plan
        self.b_ilu = factor_blocks(ps.B, ps.interior_sizes, droptol=droptol, fill_cap=fill_cap)
        self.c0_ilu = factor_blocks(plan.C0, ps.interface_sizes, droptol=droptol, fill_cap=fill_cap)
        self.dev = DeviceContext(ps, self.b_ilu, self.c0_ilu, plan.C0, plan.Cg, device=device)
        self.t = t
        self.device = self.dev.dev
        self.n, self.p, self.q, self.ng = ps.n, ps.p, ps.q, plan.nghost
        self.r = 0

    def clone(self) -> "DeviceShardOps":
        """Rank-local operators sharing this one's factors and correction (pslr_ctx_clone),
        with private scratch: a second independent apply pipeline on another stream."""
        c = object.__new__(DeviceShardOps)
        c.__dict__.update(self.__dict__)
        c.dev = self.dev.clone()
        return c

    def _call(self, name, *args):
        from . import _lib
        _lib.check(_lib.fns[name](self.dev.handle, *args, self.dev.stream()))

    def vec(self, n):
        return self.t.empty(n, dtype=self.t.float64, device=self.device)

    def zeros(self, n):
        return self.t.zeros(n, dtype=self.t.float64, device=self.device)

    def set_correction(self, V_loc, G):
        self.dev.set_correction(V_loc, G)
        self.r = int(G.shape[0])

    def first(self, b):
        y0 = self.vec(self.q)
        s = self.zeros(max(self.r, 1))
        self._call("pslr_apply_first", b.data_ptr(), y0.data_ptr(), s.data_ptr())
        return y0, s[:self.r]

    def mid(self, y0, s):
        c = self.zeros(self.q + self.ng)
        sp_ = s if self.r else self.zeros(1)
        self._call("pslr_apply_mid", y0.data_ptr(), sp_.data_ptr(), c.data_ptr())
        return c

    def horner(self, y_ext, c):
        out = self.zeros(self.q + self.ng)
        self._call("pslr_apply_horner", y_ext.data_ptr(), c.data_ptr(), out.data_ptr())
        return out

    def last(self, b, y):
        z = self.vec(self.n)
        self._call("pslr_apply_last", b.data_ptr(), y.data_ptr(), z.data_ptr())
        return z

    # two right-hand sides per launch (pslr_apply2_*): b (2, n) vector-major, interface
    # vectors (q [+ ghosts], 2) interleaved, s (2, r)
    def first2(self, b2):
        y0 = self.t.empty((self.q, 2), dtype=self.t.float64, device=self.device)
        s = self.t.zeros((2, max(self.r, 1)), dtype=self.t.float64, device=self.device)
        self._call("pslr_apply2_first", b2.data_ptr(), y0.data_ptr(), s.data_ptr())
        return y0, s[:, :self.r].contiguous()

    def mid2(self, y0, s):
        c = self.t.zeros((self.q + self.ng, 2), dtype=self.t.float64, device=self.device)
        sp_ = s if self.r else self.zeros(2)
        self._call("pslr_apply2_mid", y0.data_ptr(), sp_.data_ptr(), c.data_ptr())
        return c

    def horner2(self, y_ext, c):
        out = self.t.zeros((self.q + self.ng, 2), dtype=self.t.float64, device=self.device)
        self._call("pslr_apply2_horner", y_ext.data_ptr(), c.data_ptr(), out.data_ptr())
        return out

    def last2(self, b2, y):
        z = self.t.empty((2, self.n), dtype=self.t.float64, device=self.device)
        self._call("pslr_apply2_last", b2.data_ptr(), y.data_ptr(), z.data_ptr())
        return z

    def solve_C0(self, g):
        out = self.zeros(self.q + self.ng)
        self._call("pslr_solve_C0", g.data_ptr(), out.data_ptr())
        return out

    def halo_pending(self, event):
        """The ghosts of the vector the next horner / es_step reads land when `event` (a
        torch.cuda.Event recorded on the exchanging stream) completes (pslr_halo_pending)."""
        from . import _lib
        _lib.check(_lib.fns["pslr_halo_pending"](self.dev.handle, event.cuda_event if event is not None else None))

    def es_step(self, v_ext, do_c0):
        out = self.zeros(self.q + self.ng)
        from . import _lib
        _lib.check(_lib.fns["pslr_apply_es_step"](self.dev.handle, v_ext.data_ptr(), out.data_ptr(),
                                                  int(do_c0), self.dev.stream()))
        return out

    def spmv_A(self, x_ext):
        y = self.vec(self.n)
        from . import _lib
        _lib.check(_lib.fns["pslr_spmv"](self.dev.handle, 0, x_ext.data_ptr(), y.data_ptr(),
                                         self.dev.stream()))
        return y

    def basis(self, rows, n):
        """Krylov basis storage: `rows` vectors of length n (row-major, padded stride)."""
        return _basis(self.t, rows, n, self.device)

    def cgs_pass(self, mode, V, k, w, h0=None):
        """One CGS2 pass over V[:k] (pslr_cgs_pass): 0 -> V w ; 1 -> w -= h0 V, then V w ;
        2 -> w -= h0 V, then [w.w].  w is updated in place; returns the rank-local partial."""
        out = self.t.empty(max(k, 1) if mode != 2 else 1, dtype=self.t.float64, device=self.device)
        self._call("pslr_cgs_pass", int(mode), V.data_ptr(), int(V.stride(0)), int(w.shape[0]), int(k),
                   w.data_ptr(), h0.data_ptr() if h0 is not None else None, out.data_ptr())
        return out


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for pslr_comm_init; rank 0 makes it, the caller
    broadcasts it (torch.distributed.broadcast_object_list, MPI, a file ...)."""
    from . import _lib
    buf = ctypes.create_string_buffer(128)
    _lib.check(_lib.fns["pslr_comm_unique_id"](buf))
    return buf.raw


def attach_nccl(ops: "DeviceShardOps", plan: "ShardPlan", unique_id: bytes) -> None:
    """Give the rank-local context its own NCCL communicator and this rank's halo plan:
    pslr_apply / pslr_apply_multi / pslr_apply_Err / pslr_arnoldi / pslr_gmres / pslr_cg on
    ops.dev.handle then run the coupled problem inside libpslr (include/pslr.h
    pslr_comm_init / pslr_ctx_set_halo) — the C-ABI route a non-Python caller uses."""
    attach_nccl_ctx(ops.dev, plan, unique_id)


def attach_nccl_ctx(dev, plan: "ShardPlan", unique_id: bytes) -> None:
    """attach_nccl for a DeviceContext (the built one or a pslr_ctx_clone of it: each
    independent pipeline owns a communicator)."""
    from . import _lib
    uid = ctypes.create_string_buffer(bytes(unique_id), 128)
    _lib.check(_lib.fns["pslr_comm_init"](dev.handle, uid, int(plan.world), int(plan.rank)))
    send_counts = np.asarray([ix.size for ix in plan.send_idx], dtype=np.int64)
    send_idx = (np.concatenate(plan.send_idx).astype(np.int32) if send_counts.sum()
                else np.zeros(1, dtype=np.int32))
    recv_counts = np.ascontiguousarray(plan.recv_counts, dtype=np.int64)
    _lib.check(_lib.fns["pslr_ctx_set_halo"](dev.handle, int(plan.world), send_counts.ctypes.data,
                                             send_idx.ctypes.data, recv_counts.ctypes.data))


def _basis(t, rows, n, device):
    """rows x n view of a rows x ld buffer, ld = n rounded up to 32 doubles and made an odd
    multiple of 256 B (krylov.cu basis_ld: the columns of one row tile must not share
    cache sets)."""
    ld = (n + 31) // 32 * 32
    if (ld // 32) % 2 == 0:
        ld += 32
    return t.zeros((rows, ld), dtype=t.float64, device=device)[:, :n]


def cgs2(ops, halo, V, k, w):
    """krylov.py:75-80 / lowrank.py:62-67 over the rank's rows: three passes over the basis
    with the projections allreduced in between (h1 = V^T w; w -= V h1 with h2 = V^T w;
    w -= V h2 with ||w||^2).  w is updated in place; returns (h1 + h2 as numpy, ||w||)."""
    h1 = halo.allreduce(ops.cgs_pass(0, V, k, w))
    h2 = halo.allreduce(ops.cgs_pass(1, V, k, w, h1))
    nn = halo.allreduce(ops.cgs_pass(2, V, k, w, h2))
    return (h1 + h2).cpu().numpy(), float(nn.sqrt().item())


# ---------------------------------------------------------------------------- sharded algorithms
def sharded_arnoldi(ops, halo: Halo, q_global: int, ifc_lo: int, m: int, rank: int, seed: int = 0):
    """lowrank.py:39-73 on E_rr(m) (schur.py:104-112) with the rank's rows of V: CGS2
    projections and norms are allreduced, every operator step refreshes the ghosts first.
    Returns (V_loc q_loc x r, H r x r numpy (identical on every rank), r)."""
    t = halo.t
    q = ops.q
    rank = min(int(rank), q_global)
    if rank == 0:
        return ops.zeros(q * 0).reshape(q, 0), np.zeros((0, 0)), 0
    v0 = _start_vector(q_global, seed)[ifc_lo:ifc_lo + q]  # the rank's rows of the global draw
    V = ops.basis(rank + 1, q)  # rows = basis vectors
    V[0] = t.as_tensor(np.ascontiguousarray(v0), device=ops.device)
    Hbar = np.zeros((rank + 1, rank))
    r = rank

    def op(v):
        src = ops.solve_C0(v)
        xch = getattr(halo, "exchange_for_step", None)
        for k in range(1, m + 2):
            xch(src, ops) if xch else halo.exchange(src)
            src = ops.es_step(src, do_c0=(k != m + 1))
        return src[:q]

    for j in range(rank):
        w = op(V[j].clone()).contiguous()
        hh, nrm = cgs2(ops, halo, V, j + 1, w)
        Hbar[:j + 1, j] = hh
        Hbar[j + 1, j] = nrm
        if nrm <= BREAKDOWN_RTOL:
            r = j + 1
            break
        V[j + 1] = w / nrm
    return V[:r].T.contiguous(), np.ascontiguousarray(Hbar[:r, :r]), r


class ShardedPreconditioner:
    """The PSLR apply on the rank's rows (preconditioner.py:79-93): b_loc = [f_loc; g_loc]
    in the rank's local order (interiors, then interfaces)."""

    def __init__(self, plan: ShardPlan, ops, halo: Halo, series_degree: int, correction=None):
        self.plan, self.ops, self.halo = plan, ops, halo
        self.series_degree = int(series_degree)
        self.correction = correction

    def apply(self, b):
        ops, halo, m = self.ops, self.halo, self.series_degree
        if b.shape[0] != ops.n:
            raise ValueError(f"vector has length {b.shape[0]}, local system has {ops.n}")
        if ops.q == 0 and self.plan.world == 1:
            return ops.last(b, ops.zeros(0))
        y0, s = ops.first(b)
        if ops.r:
            halo.allreduce(s)
        c = ops.mid(y0, s)
        y = c
        if m > 0:
            xch = getattr(halo, "exchange_for_step", None) or (lambda v, _o: halo.exchange(v))
            xch(c, ops)
            for k in range(m):
                out = ops.horner(y, c)
                if k < m - 1:
                    xch(out, ops)
                y = out
        return ops.last(b, y[:ops.q].contiguous())

    def apply2(self, b2):
        """Two right-hand sides (rows of b2, shape (2, n_loc)) through one launch sequence
        and one set of collectives (halo rows carry both vectors; one allreduce of 2r);
        each result row is apply() of that row bit for bit.  Ranks without the two-vector
        kernels (p or q empty, or a backend without them) run the vectors one by one
        between the SAME collectives, so every rank issues the same sequence."""
        ops, halo, m = self.ops, self.halo, self.series_degree
        t = ops.t
        if tuple(b2.shape) != (2, ops.n):
            raise ValueError(f"expected shape (2, {ops.n}), got {tuple(b2.shape)}")
        b2 = b2.contiguous()
        if ops.q == 0 and self.plan.world == 1:
            return t.stack([ops.last(b2[v], ops.zeros(0)) for v in range(2)])
        native = ops.q > 0 and ops.p > 0 and hasattr(ops, "first2")
        cols = lambda x: [x[:, v].contiguous() for v in range(2)]  # noqa: E731
        if native:
            y0, s = ops.first2(b2)
        else:
            f = [ops.first(b2[v]) for v in range(2)]
            y0, s = t.stack([f[0][0], f[1][0]], 1), t.stack([f[0][1], f[1][1]])
        if ops.r:
            halo.allreduce(s)
        c = ops.mid2(y0, s) if native else t.stack([ops.mid(yv, s[v].clone()) for v, yv in enumerate(cols(y0))], 1)
        y = c
        if m > 0:
            # (the per-vector fallback reads copies of y: no overlap there)
            xch = (getattr(halo, "exchange_for_step", None) if native else None) or (lambda v, _o: halo.exchange(v))
            xch(c, ops)
            cc = None if native else cols(c)
            for k in range(m):
                if native:
                    out = ops.horner2(y, c)
                else:
                    out = t.stack([ops.horner(yv, cc[v]) for v, yv in enumerate(cols(y))], 1)
                if k < m - 1:
                    xch(out, ops)
                y = out
        if native:
            return ops.last2(b2, y[:ops.q].contiguous())
        return t.stack([ops.last(b2[v], yv) for v, yv in enumerate(cols(y[:ops.q]))])


def build_sharded(ps: PartitionedSystem, cfg, group=None, device=None):
    """Rank-local part of build() (preconditioner.py:120-141) for the calling rank of the
    default (or given) process group."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world > 1:
        dist.barrier(group)  # a full collective first: NCCL's first P2P batch must not be partial
    plan = plan_shard(ps, world, rank)
    ops = DeviceShardOps(plan, droptol=cfg.droptol, fill_cap=cfg.fill_cap, device=device)
    halo = Halo(plan, ops.device, group)
    Vl, H, r = sharded_arnoldi(ops, halo, ps.q, plan.ifc_lo, cfg.series_degree,
                               min(cfg.rank, ps.q), seed=cfg.seed)
    corr = build_correction(np.zeros((0, r)), H) if r else LowRankCorrection(
        V=np.zeros((0, 0)), H=H, G=np.zeros((0, 0)), rank=0)
    if r:
        ops.set_correction(Vl, corr.G)
    return ShardedPreconditioner(plan, ops, halo, cfg.series_degree, corr)


def local_rows(plan: ShardPlan, p_global: int) -> np.ndarray:
    """Global (reordered) row indices of the rank's local vector, in local order."""
    return np.concatenate([np.arange(plan.int_lo, plan.int_hi),
                           p_global + np.arange(plan.ifc_lo, plan.ifc_hi)]).astype(np.int64)


def sharded_gmres(P: ShardedPreconditioner, b, tol=1e-8, maxit=500, restart=0, precond=True,
                  flexible=False):
    """krylov.py:35-129 on the rank's rows: right-preconditioned restarted GMRES, CGS2 +
    Givens, true residual at every cycle boundary (FGMRES stores Z_j = M v_j, the config 3
    accelerator).  Vectors stay on the rank's device; per iteration one sharded apply, one
    A-SpMV with a halo refresh, two allreduced CGS2 projections and an allreduced norm.
    The Givens/least-squares scalars are replicated host numpy, as in the reference.
    Returns (x_loc, converged, iterations, final_relres, history)."""
    ops, halo = P.ops, P.halo
    t = halo.t
    n, p, q = ops.n, ops.p, ops.q
    x_ext = ops.zeros(n + ops.ng)

    def matvec(v):
        x_ext[:n] = v
        halo.exchange(x_ext[p:])
        return ops.spmv_A(x_ext)

    M = P.apply if precond else (lambda v: v)

    def norm(v):
        return float(halo.dot(v, v).sqrt().item())

    bn = norm(b)
    if bn == 0.0:
        return ops.zeros(n), True, 0, 0.0, [1.0]
    x = ops.zeros(n)
    hist, total, conv, rel = [1.0], 0, False, 1.0
    while total < maxit and not conv:
        r = b - matvec(x)
        beta = norm(r)
        rel = beta / bn
        if rel <= tol:
            conv = True
            break
        cyc = maxit - total if restart <= 0 else min(restart, maxit - total)
        V = ops.basis(cyc + 1, n)
        Z = t.zeros((cyc, n), dtype=t.float64, device=ops.device) if flexible else None
        Hc = np.zeros((cyc + 1, cyc))
        cs, sn, g = np.zeros(cyc), np.zeros(cyc), np.zeros(cyc + 1)
        g[0] = beta
        V[0] = r / beta
        j, brk = 0, False
        while j < cyc:
            zj = M(V[j].contiguous())
            if flexible:
                Z[j] = zj
            w = matvec(zj).contiguous()
            h, hn = cgs2(ops, halo, V, j + 1, w)
            if not (np.all(np.isfinite(h)) and np.isfinite(hn)):
                raise ArithmeticError("GMRES diverged: non-finite values in the recurrence")
            Hc[:j + 1, j] = h
            Hc[j + 1, j] = hn
            for i in range(j):
                tt = cs[i] * Hc[i, j] + sn[i] * Hc[i + 1, j]
                Hc[i + 1, j] = -sn[i] * Hc[i, j] + cs[i] * Hc[i + 1, j]
                Hc[i, j] = tt
            d = np.hypot(Hc[j, j], hn)
            cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (Hc[j, j] / d, hn / d)
            Hc[j, j] = d
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            j += 1
            est = abs(g[j]) / bn
            hist.append(est)
            if hn <= 1e-14 * beta:
                brk = True
                break
            if est <= tol:
                break
            if j < cyc:
                V[j] = w / hn
        if j > 0:
            y = np.zeros(j)
            for i in range(j - 1, -1, -1):
                y[i] = (g[i] - Hc[i, i + 1:j] @ y[i + 1:j]) / Hc[i, i]
            yt = t.as_tensor(y, device=ops.device)
            x = x + (yt @ Z[:j] if flexible else M((yt @ V[:j]).contiguous()))
        rel = norm(b - matvec(x)) / bn
        hist[-1] = rel
        if rel <= tol:
            conv = True
        elif brk:
            break
    if not conv and total < maxit and not np.isfinite(rel):
        raise ArithmeticError("GMRES diverged: non-finite residual")
    its = total if conv else maxit
    if not conv:
        hist.extend([rel] * (maxit + 1 - len(hist)))
    return x, conv, its, rel, hist
