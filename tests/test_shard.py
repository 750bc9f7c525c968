"""Multi-GPU sharding on CPU: the halo plan, and the sharded apply / Arnoldi
run by world_size-2 gloo process groups with an oracle backend for the rank-local
operators, against the single-process oracle (pslr/preconditioner.py:79-93,
lowrank.py:39-73)."""
import os
import socket

import numpy as np
import pytest

from oracle import pslr_oracle as O
from paper_2002_00917_b200 import shard


def _system(n=10, s=4, shift=0.5):
    A = O.laplacian3d(n, n, n, shift)
    assign = O.partition_c(A, s)
    return O.classify_and_reorder(A, assign, s)


def _ref_ranges(ps, world):
    io = np.concatenate([[0], np.cumsum(ps.interior_sizes)])
    fo = np.concatenate([[0], np.cumsum(ps.interface_sizes)])
    return io, fo


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_plan_covers_and_matches(world):
    ps = _system(8, 4)
    plans = [shard.plan_shard(ps, world, r) for r in range(world)]
    rows = np.concatenate([shard.local_rows(pl, ps.p) for pl in plans])
    assert np.array_equal(np.sort(rows), np.arange(ps.n))
    for pl in plans:
        # local blocks equal the global ones; C (with ghosts) reproduces the global rows
        loc = pl.local
        gi = np.arange(pl.int_lo, pl.int_hi)
        gf = np.arange(pl.ifc_lo, pl.ifc_hi)
        assert (loc.B != ps.B[gi][:, gi]).nnz == 0
        assert (loc.E != ps.E[gi][:, gf]).nnz == 0
        assert (loc.F != ps.F[gf][:, gi]).nnz == 0
        cols = np.concatenate([gf, pl.ghosts])
        assert (loc.C != ps.C[gf][:, cols]).nnz == 0
        assert ps.C[gf].nnz == loc.C.nnz  # nothing outside local + ghosts
        import scipy.sparse as sp
        C0e = sp.csr_matrix((pl.C0.data, pl.C0.indices, pl.C0.indptr), shape=loc.C.shape)
        assert (C0e + pl.Cg != loc.C).nnz == 0
        # the halo pattern is symmetric: what r sends to h is h's ghost slice owned by r
        for h, other in enumerate(plans):
            if h == pl.rank:
                continue
            off = np.concatenate([[0], np.cumsum(other.recv_counts)])
            theirs = other.ghosts[off[pl.rank]:off[pl.rank + 1]]
            assert np.array_equal(pl.ifc_lo + pl.send_idx[h], theirs)


class OracleShardOps:
    """Rank-local operators from the oracle (scipy), for the CPU process-group tests."""

    def __init__(self, plan):
        import torch
        self.t, self.device, self.plan = torch, "cpu", plan
        loc = plan.local
        self.n, self.p, self.q, self.ng, self.r = loc.n, loc.p, loc.q, plan.nghost, 0
        self.b = O.factor_blocks(loc.B, loc.interior_sizes)
        self.c0 = O.factor_blocks(plan.C0, loc.interface_sizes) if loc.q else None
        self.E, self.F, self.Cg = loc.E, loc.F, plan.Cg

    def _t(self, x):
        return self.t.as_tensor(np.ascontiguousarray(x, dtype=np.float64))

    def vec(self, n):
        return self.t.empty(n, dtype=self.t.float64)

    def zeros(self, n):
        return self.t.zeros(n, dtype=self.t.float64)

    def _ext(self, x):
        out = self.zeros(self.q + self.ng)
        out[:self.q] = self._t(x)
        return out

    def set_correction(self, V, G):
        self.V, self.G, self.r = np.asarray(V), np.asarray(G), G.shape[0]

    def first(self, b):
        b = b.numpy()
        y0 = b[self.p:] - self.F @ O.block_solve(self.b, b[:self.p])
        s = self.V.T @ y0 if self.r else np.zeros(0)
        return self._t(y0), self._t(s)

    def mid(self, y0, s):
        y = y0.numpy()
        if self.r:
            y = y + self.V @ (self.G @ s.numpy())
        return self._ext(O.block_solve(self.c0, y))

    def _es(self, v_ext):
        v = v_ext.numpy()
        return self.F @ O.block_solve(self.b, self.E @ v[:self.q]) - self.Cg @ v

    def horner(self, y_ext, c):
        return self._ext(O.block_solve(self.c0, self._es(y_ext)) + c.numpy()[:self.q])

    def last(self, b, y):
        b, y = b.numpy(), y.numpy()
        return self._t(np.concatenate([O.block_solve(self.b, b[:self.p] - self.E @ y), y]))

    def solve_C0(self, g):
        return self._ext(O.block_solve(self.c0, g.numpy()))

    def es_step(self, v_ext, do_c0):
        e = self._es(v_ext)
        return self._ext(O.block_solve(self.c0, e) if do_c0 else e)

    def basis(self, rows, n):
        return self.zeros(rows * n).reshape(rows, n)

    def cgs_pass(self, mode, V, k, w, h0=None):
        """The CGS2 passes in plain torch (the device backend runs pslr_cgs_pass)."""
        Vk = V[:k]
        if mode != 0:
            w -= h0 @ Vk
        return (w @ w).reshape(1) if mode == 2 else Vk @ w

    def spmv_A(self, x_ext):
        return self._t(self.plan.local.matrix @ x_ext.numpy())


def _worker(rank, world, port, n, s, m, r, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps = _system(n, s)
        plan = shard.plan_shard(ps, world, rank)
        ops = OracleShardOps(plan)
        halo = shard.Halo(plan, "cpu")
        Vl, H, rr = shard.sharded_arnoldi(ops, halo, ps.q, plan.ifc_lo, m, r, seed=0)
        corr = O.build_correction(np.zeros((0, rr)), H)
        ops.set_correction(Vl.numpy(), corr.G)
        P = shard.ShardedPreconditioner(plan, ops, halo, m)
        b = np.random.default_rng(1).standard_normal(ps.n)
        rows = shard.local_rows(plan, ps.p)
        import torch
        z = P.apply(torch.as_tensor(b[rows]))
        b2 = np.random.default_rng(2).standard_normal(ps.n)
        z2 = P.apply2(torch.as_tensor(np.stack([b[rows], b2[rows]])))
        np.savez(os.path.join(out, f"r{rank}.npz"), z=z.numpy(), z2=z2.numpy(), rows=rows, H=H, V=Vl.numpy(),
                 ifc=np.arange(plan.ifc_lo, plan.ifc_hi))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.parametrize("world,n,s", [(2, 10, 4), (2, 8, 8)])
def test_sharded_apply_matches_single_process(tmp_path, world, n, s):
    import torch.multiprocessing as mp
    m, r = 3, 6
    mp.spawn(_worker, args=(world, _free_port(), n, s, m, r, str(tmp_path)), nprocs=world, join=True)
    ps = _system(n, s)
    ctx = O.schur_context(ps)
    V, H, rr = O.arnoldi(lambda v: O.apply_Err(ctx, m, v), ps.q, r, seed=0)
    corr = O.build_correction(V, H)
    P = O.Preconditioner(ps, ctx, m, corr)
    b = np.random.default_rng(1).standard_normal(ps.n)
    z_ref = P.apply(b)
    z = np.zeros(ps.n)
    zb = np.zeros(ps.n)
    Vs = np.zeros_like(V)
    for k in range(world):
        d = np.load(tmp_path / f"r{k}.npz")
        z[d["rows"]] = d["z"]
        # apply2 (two right-hand sides, one set of collectives): row 0 is apply() exactly
        np.testing.assert_array_equal(d["z2"][0], d["z"])
        zb[d["rows"]] = d["z2"][1]
        # Arnoldi: the same H on every rank, the rank's rows of V
        assert np.allclose(d["H"], H, rtol=1e-10, atol=1e-12)
        Vs[d["ifc"]] = d["V"]
    assert np.allclose(Vs, V, rtol=1e-9, atol=1e-11)
    assert np.max(np.abs(z - z_ref)) <= 1e-10 * np.max(np.abs(z_ref))
    zb_ref = P.apply(np.random.default_rng(2).standard_normal(ps.n))
    assert np.max(np.abs(zb - zb_ref)) <= 1e-10 * np.max(np.abs(zb_ref))


def _gmres_worker(rank, world, port, n, s, m, r, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps = _system(n, s)
        plan = shard.plan_shard(ps, world, rank)
        ops = OracleShardOps(plan)
        halo = shard.Halo(plan, "cpu")
        Vl, H, rr = shard.sharded_arnoldi(ops, halo, ps.q, plan.ifc_lo, m, r, seed=0)
        ops.set_correction(Vl.numpy(), O.build_correction(np.zeros((0, rr)), H).G)
        P = shard.ShardedPreconditioner(plan, ops, halo, m)
        xs = np.random.default_rng(0).standard_normal(ps.n)
        b = ps.matrix @ xs
        rows = shard.local_rows(plan, ps.p)
        res = {}
        for flex in (False, True):
            x, conv, its, rel, hist = shard.sharded_gmres(P, torch.as_tensor(b[rows]), tol=1e-8,
                                                          maxit=60, restart=10, flexible=flex)
            res[f"x{int(flex)}"] = x.numpy()
            res[f"its{int(flex)}"] = its
            res[f"hist{int(flex)}"] = np.asarray(hist)
        np.savez(os.path.join(out, f"g{rank}.npz"), rows=rows, **res)
    finally:
        dist.destroy_process_group()


def test_sharded_gmres_matches_single_process(tmp_path):
    """GMRES / FGMRES over a gloo world of 2 == the oracle's krylov.py:35-129 (its within
    +-2, residual histories to 1e-6 relative: only reduction order differs)."""
    import torch.multiprocessing as mp
    world, n, s, m, r = 2, 10, 4, 3, 6
    mp.spawn(_gmres_worker, args=(world, _free_port(), n, s, m, r, str(tmp_path)), nprocs=world, join=True)
    ps = _system(n, s)
    ctx = O.schur_context(ps)
    V, H, rr = O.arnoldi(lambda v: O.apply_Err(ctx, m, v), ps.q, r, seed=0)
    P = O.Preconditioner(ps, ctx, m, O.build_correction(V, H))
    xs = np.random.default_rng(0).standard_normal(ps.n)
    b = ps.matrix @ xs
    x_ref, rep = O.gmres(lambda v: ps.matrix @ v, P.apply, b, tol=1e-8, maxit=60, restart=10)
    d = [np.load(tmp_path / f"g{k}.npz") for k in range(world)]
    for flex in (0, 1):
        assert abs(int(d[0][f"its{flex}"]) - rep.iterations) <= 2
        assert int(d[0][f"its{flex}"]) == int(d[1][f"its{flex}"])
        h = d[0][f"hist{flex}"]
        k = min(len(h), len(rep.history))
        assert np.allclose(h[:k], rep.history[:k], rtol=1e-6, atol=1e-14)
        x = np.zeros(ps.n)
        for dk in d:
            x[dk["rows"]] = dk[f"x{flex}"]
        rel = np.linalg.norm(ps.matrix @ x - b) / np.linalg.norm(b)
        assert abs(rel - rep.final_relres) <= 1e-3 * rep.final_relres + 1e-12


def _groups_worker(rank, world, port, n, s, m, r, out):
    """Two apply pipelines per rank on two process groups (the bench's concurrent sweep
    at N > 1): interleaved applies give the single-process results."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps = _system(n, s)
        plan = shard.plan_shard(ps, world, rank)
        g2 = dist.new_group(list(range(world)))
        pipes = []
        for grp in (None, g2):
            ops = OracleShardOps(plan)
            halo = shard.Halo(plan, "cpu", grp)
            pipes.append((ops, halo))
        Vl, H, rr = shard.sharded_arnoldi(pipes[0][0], pipes[0][1], ps.q, plan.ifc_lo, m, r, seed=0)
        G = O.build_correction(np.zeros((0, rr)), H).G
        Ps = []
        for ops, halo in pipes:
            ops.set_correction(Vl.numpy(), G)
            Ps.append(shard.ShardedPreconditioner(plan, ops, halo, m))
        rows = shard.local_rows(plan, ps.p)
        zs = []
        for k in range(4):
            b = np.random.default_rng(100 + k).standard_normal(ps.n)
            zs.append(Ps[k % 2].apply(torch.as_tensor(b[rows])).numpy())
        np.savez(os.path.join(out, f"p{rank}.npz"), rows=rows, z=np.stack(zs))
    finally:
        dist.destroy_process_group()


def test_two_pipelines_on_two_groups(tmp_path):
    import torch.multiprocessing as mp
    world, n, s, m, r = 2, 8, 4, 3, 4
    mp.spawn(_groups_worker, args=(world, _free_port(), n, s, m, r, str(tmp_path)), nprocs=world, join=True)
    ps = _system(n, s)
    ctx = O.schur_context(ps)
    V, H, rr = O.arnoldi(lambda v: O.apply_Err(ctx, m, v), ps.q, r, seed=0)
    P = O.Preconditioner(ps, ctx, m, O.build_correction(V, H))
    d = [np.load(tmp_path / f"p{k}.npz") for k in range(world)]
    for k in range(4):
        z = np.zeros(ps.n)
        for dk in d:
            z[dk["rows"]] = dk["z"][k]
        zr = P.apply(np.random.default_rng(100 + k).standard_normal(ps.n))
        assert np.max(np.abs(z - zr)) <= 1e-10 * np.max(np.abs(zr))
