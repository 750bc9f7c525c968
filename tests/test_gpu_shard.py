"""GPU: the split apply of a sharded context (pslr_apply_first/mid/horner/last with ghost
columns) against the fused single-context apply.  The ranks of a 2- and 4-way sharding run
in lockstep in this one process on one GPU; their halo exchanges are host-ordered copies
between the ranks' tensors (no kernel waits on another rank's kernel).  The process-group
form of the same orchestration is covered on CPU by tests/test_shard.py (gloo).

Bars: bit-exact with the correction off (every rank-local operation is the single-context
operation on the same rows); 1e-12 relative with rank r > 0 (V^T y sums per rank, then
across ranks)."""
import numpy as np
import pytest

from conftest import have_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")]


class LocalHalo:
    """Ghost refresh for ranks living in one process (host-ordered device copies)."""

    def __init__(self, plans, device):
        import torch
        self.t = torch
        self.plans = plans
        self.recv_off = [np.concatenate([[0], np.cumsum(p.recv_counts)]) for p in plans]
        self.send = [[torch.as_tensor(ix, device=device) for ix in p.send_idx] for p in plans]

    def exchange(self, vecs):
        for h, ph in enumerate(self.plans):
            for r, pr in enumerate(self.plans):
                if r == h or not ph.recv_counts[r]:
                    continue
                a, b = self.recv_off[h][r], self.recv_off[h][r + 1]
                vals = vecs[r][:pr.q_loc].index_select(0, self.send[r][h])
                vecs[h][ph.q_loc + a:ph.q_loc + b] = vals


class LocalHaloAsync(LocalHalo):
    """The same ghost refresh on a side stream, registered with every rank's context
    (pslr_halo_pending): the horner calls that follow start their E y kernel and B solves
    while the copies run and wait for them only before the C_g y term."""

    def __init__(self, plans, device, ops):
        super().__init__(plans, device)
        self.ops = ops
        self.side = self.t.cuda.Stream()
        self.event = self.t.cuda.Event()

    def exchange(self, vecs):
        t = self.t
        self.side.wait_stream(t.cuda.current_stream())
        for v in vecs:
            v.record_stream(self.side)
        with t.cuda.stream(self.side):
            super().exchange(vecs)
            # delay the event well past the launch of the step's first kernels, so a step
            # that did not wait before C_g y would read stale ghosts
            t.cuda._sleep(2_000_000)
            self.event.record(self.side)
        for o in self.ops:
            o.halo_pending(self.event)


def _lockstep_apply(plans, ops, halo, b, p_global, m):
    import torch
    from paper_2002_00917_b200 import shard
    bl = [b[torch.as_tensor(shard.local_rows(pl, p_global), device=b.device)].contiguous() for pl in plans]
    first = [o.first(x) for o, x in zip(ops, bl)]
    s = sum(f[1] for f in first) if ops[0].r else None
    c = [o.mid(f[0], s.clone() if s is not None else f[1]) for o, f in zip(ops, first)]
    y = c
    if m > 0:
        halo.exchange(c)
        for k in range(m):
            out = [o.horner(yy, cc) for o, yy, cc in zip(ops, y, c)]
            if k < m - 1:
                halo.exchange(out)
            y = out
    z = torch.empty_like(b)
    for pl, o, x, yy in zip(plans, ops, bl, y):
        z[torch.as_tensor(shard.local_rows(pl, p_global), device=b.device)] = o.last(x, yy[:o.q].contiguous())
    return z


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("with_corr", [False, True])
def test_split_apply_matches_fused(world, with_corr):
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import shard, workloads
    A = workloads.laplacian3d(14, 14, 14, 0.5)
    m = 3
    cfg = pg.PslrConfig(num_subdomains=8, series_degree=m, rank=8 if with_corr else 0, droptol=1e-2, seed=0)
    P = pg.build(A, cfg)
    ps = P.system
    plans = [shard.plan_shard(ps, world, r) for r in range(world)]
    ops = [shard.DeviceShardOps(pl) for pl in plans]
    if with_corr:
        V, G = np.asarray(P.correction.V), P.correction.G
        for pl, o in zip(plans, ops):
            o.set_correction(torch.as_tensor(np.ascontiguousarray(V[pl.ifc_lo:pl.ifc_hi]), device="cuda"), G)
    halo = LocalHalo(plans, "cuda")
    b = torch.as_tensor(np.random.default_rng(5).standard_normal(ps.n), device="cuda")
    z = _lockstep_apply(plans, ops, halo, b, ps.p, m).cpu().numpy()
    z_ref = P.apply(b).cpu().numpy()
    if with_corr:
        assert np.linalg.norm(z - z_ref) <= 1e-12 * np.linalg.norm(z_ref)
    else:
        np.testing.assert_array_equal(z, z_ref)
    if world > 1:
        assert sum(pl.nghost for pl in plans) > 0  # the halo was exercised


@pytest.mark.parametrize("world", [2, 4])
def test_split_apply_halo_overlapped_with_interior_phase(world):
    """pslr_halo_pending: the ghosts of y arrive on a side stream (late: the exchange is
    followed by a device sleep) while the Horner step's E y kernel and B solves already run;
    only the C_g y term waits.  Bit-exact against the fused apply (correction off), so a
    step that read the ghosts early would fail."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import shard, workloads
    A = workloads.laplacian3d(14, 14, 14, 0.5)
    m = 3
    P = pg.build(A, pg.PslrConfig(num_subdomains=8, series_degree=m, rank=0, droptol=1e-2, seed=0))
    ps = P.system
    plans = [shard.plan_shard(ps, world, r) for r in range(world)]
    ops = [shard.DeviceShardOps(pl) for pl in plans]
    assert sum(pl.nghost for pl in plans) > 0
    b = torch.as_tensor(np.random.default_rng(5).standard_normal(ps.n), device="cuda")
    z_ref = P.apply(b)
    for _ in range(3):  # repeated: buffers of the previous apply are reused
        z = _lockstep_apply(plans, ops, LocalHaloAsync(plans, "cuda", ops), b, ps.p, m)
        assert torch.equal(z, z_ref)
    # a registration is consumed by one call; clearing it is allowed
    ops[0].halo_pending(None)
    z = _lockstep_apply(plans, ops, LocalHalo(plans, "cuda"), b, ps.p, m)
    assert torch.equal(z, z_ref)


def test_sharded_arnoldi_matches_build():
    """sharded_arnoldi over a 1-rank 'process group' of the local halo type == the device
    Arnoldi of build() (same operator, CGS2 order; sums differ only in rounding)."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import shard, workloads
    A = workloads.laplacian3d(12, 12, 12, 0.5)
    cfg = pg.PslrConfig(num_subdomains=4, series_degree=3, rank=6, droptol=1e-2, seed=0)
    P = pg.build(A, cfg)
    plan = shard.plan_shard(P.system, 1, 0)
    ops = shard.DeviceShardOps(plan)

    class OneRank:
        t = torch

        def exchange(self, v):
            return v

        def allreduce(self, x):
            return x

        def dot(self, a, b):
            return (a * b).sum().reshape(1)

    V, H, r = shard.sharded_arnoldi(ops, OneRank(), P.system.q, 0, 3, 6, seed=0)
    assert r == P.correction.rank
    assert np.allclose(H, P.correction.H, rtol=1e-9, atol=1e-12)
    assert np.allclose(V.cpu().numpy(), np.asarray(P.correction.V), rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("flexible", [False, True])
def test_sharded_gmres_one_rank_matches_device_gmres(flexible):
    """shard.sharded_gmres on a one-rank sharding (device ops, no process group needed)
    == the fused device GMRES / FGMRES (pslr_gmres): iterations within +-2, histories
    to 1e-6 (reduction order differs)."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import shard, workloads
    from paper_2002_00917_b200.krylov import gmres_device
    A = workloads.laplacian3d(16, 16, 16, 0.5)
    m = 3
    cfg = pg.PslrConfig(num_subdomains=8, series_degree=m, rank=8, droptol=1e-2, seed=0)
    P = pg.build(A, cfg)
    ps = P.system
    b = ps.matrix @ np.random.default_rng(0).standard_normal(ps.n)
    x_ref, rep = gmres_device(P, b, tol=1e-8, maxit=80, restart=20, flexible=flexible)
    plan = shard.plan_shard(ps, 1, 0)
    ops = shard.DeviceShardOps(plan)
    ops.set_correction(torch.as_tensor(np.ascontiguousarray(P.correction.V), device="cuda"), P.correction.G)
    halo = shard.Halo(plan, "cuda")
    SP = shard.ShardedPreconditioner(plan, ops, halo, m)
    x, conv, its, rel, hist = shard.sharded_gmres(SP, torch.as_tensor(b, device="cuda"), tol=1e-8,
                                                  maxit=80, restart=20, flexible=flexible)
    assert abs(its - rep.iterations) <= 2
    k = min(len(hist), len(rep.history))
    assert np.allclose(np.asarray(hist[:k]), np.asarray(rep.history[:k]), rtol=1e-6, atol=1e-14)
    assert conv == rep.converged


@pytest.mark.parametrize("world", [1, 2, 4])
def test_split_apply2_matches_split_apply(world):
    """The two-vector split apply (pslr_apply2_*: one launch sequence and one halo per step
    for both vectors, interleaved interface vectors with ghosts) == the single-vector split
    apply of each vector, bit for bit, through ShardedPreconditioner.apply2 on a lockstep
    sharding (the halo object only sees 2-column tensors)."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import shard, workloads
    A = workloads.laplacian3d(14, 14, 14, 0.5)
    m = 3
    cfg = pg.PslrConfig(num_subdomains=8, series_degree=m, rank=8, droptol=1e-2, seed=0)
    P = pg.build(A, cfg)
    ps = P.system
    plans = [shard.plan_shard(ps, world, r) for r in range(world)]
    ops = [shard.DeviceShardOps(pl) for pl in plans]
    V, G = np.asarray(P.correction.V), P.correction.G
    for pl, o in zip(plans, ops):
        o.set_correction(torch.as_tensor(np.ascontiguousarray(V[pl.ifc_lo:pl.ifc_hi]), device="cuda"), G)
    halo = LocalHalo(plans, "cuda")
    rng = np.random.default_rng(9)
    B = [torch.as_tensor(rng.standard_normal(ps.n), device="cuda") for _ in range(2)]
    z1 = [_lockstep_apply(plans, ops, halo, b, ps.p, m) for b in B]
    # lockstep apply2: the same orchestration on (q, 2) / (2, r) tensors
    rows = [torch.as_tensor(shard.local_rows(pl, ps.p), device="cuda") for pl in plans]
    b2 = [torch.stack([B[0][r_], B[1][r_]]).contiguous() for r_ in rows]
    first = [o.first2(x) for o, x in zip(ops, b2)]
    s = sum(f[1] for f in first)
    c = [o.mid2(f[0], s.clone()) for o, f in zip(ops, first)]
    y = c
    halo.exchange(c)
    for k in range(m):
        out = [o.horner2(yy, cc) for o, yy, cc in zip(ops, y, c)]
        if k < m - 1:
            halo.exchange(out)
        y = out
    z2 = torch.empty((2, ps.n), dtype=torch.float64, device="cuda")
    for r_, o, x, yy in zip(rows, ops, b2, y):
        z2[:, r_] = o.last2(x, yy[:o.q].contiguous())
    for v in range(2):
        assert torch.equal(z2[v], z1[v]), v
    # and the ShardedPreconditioner entry point on a one-rank sharding
    if world == 1:
        SP = shard.ShardedPreconditioner(plans[0], ops[0], shard.Halo(plans[0], "cuda"), m)
        zz = SP.apply2(b2[0])
        assert torch.equal(zz[0], SP.apply(b2[0][0].contiguous()))
        assert torch.equal(zz[1], SP.apply(b2[0][1].contiguous()))


def test_native_comm_world1_apply_err_arnoldi_gmres_cg():
    """The C-ABI multi-GPU route (pslr_comm_init + pslr_ctx_set_halo, include/pslr.h) on a
    one-rank NCCL communicator: pslr_apply / pslr_apply_Err / pslr_arnoldi / pslr_gmres /
    pslr_cg on the rank-local context run the sharded sequence inside libpslr (allreduces
    and halos are the world-1 no-ops) and must equal the fused context's results: apply and
    E_rr bit-exact, Arnoldi V/H to 1e-12, GMRES / CG iterations and histories identical."""
    import ctypes
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib, shard, workloads
    from paper_2002_00917_b200.krylov import cg_device, gmres_device
    A = workloads.laplacian3d(14, 12, 10, 0.3)
    m, r = 3, 8
    P = pg.build(A, pg.PslrConfig(num_subdomains=6, series_degree=m, rank=r))
    ps = P.system
    plan = shard.plan_shard(ps, 1, 0)
    ops = shard.DeviceShardOps(plan)
    shard.attach_nccl(ops, plan, shard.nccl_unique_id())
    V = torch.as_tensor(np.ascontiguousarray(P.correction.V), device="cuda")
    ops.set_correction(V, P.correction.G)
    h, st = ops.dev.handle, ops.dev.stream()
    b = torch.as_tensor(np.random.default_rng(0).standard_normal(ps.n), device="cuda")
    z = torch.empty_like(b)
    _lib.check(_lib.fns["pslr_apply"](h, m, b.data_ptr(), z.data_ptr(), st))
    assert torch.equal(z, P.apply(b))
    v = torch.as_tensor(np.random.default_rng(1).standard_normal(ps.q), device="cuda")
    e = torch.empty_like(v)
    _lib.check(_lib.fns["pslr_apply_Err"](h, m, v.data_ptr(), e.data_ptr(), st))
    assert torch.equal(e, pg.apply_Err(P.ctx, m, v))
    # Arnoldi through the communicator context == the build's device Arnoldi
    from paper_2002_00917_b200.lowrank import _start_vector
    v0 = np.ascontiguousarray(_start_vector(ps.q, 0))
    Vd = torch.empty((ps.q, r), dtype=torch.float64, device="cuda")
    H = np.zeros((r, r))
    ro = ctypes.c_int64()
    _lib.check(_lib.fns["pslr_arnoldi"](h, m, r, v0.ctypes.data, Vd.data_ptr(), H.ctypes.data, ctypes.byref(ro), st))
    assert ro.value == P.correction.rank
    assert np.abs(Vd.cpu().numpy() - P.correction.V).max() <= 1e-12
    assert np.abs(H - P.correction.H).max() <= 1e-12 * np.abs(P.correction.H).max()
    # GMRES and CG: the Python wrappers on a preconditioner-like view of the rank context
    bb = torch.as_tensor(ps.matrix @ np.random.default_rng(2).standard_normal(ps.n), device="cuda")

    class View:  # what gmres_device / cg_device read from a preconditioner
        device, series_degree, correction, system = ops.dev, m, P.correction, ps
    ops.dev._bound = P.correction  # the correction is already on the rank context
    for flexible in (False, True):
        x1, r1 = gmres_device(P, bb, tol=1e-8, maxit=60, restart=20, flexible=flexible)
        x2, r2 = gmres_device(View, bb, tol=1e-8, maxit=60, restart=20, flexible=flexible)
        assert r1.iterations == r2.iterations and r1.history == r2.history
        assert torch.equal(x1, x2)
    Q = pg.build(workloads.laplacian3d(10, 10, 9, 0.0), pg.PslrConfig(num_subdomains=4, series_degree=3, rank=0))
    qplan = shard.plan_shard(Q.system, 1, 0)
    qops = shard.DeviceShardOps(qplan)
    shard.attach_nccl(qops, qplan, shard.nccl_unique_id())

    class QView:
        device, series_degree, correction, system = qops.dev, 3, Q.correction, Q.system
    qops.dev._bound = Q.correction
    bq = torch.as_tensor(Q.system.matrix @ np.random.default_rng(3).standard_normal(Q.system.n), device="cuda")
    x1, r1 = cg_device(Q, bq, tol=1e-8)
    x2, r2 = cg_device(QView, bq, tol=1e-8)
    assert r1.converged and r1.iterations == r2.iterations and r1.history == r2.history


@pytest.mark.parametrize("overlap", ["1", "0"])
def test_native_comm_world1_pipelines_two_vectors(overlap, monkeypatch):
    """(overlap: PSLR_HALO_OVERLAP, read by pslr_comm_init — the halo on the context's
    communication stream, consumed before the C_g y term, or stream-ordered.)
    The bench's N>1 data plane on one rank: clones of the rank-local context, each with
    its OWN one-rank communicator (pslr_comm_init on a clone), run pslr_apply_multi with two
    right-hand sides (op_apply2_sharded: paired halos, one allreduce of 2r) concurrently on
    their own streams; every vector equals the fused single-vector apply bit for bit."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib, shard, workloads
    A = workloads.laplacian3d(14, 12, 10, 0.3)
    m, r = 3, 8
    P = pg.build(A, pg.PslrConfig(num_subdomains=6, series_degree=m, rank=r))
    ps = P.system
    plan = shard.plan_shard(ps, 1, 0)
    ops = shard.DeviceShardOps(plan)
    ops.set_correction(torch.as_tensor(np.ascontiguousarray(P.correction.V), device="cuda"), P.correction.G)
    ctxs = [ops.dev] + [ops.dev.clone() for _ in range(2)]
    monkeypatch.setenv("PSLR_HALO_OVERLAP", overlap)
    for c in ctxs:
        shard.attach_nccl_ctx(c, plan, shard.nccl_unique_id())
    streams = [torch.cuda.Stream() for _ in ctxs]
    B = torch.as_tensor(np.random.default_rng(5).standard_normal((6, ps.n)), device="cuda")
    Z = torch.empty_like(B)
    torch.cuda.synchronize()
    for j, c in enumerate(ctxs):
        _lib.check(_lib.fns["pslr_apply_multi"](c.handle, m, 2, B[2 * j].data_ptr(), Z[2 * j].data_ptr(),
                                                streams[j].cuda_stream))
    torch.cuda.synchronize()
    for v in range(6):
        assert torch.equal(Z[v], P.apply(B[v]))
    # an odd count: the pair through the two-vector path, the last vector alone
    Z3 = torch.empty((3, ps.n), dtype=torch.float64, device="cuda")
    _lib.check(_lib.fns["pslr_apply_multi"](ctxs[1].handle, m, 3, B[:3].contiguous().data_ptr(), Z3.data_ptr(),
                                            streams[1].cuda_stream))
    torch.cuda.synchronize()
    for v in range(3):
        assert torch.equal(Z3[v], P.apply(B[v]))
