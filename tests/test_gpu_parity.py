"""GPU parity: the sm_100a hot path (through the C-ABI) against the reference's
golden outputs and the CPU oracle on the same inputs.

Bars (written per assertion):
  * bit-exact: block solves (B, C0), every SpMV, apply_Es, apply_S, the Horner
    series and E_rr(m) — the device reproduces scipy's per-row operation order;
  * 1e-10 relative 2-norm (north star) for the full apply with the reference's
    (V, H, G) injected — observed ~1e-16: only the rank-r BLAS reductions differ;
  * GMRES iterations within +-2 of the reference (SURVEY §8d rule; both-fail-at-maxit
    for cfg1).
"""

import numpy as np
import pytest

from conftest import SMALL_APPLY_CASES, csr_from, csr_sha, golden, have_cuda, load_npz

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")]

G = golden()


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


_CACHE = {}


def _build(name):
    if name not in _CACHE:
        import paper_2002_00917_b200 as pg
        meta = G["apply"][name]
        d = load_npz(f"apply_{name}.npz")
        A = csr_from(d, "A")
        cfg = pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"],
                            droptol=meta["droptol"], seed=meta["seed"])
        _CACHE[name] = (pg.build(A, cfg), meta, d, A)
    return _CACHE[name]


@pytest.mark.parametrize("name", SMALL_APPLY_CASES)
def test_device_operators_bitexact(name):
    import paper_2002_00917_b200 as pg
    P, meta, d, A = _build(name)
    ctx = P.ctx
    for key, M in (("LB", ctx.b_ilu.L), ("UB", ctx.b_ilu.U), ("LC", ctx.c0_ilu.L), ("UC", ctx.c0_ilu.U)):
        assert csr_sha(M) == meta[key + "_sha"], key
    # bit-exact against the reference's own outputs (tests/golden)
    np.testing.assert_array_equal(pg.solve_B(ctx, d["f"]), d["solve_B"])
    if P.system.q:
        m = meta["m"]
        np.testing.assert_array_equal(pg.solve_C0(ctx, d["v"]), d["solve_C0"])
        np.testing.assert_array_equal(pg.apply_Es(ctx, d["v"]), d["apply_Es"])
        np.testing.assert_array_equal(pg.apply_neumann(ctx, m, d["v"]), d["apply_neumann"])
        np.testing.assert_array_equal(pg.apply_Err(ctx, m, d["v"]), d["apply_Err"])
    # SpMV of the reordered A (cli.py:137): scipy csr_matvec order
    x = np.random.default_rng(3).standard_normal(P.system.n)
    np.testing.assert_array_equal(P.matvec(x), P.system.matrix @ x)


@pytest.mark.parametrize("name", SMALL_APPLY_CASES)
def test_device_apply_S_matches_oracle(name):
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    P, meta, d, A = _build(name)
    if not P.system.q:
        pytest.skip("no interface")
    ps = P.system
    octx = O.Context(O.System(ps.matrix, O.Perm(ps.perm.forward, ps.perm.inverse), ps.num_parts,
                              ps.p, ps.q, ps.interior_sizes, ps.interface_sizes, ps.B, ps.E, ps.F, ps.C),
                     O.BlockFactors([], P.ctx.b_ilu.offsets, P.ctx.b_ilu.L, P.ctx.b_ilu.U),
                     O.BlockFactors([], P.ctx.c0_ilu.offsets, P.ctx.c0_ilu.L, P.ctx.c0_ilu.U),
                     P.ctx.C0, P.ctx.Cg)
    np.testing.assert_array_equal(pg.apply_S(P.ctx, d["v"]), O.apply_S(octx, d["v"]))


@pytest.mark.parametrize("name", SMALL_APPLY_CASES)
def test_device_apply_with_reference_correction(name):
    """Alg. 3.2 with the reference's (V, H, G) injected: <= 1e-10 relative (north star)."""
    import paper_2002_00917_b200 as pg
    P, meta, d, A = _build(name)
    Q = pg.with_correction(P, d["V"], d["H"], d["G"])
    z = Q.apply(d["b"])
    assert _rel(z, d["apply"]) <= 1e-10
    assert _rel(Q.apply_original(d["b"]), d["apply_original"]) <= 1e-10
    if P.system.q and Q.correction.rank:
        assert _rel(pg.apply_correction(Q.correction, d["v"]), d["apply_correction"]) <= 1e-12
    # zero-copy CUDA-tensor path gives the same bits as the numpy path
    import torch
    zt = Q.apply(torch.from_numpy(d["b"]).cuda())
    np.testing.assert_array_equal(zt.cpu().numpy(), z)


@pytest.mark.parametrize("name", [c for c in SMALL_APPLY_CASES if c != "cfg1"])
def test_device_arnoldi_matches_reference(name):
    """Device Arnoldi on E_rr(m) reproduces the reference V, H (well-conditioned cases)."""
    P, meta, d, A = _build(name)
    r = meta["achieved_rank"]
    assert P.correction.rank == r
    if r:
        assert _rel(P.correction.H, d["H"]) <= 1e-8
        assert _rel(P.correction.V, d["V"]) <= 1e-8
        assert _rel(P.apply(d["b"]), d["apply"]) <= 1e-8


def test_device_arnoldi_cfg1_orthonormal():
    """cfg1: E_rr(3) has spectral radius ~778, so V drifts ~1e-4 from the reference
    (SURVEY §0.4); check the Arnoldi contract instead and judge end-to-end in GMRES."""
    P, meta, d, A = _build("cfg1")
    V, H = P.correction.V, P.correction.H
    assert np.max(np.abs(V.T @ V - np.eye(V.shape[1]))) <= 1e-12
    assert np.max(np.abs(np.tril(H, -2))) == 0.0
    assert _rel(H, d["H"]) <= 1e-2


def test_device_determinism():
    """TestDeterminism (test_preconditioner.py:126-136): bitwise-identical rebuilds/applies."""
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    A = O.laplacian3d(5, 5, 5, shift=0.1)
    cfg = pg.PslrConfig(num_subdomains=4, rank=6, seed=7)
    P1, P2 = pg.build(A, cfg), pg.build(A, cfg)
    np.testing.assert_array_equal(P1.correction.V, P2.correction.V)
    np.testing.assert_array_equal(P1.correction.G, P2.correction.G)
    b = np.random.default_rng(8).standard_normal(A.shape[0])
    np.testing.assert_array_equal(P1.apply_original(b), P2.apply_original(b))


def test_length_checked():
    import paper_2002_00917_b200 as pg
    from conftest import lap1d
    P = pg.build(lap1d(10), pg.PslrConfig(num_subdomains=2, rank=2))
    with pytest.raises(ValueError):
        P.apply(np.ones(11))
    with pytest.raises(ValueError):
        pg.solve_C0(P.ctx, np.ones(P.system.q + 1))


def test_empty_interior_blocks():
    """Ragged partitions: a 1D Laplacian of 12 vertices in 6 subdomains leaves four
    subdomains with NO interior rows (interior sizes [1,0,0,0,0,1], interfaces
    [1,2,2,2,2,1]); the device apply (oracle correction injected) matches the oracle, and
    GMRES converges as in the reference driver."""
    import scipy.sparse as sp
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    A = sp.diags([-np.ones(11), 2 * np.ones(12), -np.ones(11)], [-1, 0, 1], format="csr")
    OP = O.build(A, 6, 2, 2)
    assert list(OP.system.interior_sizes) == [1, 0, 0, 0, 0, 1]
    P = pg.build(A, pg.PslrConfig(num_subdomains=6, series_degree=2, rank=2))
    Q = pg.with_correction(P, OP.corr.V, OP.corr.H, OP.corr.G)
    b = np.random.default_rng(0).standard_normal(12)
    assert _rel(Q.apply(b), OP.apply(b)) <= 1e-12
    np.testing.assert_array_equal(pg.solve_B(P.ctx, b[:P.system.p]), O.solve_B(OP.ctx, b[:P.system.p]))
    x, rep = pg.gmres(P.matvec_original, P.apply_original, A @ np.ones(12), tol=1e-10)
    assert rep.converged and np.allclose(x, np.ones(12), atol=1e-8)


def test_single_subdomain_ilu_only():
    """q == 0 path (test_preconditioner.py:69-76)."""
    import paper_2002_00917_b200 as pg
    from conftest import lap1d
    A = lap1d(30)
    P = pg.build(A, pg.PslrConfig(num_subdomains=1, droptol=0.0))
    assert P.system.q == 0
    b = np.random.default_rng(5).standard_normal(30)
    ref = np.linalg.solve(A.toarray(), b)
    assert _rel(P.apply_original(b), ref) <= 1e-10


# ---------------------------------------------------------------- GMRES on the device
def _solve(P, A, tol, maxit, restart, seed=0, flexible=False):
    import paper_2002_00917_b200 as pg
    b = A @ np.random.default_rng(seed).standard_normal(A.shape[0])
    bp = b[P.system.perm.inverse]
    x, rep = pg.gmres(P.matvec, P.apply, bp, tol=tol, maxit=maxit, restart=restart, flexible=flexible)
    return x, rep, bp


def test_gmres_crit11_13_iterations():
    P, meta, d, A = _build("crit11")
    x, rep, bp = _solve(P, A, 1e-8, 500, 0)
    ref = G["gmres"]["crit11"]
    assert rep.converged and abs(rep.iterations - ref["iterations"]) <= 2
    assert len(rep.history) == rep.iterations + 1 and rep.history[0] == 1.0
    assert np.linalg.norm(bp - P.system.matrix @ x) <= 1e-8 * np.linalg.norm(bp)


def test_gmres_cfg1_fails_at_maxit_like_reference():
    P, meta, d, A = _build("cfg1")
    Q = __import__("paper_2002_00917_b200").with_correction(P, d["V"], d["H"], d["G"])
    x, rep, bp = _solve(Q, A, 1e-6, 500, 50)
    ref = G["gmres"]["cfg1_gmres50"]
    assert not rep.converged and rep.iterations == 500 and len(rep.history) == 501
    h = np.array(rep.history[:50])
    hr = np.array(ref["history_first_cycle"][:50])
    # E_rr(3) has spectral radius ~778 on cfg1: rounding differences in the
    # BLAS-ordered correction and CGS2 reductions grow along the cycle.  Bit-identical for
    # the first ~7 estimates, ~5e-3 relative by the end of the first cycle (measured).
    assert np.max(np.abs(h[:7] - hr[:7]) / hr[:7]) <= 1e-10
    assert np.max(np.abs(h - hr) / hr) <= 2e-2


@pytest.mark.parametrize("cfg,relres", [("cfg2", 1.56e-5), ("cfg3", 1.55e-3)])
def test_gmres_full_size_fails_at_maxit_like_reference(cfg, relres):
    """SURVEY §8d rule at BASELINE size: the reference fails at maxit 500 on cfg2
    (GMRES(50), relres 1.56e-5) and cfg3 (restart 50, stagnating at 1.55e-3);
    the device solve must fail at maxit too, at the same residual level."""
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import workloads
    wl = workloads.CONFIGS[cfg]
    A = wl.matrix()
    P = pg.build(A, wl.config())
    b = workloads.seeded_rhs(A, 0)
    x, rep = pg.gmres(P.matvec_original, P.apply_original, b, tol=wl.tol, maxit=wl.maxit,
                      restart=wl.restart, flexible=wl.flexible)
    assert not rep.converged and rep.iterations == wl.maxit and len(rep.history) == wl.maxit + 1
    true_rel = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
    assert abs(true_rel - relres) <= 0.02 * relres  # the survey quotes 3 significant digits
    assert abs(rep.final_relres - true_rel) <= 1e-6 * true_rel


@pytest.mark.parametrize("m,its", [(3, 4), (5, 3)])
def test_gmres_crit06_n2000_exact_factors(m, its):
    """Acceptance criterion 06 (test_acceptance.py:136-150; golden pkg/test_output.txt):
    1 x 8 x 250 Laplacian, s=5, EXACT factors (droptol 0), rank 15, full GMRES tol 1e-8,
    original space -> 4 iterations at m=3, 3 at m=5."""
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    A = O.laplacian3d(1, 8, 250, 0.0)
    P = pg.build(A, pg.PslrConfig(num_subdomains=5, series_degree=m, rank=15, droptol=0.0))
    b = A @ np.random.default_rng(0).standard_normal(A.shape[0])
    x, rep = pg.gmres(P.matvec_original, P.apply_original, b, tol=1e-8)
    assert rep.converged and abs(rep.iterations - its) <= 2
    assert np.linalg.norm(b - A @ x) <= 1e-8 * np.linalg.norm(b)


@pytest.mark.parametrize("rank,its", [(0, 136), (30, 145)])
def test_gmres_crit08_rank_dichotomy_counts(rank, its):
    """Acceptance criterion 08 (test_acceptance.py:169-183), the reference's known-red test:
    32^3 shift 0.16, s=35, m=3, seed 0, full GMRES tol 1e-8 — the reference converges in 136
    iterations at rank 0 (so its own criterion fails) and 145 at rank 30; the device path
    reproduces both counts (+-2)."""
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    A = O.laplacian3d(32, 32, 32, shift=0.16)
    P = pg.build(A, pg.PslrConfig(num_subdomains=35, series_degree=3, rank=rank, seed=0))
    b = A @ np.random.default_rng(0).standard_normal(A.shape[0])
    x, rep = pg.gmres(P.matvec_original, P.apply_original, b, tol=1e-8, maxit=500)
    assert rep.converged and abs(rep.iterations - its) <= 2


def test_gmres_twin_cfg3_hv1_21_iterations():
    """SURVEY §4 twin table: upwind 32^3, shift 0.2, hv = 1.0 (the other cell-Peclet
    reading), s=16, m=5, r=64, GMRES(50) tol 1e-6 -> 21 iterations (reference)."""
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import workloads
    A = workloads.upwind3d(32, 32, 32, 0.2, 1.0)
    P = pg.build(A, pg.PslrConfig(num_subdomains=16, series_degree=5, rank=64))
    b = workloads.seeded_rhs(A, 0)
    for flexible in (False, True):
        x, rep = pg.gmres(P.matvec_original, P.apply_original, b, tol=1e-6, maxit=500, restart=50,
                          flexible=flexible)
        assert rep.converged and abs(rep.iterations - 21) <= 2


@pytest.mark.parametrize("m", [3, 5])
def test_gmres_crit07(m):
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    A = O.laplacian3d(32, 32, 32, shift=0.16)
    P = pg.build(A, pg.PslrConfig(num_subdomains=35, series_degree=m, rank=15, seed=2))
    x, rep, bp = _solve(P, A, 1e-8, 500, 0, seed=2)
    ref = G["gmres"]["crit07"][f"{m}_reordered"]
    assert rep.converged and abs(rep.iterations - ref["iterations"]) <= 2


@pytest.mark.parametrize("twin,flexible", [("twin_cfg2", False), ("twin_cfg3", False),
                                           ("twin_cfg3", True)])
def test_gmres_twins(twin, flexible):
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    meta = G["apply"][twin]
    A = O.laplacian3d(32, 32, 32, shift=0.16) if twin == "twin_cfg2" else O.upwind3d(32, 32, 32, 0.2, 0.5)
    P = pg.build(A, pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"]))
    x, rep, bp = _solve(P, A, 1e-6, 500, 50, flexible=flexible)
    ref = G["gmres"][twin]
    assert rep.converged == ref["converged"] and abs(rep.iterations - ref["iterations"]) <= 2


def test_gmres_original_space_driver():
    """Acceptance-test driver form: gmres(P.matvec_original, P.apply_original, b)."""
    import paper_2002_00917_b200 as pg
    P, meta, d, A = _build("crit11")
    b = A @ np.random.default_rng(0).standard_normal(A.shape[0])
    x, rep = pg.gmres(P.matvec_original, P.apply_original, b, tol=1e-8)
    assert rep.converged and abs(rep.iterations - 13) <= 2
    assert np.linalg.norm(b - A @ x) <= 1e-8 * np.linalg.norm(b)


# ---------------------------------------------------------------- BASELINE-size parity
@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_full_size_apply_matches_oracle(cfg):
    """BASELINE sizes — cfg2 (64^3, s=16, m=3, r=32), cfg3 (128^3 upwind, s=64, m=5, r=64),
    cfg4 (2048^2 2D, s=128, m=5, r=128: up to 1421 + 2130 dependent levels per B solve),
    cfg5 (the bench workload: 128^3, s=32, m=3, r=64): device apply vs the oracle's on
    identical factors and correction state; solves bit-exact, apply <= 1e-10."""
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import workloads
    from oracle import pslr_oracle as O
    wl = workloads.CONFIGS[cfg]
    A = wl.matrix()
    P = pg.build(A, wl.config())
    ps = P.system
    octx = O.Context(O.System(ps.matrix, O.Perm(ps.perm.forward, ps.perm.inverse), ps.num_parts,
                              ps.p, ps.q, ps.interior_sizes, ps.interface_sizes, ps.B, ps.E, ps.F, ps.C),
                     O.BlockFactors([], P.ctx.b_ilu.offsets, P.ctx.b_ilu.L, P.ctx.b_ilu.U),
                     O.BlockFactors([], P.ctx.c0_ilu.offsets, P.ctx.c0_ilu.L, P.ctx.c0_ilu.U),
                     P.ctx.C0, P.ctx.Cg)
    corr = O.Correction(P.correction.V, P.correction.H, P.correction.G, P.correction.rank)
    OP = O.Preconditioner(ps, octx, wl.m, corr)
    rng = np.random.default_rng(0)
    b = rng.standard_normal(ps.n)
    f = rng.standard_normal(ps.p)
    np.testing.assert_array_equal(pg.solve_B(P.ctx, f), O.solve_B(octx, f))
    assert _rel(P.apply(b), OP.apply(b)) <= 1e-10
    # size-independent properties at full size: determinism and linearity
    z1 = P.apply(b)
    np.testing.assert_array_equal(z1, P.apply(b))
    b2 = rng.standard_normal(ps.n)
    assert _rel(P.apply(2.0 * b + b2), 2.0 * z1 + P.apply(b2)) <= 1e-10


def test_explicit_sd_layout_bitexact(monkeypatch):
    """The general U-segment layout (explicit sd / rcp arrays, used when a scaled diagonal
    is neither 1 nor 1 - 2^-53) gives the same bits as the flag layout."""
    import paper_2002_00917_b200 as pg
    name = "lap3d6_s4_dt1e-2"
    meta = G["apply"][name]
    d = load_npz(f"apply_{name}.npz")
    A = csr_from(d, "A")
    cfg = pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"],
                        droptol=meta["droptol"], seed=meta["seed"])
    monkeypatch.setenv("PSLR_EXPLICIT_SD", "1")
    P = pg.build(A, cfg)
    np.testing.assert_array_equal(pg.solve_B(P.ctx, d["f"]), d["solve_B"])
    np.testing.assert_array_equal(pg.apply_neumann(P.ctx, meta["m"], d["v"]), d["apply_neumann"])


def test_ey_prepass_and_all_sm_kernel_bitexact(monkeypatch):
    """The work moved off the step kernel's critical blocks gives the same bits as doing it
    inside: the E y / C_g y pre-step kernel (vs PSLR_EY_ALLSM=0), the split interface phase
    (vs PSLR_SPLIT_IFACE=0) and the shared-memory far-ring (vs PSLR_FAR_SLOTS=0) — apply_Es,
    the Horner series, E_rr and the full apply (one and two vectors per call)."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib
    name = "lap3d6_s4_dt1e-2"
    meta = G["apply"][name]
    d = load_npz(f"apply_{name}.npz")
    A = csr_from(d, "A")
    cfg = pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"],
                        droptol=meta["droptol"], seed=meta["seed"])
    out = []
    for env in ("1", "0"):
        monkeypatch.setenv("PSLR_EY_ALLSM", env)
        monkeypatch.setenv("PSLR_SPLIT_IFACE", env)  # the interface phase as its own all-SM kernel
        monkeypatch.setenv("PSLR_FAR_SLOTS", "4096" if env == "1" else "0")  # far-ring vs global far reads
        P = pg.build(A, cfg)
        n = P.system.n
        B2 = torch.from_numpy(np.random.default_rng(3).standard_normal((2, n))).cuda()
        Z2 = torch.empty_like(B2)
        P.device.ensure_correction(P.correction)
        _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, meta["m"], 2, B2.data_ptr(), Z2.data_ptr(),
                                                P.device.stream()))
        torch.cuda.synchronize()
        out.append((pg.apply_Es(P.ctx, d["v"]), pg.apply_neumann(P.ctx, meta["m"], d["v"]),
                    pg.apply_Err(P.ctx, meta["m"], d["v"]), P.apply(d["b"]), Z2.cpu().numpy()))
    for a, b in zip(*out):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(out[0][0], d["apply_Es"])
    np.testing.assert_array_equal(out[0][1], d["apply_neumann"])


@pytest.mark.parametrize("threads", ["128", "480"])
@pytest.mark.parametrize("alt", ["0", "3"])
def test_consumer_thread_count_and_warp_groups_bitexact(threads, alt, monkeypatch):
    """The step kernel's two instantiations (480 and 128 consumer threads, chosen per system
    from the rows per level; PSLR_STEP_THREADS_RT forces one) and the packer's alternating
    warp groups (PSLR_ALT_GROUPS) only change which thread owns a row: every operator is
    the reference's output bit for bit in each combination, one and two vectors per call."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib
    name = "lap3d6_s4_dt1e-2"
    meta = G["apply"][name]
    d = load_npz(f"apply_{name}.npz")
    A = csr_from(d, "A")
    cfg = pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"],
                        droptol=meta["droptol"], seed=meta["seed"])
    ref = pg.build(A, cfg)
    monkeypatch.setenv("PSLR_STEP_THREADS_RT", threads)
    monkeypatch.setenv("PSLR_ALT_GROUPS", alt)
    P = pg.build(A, cfg)
    np.testing.assert_array_equal(pg.solve_B(P.ctx, d["f"]), d["solve_B"])
    np.testing.assert_array_equal(pg.solve_C0(P.ctx, d["v"]), d["solve_C0"])
    np.testing.assert_array_equal(pg.apply_Es(P.ctx, d["v"]), d["apply_Es"])
    np.testing.assert_array_equal(pg.apply_neumann(P.ctx, meta["m"], d["v"]), d["apply_neumann"])
    np.testing.assert_array_equal(pg.apply_Err(P.ctx, meta["m"], d["v"]), d["apply_Err"])
    np.testing.assert_array_equal(P.apply(d["b"]), ref.apply(d["b"]))
    n = P.system.n
    B2 = torch.from_numpy(np.random.default_rng(3).standard_normal((2, n))).cuda()
    Z2 = torch.empty_like(B2)
    P.device.ensure_correction(P.correction)
    _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, meta["m"], 2, B2.data_ptr(), Z2.data_ptr(),
                                            P.device.stream()))
    torch.cuda.synchronize()
    for v in range(2):
        assert torch.equal(Z2[v], ref.apply(B2[v].contiguous()))


def _oracle_ctx(P):
    from oracle import pslr_oracle as O
    ps = P.system
    return O.Context(O.System(ps.matrix, O.Perm(ps.perm.forward, ps.perm.inverse), ps.num_parts,
                              ps.p, ps.q, ps.interior_sizes, ps.interface_sizes, ps.B, ps.E, ps.F, ps.C),
                     O.BlockFactors([], P.ctx.b_ilu.offsets, P.ctx.b_ilu.L, P.ctx.b_ilu.U),
                     O.BlockFactors([], P.ctx.c0_ilu.offsets, P.ctx.c0_ilu.L, P.ctx.c0_ilu.U),
                     P.ctx.C0, P.ctx.Cg)


@pytest.mark.parametrize("m", [0, 1, 5, 8])
def test_series_degree_edge_cases(m):
    """Alg. 3.2 at series degrees other than the configs' 3/5 (m = 0: no Horner step):
    the apply against the oracle with the same factors and correction (1e-10), and the
    correction-free operators bit-exact (preconditioner.py:79-93, schur.py:89-112)."""
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    P, meta, d, A = _build("lap3d6_s4_dt1e-2")
    octx = _oracle_ctx(P)
    corr = P.correction
    OP = O.Preconditioner(octx.system, octx, m, O.Correction(np.asarray(corr.V), corr.H, corr.G, corr.rank))
    b = np.random.default_rng(7).standard_normal(P.system.n)
    P.device.ensure_correction(corr)
    z = P.device.vec_op("pslr_apply", b, P.system.n, P.system.n, m)
    assert _rel(z, OP.apply(b)) <= 1e-10
    v = np.random.default_rng(8).standard_normal(P.system.q)
    np.testing.assert_array_equal(pg.apply_neumann(P.ctx, m, v), O.apply_neumann(octx, m, v))
    np.testing.assert_array_equal(pg.apply_Err(P.ctx, m, v), O.apply_Err(octx, m, v))


def test_rank_zero_apply_bitexact():
    """rank = 0 (no low-rank correction, lowrank.py:98-105 identity): every step of the
    apply is a correction-free operator, so it is bit-exact with the oracle."""
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    meta = G["apply"]["lap3d6_s4_dt1e-2"]
    d = load_npz("apply_lap3d6_s4_dt1e-2.npz")
    A = csr_from(d, "A")
    P = pg.build(A, pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=0,
                                  droptol=meta["droptol"], seed=meta["seed"]))
    assert P.correction.rank == 0
    octx = _oracle_ctx(P)
    OP = O.Preconditioner(octx.system, octx, meta["m"], O.Correction(np.zeros((P.system.q, 0)),
                                                                      np.zeros((0, 0)), np.zeros((0, 0)), 0))
    b = np.random.default_rng(9).standard_normal(P.system.n)
    np.testing.assert_array_equal(P.apply(b), OP.apply(b))


def test_gmres_nonfinite_raises():
    """krylov.py:81-82: a non-finite recurrence raises ArithmeticError on the device path too."""
    import paper_2002_00917_b200 as pg
    P, meta, d, A = _build("lap3d6_s4_dt1e-2")
    b = np.random.default_rng(0).standard_normal(P.system.n)
    b[3] = np.nan
    with pytest.raises(ArithmeticError):
        pg.gmres(P.matvec, P.apply, b, tol=1e-8, maxit=20)


def test_clones_run_concurrently_bitexact():
    """pslr_ctx_clone: clones share the factors / correction and own their scratch, so
    independent applies on separate streams give the bits of the sequential apply."""
    import torch
    from paper_2002_00917_b200 import _lib
    P, meta, d, A = _build("lap3d6_s4_dt1e-2")
    P.device.ensure_correction(P.correction)
    clones = [P.device.clone() for _ in range(3)]
    devs = [P.device] + clones
    n, m = P.system.n, P.series_degree
    rng = np.random.default_rng(11)
    bs = [torch.as_tensor(rng.standard_normal(n), device="cuda") for _ in range(8)]
    ref = [P.apply(b).clone() for b in bs]
    streams = [torch.cuda.Stream() for _ in devs]
    outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in bs]
    torch.cuda.synchronize()
    for k, b in enumerate(bs):
        j = k % len(devs)
        _lib.check(_lib.fns["pslr_apply"](devs[j].handle, m, b.data_ptr(), outs[k].data_ptr(),
                                          streams[j].cuda_stream))
    torch.cuda.synchronize()
    for k in range(len(bs)):
        assert torch.equal(outs[k], ref[k])
    with pytest.raises(ValueError):  # clones share the correction: it cannot be reset on them
        clones[0].set_correction(None, None)


@pytest.mark.parametrize("name,nv", [("lap3d6_s4_dt1e-2", 2), ("lap3d6_s4_dt1e-2", 3), ("upw3d8_s4", 2),
                                     ("cfg1", 2), ("crit11", 4)])
def test_apply_multi_bitexact(name, nv):
    """pslr_apply_multi: pairs of vectors share each launch (interleaved right-hand sides);
    every vector's result is the single-vector apply bit for bit."""
    import torch
    from paper_2002_00917_b200 import _lib
    P, meta, d, A = _build(name)
    P.device.ensure_correction(P.correction)
    n = P.system.n
    B = torch.as_tensor(np.random.default_rng(12).standard_normal((nv, n)), device="cuda").contiguous()
    Z = torch.empty_like(B)
    _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, P.series_degree, nv, B.data_ptr(), Z.data_ptr(),
                                            P.device.stream()))
    for v in range(nv):
        np.testing.assert_array_equal(Z[v].cpu().numpy(), P.apply(B[v]).cpu().numpy())


def test_apply_multi_host_async_bitexact():
    """pslr_apply_multi_host_async (pinned host buffers, pairs through one launch sequence,
    the odd vector through the single-vector path) == pslr_apply per vector, on a clone
    context and its own stream."""
    import torch
    from paper_2002_00917_b200 import _lib
    P, meta, d, A = _build("cfg1")
    P.device.ensure_correction(P.correction)
    n, nv = P.system.n, 3
    c = P.device.clone()
    st = torch.cuda.Stream()
    B = torch.from_numpy(np.random.default_rng(13).standard_normal((nv, n))).pin_memory()
    Z = torch.empty((nv, n), dtype=torch.float64).pin_memory()
    _lib.check(_lib.fns["pslr_apply_multi_host_async"](c.handle, P.series_degree, nv, B.data_ptr(),
                                                       Z.data_ptr(), st.cuda_stream))
    st.synchronize()
    for v in range(nv):
        np.testing.assert_array_equal(Z[v].numpy(), P.apply(B[v].cuda()).cpu().numpy())
    del c


def _multi(P, m, B):
    import torch
    from paper_2002_00917_b200 import _lib
    Bt = torch.as_tensor(np.ascontiguousarray(B), device="cuda")
    Z = torch.empty_like(Bt)
    _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, m, Bt.shape[0], Bt.data_ptr(), Z.data_ptr(),
                                            P.device.stream()))
    return Z.cpu().numpy()


@pytest.mark.parametrize("m", [0, 1, 5])
def test_apply_multi_series_degrees(m):
    """Two vectors per launch at series degrees 0 (no Horner launch), 1 and 5: each vector
    equals the single-vector apply bit for bit."""
    P, meta, d, A = _build("lap3d6_s4_dt1e-2")
    P.device.ensure_correction(P.correction)
    n = P.system.n
    B = np.random.default_rng(20 + m).standard_normal((2, n))
    Z = _multi(P, m, B)
    for v in range(2):
        np.testing.assert_array_equal(Z[v], P.device.vec_op("pslr_apply", B[v], n, n, m))


def test_apply_multi_rank_zero_and_explicit_sd(monkeypatch):
    """Two vectors per launch with no low-rank correction (bit-exact with the oracle's
    apply) and with the explicit sd / rcp U layout (bit-exact with the flag layout)."""
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    meta = G["apply"]["lap3d6_s4_dt1e-2"]
    d = load_npz("apply_lap3d6_s4_dt1e-2.npz")
    A = csr_from(d, "A")
    P = pg.build(A, pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=0,
                                  droptol=meta["droptol"], seed=meta["seed"]))
    octx = _oracle_ctx(P)
    OP = O.Preconditioner(octx.system, octx, meta["m"], O.Correction(np.zeros((P.system.q, 0)),
                                                                      np.zeros((0, 0)), np.zeros((0, 0)), 0))
    B = np.random.default_rng(21).standard_normal((2, P.system.n))
    Z = _multi(P, meta["m"], B)
    for v in range(2):
        np.testing.assert_array_equal(Z[v], OP.apply(B[v]))
    monkeypatch.setenv("PSLR_EXPLICIT_SD", "1")
    Pe = pg.build(A, pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=0,
                                   droptol=meta["droptol"], seed=meta["seed"]))
    np.testing.assert_array_equal(_multi(Pe, meta["m"], B), Z)


def test_apply_multi_small_counts_and_errors():
    """nv = 0 is a no-op, nv = 1 is pslr_apply; negative nv / m are rejected (ValueError)."""
    import torch
    from paper_2002_00917_b200 import _lib
    P, meta, d, A = _build("lap3d6_s4_dt1e-2")
    P.device.ensure_correction(P.correction)
    n, m = P.system.n, meta["m"]
    B = np.random.default_rng(22).standard_normal((1, n))
    np.testing.assert_array_equal(_multi(P, m, B)[0], P.apply(B[0]))
    Z = torch.full((1, n), 7.0, dtype=torch.float64, device="cuda")
    Bt = torch.as_tensor(B, device="cuda")
    _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, m, 0, Bt.data_ptr(), Z.data_ptr(), P.device.stream()))
    assert bool((Z == 7.0).all())
    for bad_m, bad_nv in ((-1, 2), (m, -1)):
        with pytest.raises(ValueError):
            _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, bad_m, bad_nv, Bt.data_ptr(), Z.data_ptr(),
                                                    P.device.stream()))


# ---------------------------------------------------------------- randomized structure sweep
@pytest.mark.parametrize("seed,n,density,s,m,r,droptol", [
    (11, 300, 0.04, 3, 2, 6, 1e-2), (12, 500, 0.03, 5, 3, 8, 1e-3), (13, 700, 0.02, 8, 1, 4, 1e-2),
    (14, 400, 0.05, 4, 4, 10, 0.0), (15, 900, 0.015, 6, 3, 12, 1e-2), (16, 250, 0.08, 2, 2, 5, 1e-4),
])
def test_random_structures_bitexact(seed, n, density, s, m, r, droptol):
    """Nonsymmetric random sparse matrices (the reference helper, pkg/tests/conftest.py:25-29)
    with varied sizes, partitions, series degrees, ranks and drop tolerances: long and ragged
    ILUT rows (many slot groups per row), deep and shallow level structures, far
    dependencies.  Every device operator is bit-identical to the oracle on the same factors;
    the full apply with the oracle's correction injected to 1e-12."""
    import paper_2002_00917_b200 as pg
    from conftest import random_sparse
    from oracle import pslr_oracle as O
    A = random_sparse(n, density=density, seed=seed)
    P = pg.build(A, pg.PslrConfig(num_subdomains=s, series_degree=m, rank=r, droptol=droptol))
    ps = P.system
    octx = O.Context(O.System(ps.matrix, O.Perm(ps.perm.forward, ps.perm.inverse), ps.num_parts,
                              ps.p, ps.q, ps.interior_sizes, ps.interface_sizes, ps.B, ps.E, ps.F, ps.C),
                     O.BlockFactors([], P.ctx.b_ilu.offsets, P.ctx.b_ilu.L, P.ctx.b_ilu.U),
                     O.BlockFactors([], P.ctx.c0_ilu.offsets, P.ctx.c0_ilu.L, P.ctx.c0_ilu.U),
                     P.ctx.C0, P.ctx.Cg)
    rng = np.random.default_rng(seed)
    f = rng.standard_normal(ps.p)
    np.testing.assert_array_equal(pg.solve_B(P.ctx, f), O.solve_B(octx, f))
    if ps.q:
        v = rng.standard_normal(ps.q)
        np.testing.assert_array_equal(pg.solve_C0(P.ctx, v), O.solve_C0(octx, v))
        np.testing.assert_array_equal(pg.apply_Es(P.ctx, v), O.apply_Es(octx, v))
        np.testing.assert_array_equal(pg.apply_neumann(P.ctx, m, v), O.apply_neumann(octx, m, v))
        np.testing.assert_array_equal(pg.apply_Err(P.ctx, m, v), O.apply_Err(octx, m, v))
    corr = O.Correction(P.correction.V, P.correction.H, P.correction.G, P.correction.rank)
    OP = O.Preconditioner(ps, octx, m, corr)
    b = rng.standard_normal(ps.n)
    assert _rel(P.apply(b), OP.apply(b)) <= 1e-12
    B2 = np.ascontiguousarray(np.stack([b, rng.standard_normal(ps.n)]))
    import torch
    from paper_2002_00917_b200 import _lib
    Bd = torch.as_tensor(B2, device="cuda")
    Zd = torch.empty_like(Bd)
    _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, m, 2, Bd.data_ptr(), Zd.data_ptr(),
                                            P.device.stream()))
    torch.cuda.synchronize()
    assert torch.equal(Zd[0], P.apply(Bd[0].contiguous()))
