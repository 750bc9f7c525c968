"""GPU parity of the level-merged factors (PSLR_MERGE, pack.cpp merge_levels).

A merged row at an odd dependency level has its previous-level dependencies substituted,
so the level count halves; the operator is the reference's B^{-1} / C0^{-1} exactly, the
rounding is not (different summation).  Bars:
  * solves, E_s, the Neumann series and E_rr within 1e-12 relative of the reference's own
    outputs (observed ~1e-16);
  * the apply within 1e-10 relative 2-norm (north star) on the golden cases and at
    BASELINE sizes against the oracle on identical factors;
  * GMRES / FGMRES iterations within +-2 of the reference.
Modes: 2 = merged C0 factors (the product default), 3 = B and C0 (B merging is slower on
cfg5: DESIGN §9), 3 with every B level pair merged (PSLR_MERGE_W=0).
"""

import numpy as np
import pytest

from conftest import SMALL_APPLY_CASES, csr_from, golden, have_cuda, load_npz

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")]

G = golden()
MODES = [("2", None), ("3", None), ("3", "0")]


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _env(monkeypatch, mode, w):
    monkeypatch.setenv("PSLR_MERGE", mode)
    if w is None:
        monkeypatch.delenv("PSLR_MERGE_W", raising=False)
    else:
        monkeypatch.setenv("PSLR_MERGE_W", w)


def _build_case(name):
    import paper_2002_00917_b200 as pg
    meta = G["apply"][name]
    d = load_npz(f"apply_{name}.npz")
    A = csr_from(d, "A")
    cfg = pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"],
                        droptol=meta["droptol"], seed=meta["seed"])
    return pg.build(A, cfg), meta, d, A


@pytest.mark.parametrize("mode,w", MODES)
@pytest.mark.parametrize("name", SMALL_APPLY_CASES)
def test_merged_operators_match_reference(monkeypatch, name, mode, w):
    import paper_2002_00917_b200 as pg
    _env(monkeypatch, mode, w)
    P, meta, d, A = _build_case(name)
    ctx = P.ctx
    assert _rel(pg.solve_B(ctx, d["f"]), d["solve_B"]) <= 1e-12
    if P.system.q:
        m = meta["m"]
        assert _rel(pg.solve_C0(ctx, d["v"]), d["solve_C0"]) <= 1e-12
        assert _rel(pg.apply_Es(ctx, d["v"]), d["apply_Es"]) <= 1e-12
        # the series amplifies round-off by up to rho(E_s)^m (cfg1: ~778^3)
        tol = 1e-6 if name == "cfg1" else 1e-11
        assert _rel(pg.apply_neumann(ctx, m, d["v"]), d["apply_neumann"]) <= tol
        assert _rel(pg.apply_Err(ctx, m, d["v"]), d["apply_Err"]) <= tol
    Q = pg.with_correction(P, d["V"], d["H"], d["G"])
    tol = 1e-6 if name == "cfg1" else 1e-10
    assert _rel(Q.apply(d["b"]), d["apply"]) <= tol
    assert _rel(Q.apply_original(d["b"]), d["apply_original"]) <= tol


@pytest.mark.parametrize("mode,w", MODES)
def test_merged_depths_halve(monkeypatch, mode, w):
    """The merged factors' level counts: every C0 pair merges (ceil(depth / 2)); B merges
    only the pairs the width limit admits (all of them with PSLR_MERGE_W=0)."""
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    A = O.laplacian3d(16, 16, 16, shift=0.3)
    cfg = pg.PslrConfig(num_subdomains=4, series_degree=3, rank=8)
    monkeypatch.setenv("PSLR_MERGE", "0")
    i0 = pg.build(A, cfg).device.info()
    _env(monkeypatch, mode, w)
    i1 = pg.build(A, cfg).device.info()
    for f in ("LC", "UC"):
        assert i1["maxdepth_" + f] == (i0["maxdepth_" + f] + 1) // 2, f
    for f in ("LB", "UB"):
        if mode == "3" and w == "0":
            assert i1["maxdepth_" + f] == (i0["maxdepth_" + f] + 1) // 2, f
        else:
            assert (i0["maxdepth_" + f] + 1) // 2 <= i1["maxdepth_" + f] <= i0["maxdepth_" + f], f


@pytest.mark.parametrize("twin,flexible", [("twin_cfg2", False), ("twin_cfg3", True)])
def test_merged_gmres_twins(monkeypatch, twin, flexible):
    import paper_2002_00917_b200 as pg
    from oracle import pslr_oracle as O
    monkeypatch.setenv("PSLR_MERGE", "2")
    meta = G["apply"][twin]
    A = O.laplacian3d(32, 32, 32, shift=0.16) if twin == "twin_cfg2" else O.upwind3d(32, 32, 32, 0.2, 0.5)
    P = pg.build(A, pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"]))
    b = A @ np.random.default_rng(0).standard_normal(A.shape[0])
    bp = b[P.system.perm.inverse]
    x, rep = pg.gmres(P.matvec, P.apply, bp, tol=1e-6, maxit=500, restart=50, flexible=flexible)
    ref = G["gmres"][twin]
    assert rep.converged == ref["converged"] and abs(rep.iterations - ref["iterations"]) <= 2
    assert np.linalg.norm(bp - P.system.matrix @ x) <= 1e-6 * np.linalg.norm(bp)


def test_merged_two_vector_apply_matches_single(monkeypatch):
    """Two right-hand sides per launch (pslr_apply_multi) with merged factors: each vector
    is the single-vector merged apply bit for bit (same per-row arithmetic)."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib
    monkeypatch.setenv("PSLR_MERGE", "3")
    monkeypatch.setenv("PSLR_MERGE_W", "0")
    P, meta, d, A = _build_case("lap3d6_s4_dt1e-2")
    n = P.system.n
    rng = np.random.default_rng(5)
    b = torch.from_numpy(rng.standard_normal((2, n))).cuda()
    z = torch.empty_like(b)
    dev = P.device
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.fns["pslr_apply_multi"](dev.handle, meta["m"], 2, b.data_ptr(), z.data_ptr(), s))
    torch.cuda.synchronize()
    for v in range(2):
        np.testing.assert_array_equal(z[v].cpu().numpy(), P.apply(b[v].cpu().numpy()))


@pytest.mark.parametrize("cfg", ["cfg2", "cfg5"])
def test_merged_full_size_apply_matches_oracle(monkeypatch, cfg):
    """BASELINE sizes with the product default (merged C0): apply <= 1e-10 against the
    oracle on identical factors and correction state; linearity and determinism."""
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import workloads
    from oracle import pslr_oracle as O
    monkeypatch.setenv("PSLR_MERGE", "2")
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
    z1 = P.apply(b)
    assert _rel(z1, OP.apply(b)) <= 1e-10
    g = rng.standard_normal(ps.q)
    assert _rel(pg.solve_C0(P.ctx, g), O.solve_C0(octx, g)) <= 1e-12
    np.testing.assert_array_equal(z1, P.apply(b))
    b2 = rng.standard_normal(ps.n)
    assert _rel(P.apply(2.0 * b + b2), 2.0 * z1 + P.apply(b2)) <= 1e-10
