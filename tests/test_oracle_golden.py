"""Pin the oracle (oracle/pslr_oracle.py + oracle/csrc/oracle_setup.c) against the
golden fixtures generated from the real reference (tests/golden/make_golden.py).

CPU only.  Tolerances: bit-exact for partitions, reorderings and ILUT factors
(integer/index work and identical scalar arithmetic); bit-exact for the
scipy-only operators (block solves, SpMVs, Horner, E_rr); 1e-12 relative for
anything that goes through BLAS (V, H, G, the correction, the full apply),
because the BLAS build on the machine running the test may differ.
"""

import numpy as np
import pytest

from conftest import (SMALL_APPLY_CASES, csr_from, csr_sha, golden, load_npz,
                      partition_case_matrix)
from oracle import pslr_oracle as O

G = golden()


def _same_csr(A, B):
    return (np.array_equal(np.asarray(A.indptr, np.int64), np.asarray(B.indptr, np.int64))
            and np.array_equal(A.indices, B.indices) and np.array_equal(A.data, B.data))


@pytest.mark.parametrize("name", sorted(G["ilut"]))
@pytest.mark.parametrize("impl", ["python", "c"])
def test_ilut_bitexact(name, impl):
    d = load_npz("ilut_cases.npz")
    meta = G["ilut"][name]
    A = csr_from(d, name + "_A")
    fn = O.ilut if impl == "python" else O.ilut_c
    f = fn(A, meta["droptol"], meta["fill_cap"])
    assert _same_csr(f.L, csr_from(d, name + "_L"))
    assert _same_csr(f.U, csr_from(d, name + "_U"))
    assert f.pivot_repairs == meta["pivot_repairs"]


@pytest.mark.parametrize("name", sorted(G["partition"]))
@pytest.mark.parametrize("impl", ["python", "c"])
def test_partition_bitexact(name, impl):
    d = load_npz("partition_cases.npz")
    meta = G["partition"][name]
    A = partition_case_matrix(name)
    if impl == "python" and A.shape[0] > 5000:
        pytest.skip("pure-Python BFS restatement only on small graphs")
    assign = (O.partition_graph if impl == "python" else O.partition_c)(A, meta["s"])
    np.testing.assert_array_equal(assign, d[name + "_assignment"])
    ps = O.classify_and_reorder(A, assign, meta["s"])
    np.testing.assert_array_equal(ps.perm.forward, d[name + "_forward"])
    assert ps.p == meta["p"] and ps.q == meta["q"]
    assert ps.interior_sizes.tolist() == meta["interior_sizes"]
    assert ps.interface_sizes.tolist() == meta["interface_sizes"]
    for blk in ("matrix", "B", "E", "F", "C"):
        assert csr_sha(getattr(ps, blk)) == meta[blk + "_sha"], blk


def _oracle_build(name, use_c=False):
    meta = G["apply"][name]
    d = load_npz(f"apply_{name}.npz")
    A = csr_from(d, "A")
    P = O.build(A, meta["s"], meta["m"], meta["rank"], meta["droptol"], meta["seed"], use_c=use_c)
    return P, meta, d


@pytest.mark.parametrize("name", SMALL_APPLY_CASES)
def test_oracle_operators_match_reference(name):
    P, meta, d = _oracle_build(name)
    ctx = P.ctx
    assert P.system.p == meta["p"] and P.system.q == meta["q"]
    for key, M in (("LB", ctx.b_ilu.L), ("UB", ctx.b_ilu.U), ("LC", ctx.c0_ilu.L), ("UC", ctx.c0_ilu.U)):
        assert csr_sha(M) == meta[key + "_sha"], key
    assert csr_sha(ctx.Cg) == meta["Cg_sha"]
    # scipy-only operators: bit-exact
    np.testing.assert_array_equal(O.solve_B(ctx, d["f"]), d["solve_B"])
    if P.system.q:
        np.testing.assert_array_equal(O.solve_C0(ctx, d["v"]), d["solve_C0"])
        np.testing.assert_array_equal(O.apply_Es(ctx, d["v"]), d["apply_Es"])
        np.testing.assert_array_equal(O.apply_neumann(ctx, meta["m"], d["v"]), d["apply_neumann"])
        np.testing.assert_array_equal(O.apply_Err(ctx, meta["m"], d["v"]), d["apply_Err"])
    # BLAS-touched state: tight tolerance
    assert P.corr.rank == meta["achieved_rank"]
    if P.corr.rank:
        for key, X in (("V", P.corr.V), ("H", P.corr.H), ("G", P.corr.G)):
            ref = d[key]
            assert np.linalg.norm(X - ref) <= 1e-12 * max(np.linalg.norm(ref), 1.0), key
        ac = O.apply_correction(P.corr, d["v"])
        assert np.linalg.norm(ac - d["apply_correction"]) <= 1e-12 * np.linalg.norm(d["apply_correction"])
    z = P.apply(d["b"])
    assert np.linalg.norm(z - d["apply"]) <= 1e-12 * np.linalg.norm(d["apply"])
    zo = P.apply_original(d["b"])
    assert np.linalg.norm(zo - d["apply_original"]) <= 1e-12 * np.linalg.norm(d["apply_original"])


def test_oracle_c_setup_same_build():
    """The C restatement of ILUT/bisection gives the same build as the Python one."""
    P1, meta, d = _oracle_build("cfg1", use_c=False)
    P2, _, _ = _oracle_build("cfg1", use_c=True)
    np.testing.assert_array_equal(P1.system.perm.forward, P2.system.perm.forward)
    assert _same_csr(P1.ctx.b_ilu.L, P2.ctx.b_ilu.L) and _same_csr(P1.ctx.b_ilu.U, P2.ctx.b_ilu.U)
    np.testing.assert_array_equal(P1.apply(d["b"]), P2.apply(d["b"]))


def _solve_reordered(P, A, tol, maxit, restart, seed=0):
    b = A @ np.random.default_rng(seed).standard_normal(A.shape[0])
    bp = b[P.system.perm.inverse]
    Ap = P.system.matrix
    return O.gmres(lambda v: Ap @ v, P.apply, bp, tol=tol, maxit=maxit, restart=restart)[1]


def test_oracle_gmres_crit11():
    P, meta, d = _oracle_build("crit11")
    rep = _solve_reordered(P, csr_from(d, "A"), 1e-8, 500, 0)
    ref = G["gmres"]["crit11"]
    assert rep.converged == ref["converged"] and rep.iterations == ref["iterations"] == 13


def test_oracle_gmres_cfg1_fails_like_reference():
    P, meta, d = _oracle_build("cfg1", use_c=True)
    rep = _solve_reordered(P, csr_from(d, "A"), 1e-6, 500, 50)
    ref = G["gmres"]["cfg1_gmres50"]
    assert not rep.converged and rep.iterations == ref["iterations"] == 500
    assert len(rep.history) == 501
    h = np.array(rep.history[:50])
    hr = np.array(ref["history_first_cycle"][:50])
    assert np.max(np.abs(h - hr) / hr) <= 1e-6


@pytest.mark.parametrize("m", [3, 5])
def test_oracle_gmres_crit07(m):
    """Criterion 07 instance (32^3, shift 0.16, s=35, r=15, seed 2), full GMRES tol 1e-8."""
    A = O.laplacian3d(32, 32, 32, shift=0.16)
    P = O.build(A, 35, m, 15, 1e-2, seed=2, use_c=True)
    rep = _solve_reordered(P, A, 1e-8, 500, 0, seed=2)
    ref = G["gmres"]["crit07"][f"{m}_reordered"]
    assert rep.converged and abs(rep.iterations - ref["iterations"]) <= 2


@pytest.mark.parametrize("twin", ["twin_cfg2", "twin_cfg3"])
def test_oracle_gmres_twins(twin):
    if twin not in G["gmres"]:
        pytest.skip("twin not generated")
    meta = G["apply"][twin]
    A = O.laplacian3d(32, 32, 32, shift=0.16) if twin == "twin_cfg2" else O.upwind3d(32, 32, 32, 0.2, 0.5)
    P = O.build(A, meta["s"], meta["m"], meta["rank"], 1e-2, 0, use_c=True)
    rep = _solve_reordered(P, A, 1e-6, 500, 50)
    ref = G["gmres"][twin]
    assert rep.converged == ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= 2
