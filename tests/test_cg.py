"""CG (krylov.py:132-174): the oracle against golden vectors of the
real reference (tests/golden/make_golden_cg.py) and — on a GPU — the device CG: on
generic operators (pslr_cg_op, operator callbacks) against the reference's own CG tests
(pkg/tests/test_krylov.py:105-140), and on the PSLR operators (pslr_cg through the C-ABI)
against the golden iteration counts.

Bars: oracle iterations exact and histories to 1e-9 relative (rank-0 PSLR applies are
scipy-only, so the oracle reproduces the reference's arithmetic); device iterations
within +-2 of the reference (SURVEY §8d rule), same converged flag, failure contract
(iterations == maxit, maxit+1 history entries) exact.
"""

import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN_DIR, have_cuda, lap1d
from oracle import pslr_oracle as O

with open(os.path.join(GOLDEN_DIR, "cg_cases.json")) as fh:
    CG = json.load(fh)["cases"]
PSLR_CASES = [k for k in CG if "grid" in CG[k]]


def _problem(meta):
    A = O.laplacian3d(*meta["grid"], shift=meta["shift"])
    b = A @ np.random.default_rng(0).standard_normal(A.shape[0])
    return A, b


# ---------------------------------------------------------------- CPU: the oracle pinned
@pytest.mark.parametrize("name", PSLR_CASES)
def test_oracle_cg_matches_reference(name):
    meta = CG[name]
    A, b = _problem(meta)
    P = O.build(A, meta["s"], meta["m"], meta["rank"])
    Ap, perm = P.system.matrix, P.system.perm
    x, rep = O.cg(lambda v: Ap @ v, P.apply, b[perm.inverse], tol=meta["tol"], maxit=meta["maxit"])
    assert rep.converged == meta["converged"]
    assert rep.iterations == meta["iterations"]
    np.testing.assert_allclose(rep.history, meta["history"], rtol=1e-9, atol=0)


def test_oracle_cg_failure_contract():
    ref = CG["lap1d400_noprec_maxit10"]
    A = lap1d(400)
    x, rep = O.cg(lambda v: A @ v, None, np.ones(400), tol=1e-14, maxit=10)
    assert (rep.converged, rep.iterations) == (ref["converged"], ref["iterations"])
    np.testing.assert_allclose(rep.history, ref["history"], rtol=1e-12)


# ---------------------------------------------------------------- GPU: generic operators
def _dense_spd(n, seed):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((n, n))
    return Q @ Q.T + n * np.eye(n)


@pytest.mark.gpu
@pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("as_matrix", [False, True])
def test_generic_cg_matches_oracle_spd(as_matrix):
    """The device CG on a generic operator (a host callable, or the scipy matrix itself:
    libpslr's CSR SpMV) against the oracle's restatement of the reference loop."""
    import paper_2002_00917_b200 as pg
    A = sp.csr_matrix(_dense_spd(60, 10))
    b = A @ np.random.default_rng(11).standard_normal(60)
    x, rep = pg.cg(A if as_matrix else (lambda v: A @ v), None, b, tol=1e-10)
    xo, repo = O.cg(lambda v: A @ v, None, b, tol=1e-10)
    assert rep.converged and rep.iterations == repo.iterations
    np.testing.assert_allclose(x, xo, rtol=0, atol=1e-10 * np.abs(xo).max())
    np.testing.assert_allclose(rep.history, repo.history, rtol=1e-8)


@pytest.mark.gpu
@pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")
def test_generic_cg_reference_contracts():
    """pkg/tests/test_krylov.py:115-140: Jacobi helps, indefinite raises, failure
    contract, zero right-hand side."""
    import paper_2002_00917_b200 as pg
    A = lap1d(300).toarray() + np.diag(np.linspace(0, 10, 300))
    b = np.ones(300)
    _, rep0 = pg.cg(lambda v: A @ v, None, b)
    d = 1.0 / np.diag(A)
    _, rep1 = pg.cg(lambda v: A @ v, lambda v: d * v, b)
    assert rep1.converged and rep1.iterations <= rep0.iterations
    with pytest.raises(pg.NotSpdError):
        pg.cg(lambda v: np.diag([1.0, -1.0, 2.0]) @ v, None, np.ones(3))
    A4 = lap1d(400)
    _, rep = pg.cg(lambda v: A4 @ v, None, np.ones(400), tol=1e-14, maxit=10)
    assert not rep.converged and rep.iterations == 10 and len(rep.history) == 11 and rep.history[0] == 1.0
    x, rep = pg.cg(lambda v: v, None, np.zeros(3))
    assert rep.converged and rep.iterations == 0 and not x.any()


# ---------------------------------------------------------------- GPU: the device CG
def _device_build(meta):
    import paper_2002_00917_b200 as pg
    A, b = _problem(meta)
    P = pg.build(A, pg.PslrConfig(num_subdomains=meta["s"], series_degree=meta["m"], rank=meta["rank"]))
    return pg, P, A, b


@pytest.mark.parametrize("name", PSLR_CASES)
@pytest.mark.gpu
@pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")
def test_device_cg_iterations(name):
    meta = CG[name]
    pg, P, A, b = _device_build(meta)
    perm = P.system.perm
    x, rep = pg.cg(P.matvec, P.apply, b[perm.inverse], tol=meta["tol"], maxit=meta["maxit"])
    assert rep.converged == meta["converged"]
    if meta["converged"]:
        assert abs(rep.iterations - meta["iterations"]) <= 2
        xo = x[perm.forward]
        assert np.linalg.norm(b - A @ xo) <= 10 * meta["tol"] * np.linalg.norm(b)
    else:  # failure contract
        assert rep.iterations == meta["maxit"] and len(rep.history) == meta["maxit"] + 1
    n = min(len(rep.history), len(meta["history"]), 6)
    np.testing.assert_allclose(rep.history[:n], meta["history"][:n], rtol=1e-6)


@pytest.mark.gpu
@pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")
def test_device_cg_original_space_zero_rhs_and_not_spd():
    import paper_2002_00917_b200 as pg
    meta = CG["cli_lap3d6_s4_r0"]
    pg, P, A, b = _device_build(meta)
    x, rep = pg.cg(P.matvec_original, P.apply_original, b, tol=1e-8)
    assert rep.converged and abs(rep.iterations - meta["iterations"]) <= 2
    assert np.linalg.norm(b - A @ x) <= 1e-7 * np.linalg.norm(b)
    x0, rep0 = pg.cg(P.matvec, P.apply, np.zeros(A.shape[0]))
    assert rep0.converged and rep0.iterations == 0 and not x0.any() and rep0.history == [1.0]
    with pytest.raises(ValueError):
        pg.cg(P.matvec, P.apply, np.zeros(A.shape[0] + 1))
    # indefinite (shifted) Laplacian: CG meets a non-positive curvature direction
    Ai = O.laplacian3d(8, 8, 8, shift=1.5)
    Pi = pg.build(Ai, pg.PslrConfig(num_subdomains=4, series_degree=3, rank=0))
    bi = Ai @ np.random.default_rng(0).standard_normal(Ai.shape[0])
    with pytest.raises(pg.NotSpdError):
        pg.cg(Pi.matvec, Pi.apply, bi[Pi.system.perm.inverse], maxit=500)
