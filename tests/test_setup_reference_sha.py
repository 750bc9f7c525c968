"""SURVEY §8f rank 1 acceptance at the BASELINE configs: the product's native host setup
(BFS bisection + reorder + ILUT, csrc/setup.cpp) gives the REFERENCE's matrix, partition
assignment, permutation and L_B / U_B / L_C0 / U_C0 / C_g bit for bit on cfg2, cfg3, cfg5
and cfg4.  The reference hashes come from tests/golden/make_golden_r2.py, which ran the
real reference setup in the build container (cfg5: 110 s, cfg4: several minutes there;
the native setup takes seconds).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import csr_sha, golden

G = golden()
CASES = sorted(G.get("setup_sha", {}))


def _sha(a):
    h = hashlib.sha256()
    a = np.ascontiguousarray(a)
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", CASES)
def test_native_setup_matches_reference_hashes(name):
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import workloads
    from paper_2002_00917_b200.schur import _block_diag_part
    ref = G["setup_sha"][name]
    wl = workloads.CONFIGS[name]
    A = wl.matrix()
    assert csr_sha(A) == ref["A_sha"], "generator differs from the reference's matrix"
    spec = pg.partition_graph(A, ref["s"], seed=0)
    assert _sha(np.asarray(spec.assignment).astype(np.int64)) == ref["assignment_sha"]
    ps = pg.classify_and_reorder(A, spec)
    assert (ps.n, ps.p, ps.q) == (ref["n"], ref["p"], ref["q"])
    assert _sha(ps.perm.forward.astype(np.int64)) == ref["forward_sha"]
    assert csr_sha(ps.matrix) == ref["matrix_sha"]
    b = pg.factor_blocks(ps.B, ps.interior_sizes, droptol=1e-2)
    assert csr_sha(b.L) == ref["LB_sha"] and csr_sha(b.U) == ref["UB_sha"]
    C0 = _block_diag_part(ps.C, ps.interface_sizes)
    c = pg.factor_blocks(C0, ps.interface_sizes, droptol=1e-2)
    assert csr_sha(c.L) == ref["LC_sha"] and csr_sha(c.U) == ref["UC_sha"]
    from paper_2002_00917_b200.sparse import canonical
    assert csr_sha(canonical(ps.C - C0)) == ref["Cg_sha"]  # schur.py:57
