"""The product's native host setup (csrc/setup.cpp via ctypes) is bit-identical to the
reference: ILUT factors, BFS-bisection assignments, the reordered block system.
CPU only (no device calls)."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2002_00917_b200 as pg
from paper_2002_00917_b200 import ilu as pilu
from paper_2002_00917_b200 import sparse as psparse
from conftest import csr_from, csr_sha, golden, load_npz, partition_case_matrix, random_sparse
from oracle import pslr_oracle as O

G = golden()


def _same_csr(A, B):
    return (np.array_equal(np.asarray(A.indptr, np.int64), np.asarray(B.indptr, np.int64))
            and np.array_equal(np.asarray(A.indices, np.int64), np.asarray(B.indices, np.int64))
            and np.array_equal(A.data, B.data))


@pytest.mark.parametrize("name", sorted(G["ilut"]))
def test_native_ilut_matches_reference(name):
    d = load_npz("ilut_cases.npz")
    meta = G["ilut"][name]
    f = pg.ilut(csr_from(d, name + "_A"), meta["droptol"], meta["fill_cap"])
    assert _same_csr(f.L, csr_from(d, name + "_L"))
    assert _same_csr(f.U, csr_from(d, name + "_U"))
    assert f.pivot_repairs == meta["pivot_repairs"]


@pytest.mark.parametrize("name", sorted(G["partition"]))
def test_native_partition_matches_reference(name):
    d = load_npz("partition_cases.npz")
    meta = G["partition"][name]
    A = partition_case_matrix(name)
    spec = pg.partition_graph(A, meta["s"])
    np.testing.assert_array_equal(spec.assignment, d[name + "_assignment"])
    ps = pg.classify_and_reorder(A, spec)
    np.testing.assert_array_equal(ps.perm.forward, d[name + "_forward"])
    assert ps.interior_sizes.tolist() == meta["interior_sizes"]
    assert ps.interface_sizes.tolist() == meta["interface_sizes"]
    for blk in ("matrix", "B", "E", "F", "C"):
        assert csr_sha(getattr(ps, blk)) == meta[blk + "_sha"], blk


@pytest.mark.parametrize("name", ["lap3d6_s4_dt1e-2", "rand80_s4", "upw3d8_s4", "cfg1", "crit11"])
def test_native_block_factors_match_reference(name):
    meta = G["apply"][name]
    d = load_npz(f"apply_{name}.npz")
    A = csr_from(d, "A")
    ps = pg.classify_and_reorder(A, pg.partition_graph(A, meta["s"]))
    b = pg.factor_blocks(ps.B, ps.interior_sizes, droptol=meta["droptol"])
    assert csr_sha(b.L) == meta["LB_sha"] and csr_sha(b.U) == meta["UB_sha"]
    assert b.nnz == meta["nnz_LB"] + meta["nnz_UB"]
    from paper_2002_00917_b200.schur import _block_diag_part
    C0 = _block_diag_part(ps.C, ps.interface_sizes)
    c = pg.factor_blocks(C0, ps.interface_sizes, droptol=meta["droptol"])
    assert csr_sha(c.L) == meta["LC_sha"] and csr_sha(c.U) == meta["UC_sha"]
    assert csr_sha(pg.canonical(ps.C - C0)) == meta["Cg_sha"]


def test_threads_do_not_change_factors():
    A = O.laplacian3d(16, 16, 16, shift=0.3)
    ps = pg.classify_and_reorder(A, pg.partition_graph(A, 8))
    f1 = pg.factor_blocks(ps.B, ps.interior_sizes, nthreads=1)
    f8 = pg.factor_blocks(ps.B, ps.interior_sizes, nthreads=8)
    assert _same_csr(f1.L, f8.L) and _same_csr(f1.U, f8.U)


def test_native_matches_c_oracle_at_scale():
    """48^3 upwind (110K rows): native C++ setup == the oracle's C restatement."""
    A = O.upwind3d(48, 48, 48, 0.2, 0.5)
    a_native = pg.partition_graph(A, 24).assignment
    a_oracle = O.partition_c(A, 24)
    np.testing.assert_array_equal(a_native, a_oracle)
    ps = pg.classify_and_reorder(A, pg.PartitionSpec(24, a_native))
    po = O.classify_and_reorder(A, a_oracle, 24)
    assert _same_csr(ps.matrix, po.matrix)
    f = pg.factor_blocks(ps.B, ps.interior_sizes)
    fo = O.factor_blocks(po.B, po.interior_sizes, use_c=True)
    assert _same_csr(f.L, fo.L) and _same_csr(f.U, fo.U)


@pytest.mark.parametrize("length", [1, 2, 7, 8, 9, 15, 16, 17, 64, 127, 128, 129, 200, 513])
def test_row_norms_match_numpy(length):
    rng = np.random.default_rng(length)
    A = sp.csr_matrix(rng.standard_normal((3, length)) * 10.0 ** rng.integers(-3, 3, (3, length)))
    ref = np.sqrt(np.asarray(A.multiply(A).sum(axis=1)).ravel())
    np.testing.assert_array_equal(pilu.row_norms(A), ref)


def test_permute_symmetric_matches_scipy_indexing():
    A = random_sparse(300, density=0.05, seed=11)
    perm = pg.Permutation.from_forward(np.random.default_rng(1).permutation(300))
    got = psparse.permute_symmetric(A, perm)
    ref = O.permute_symmetric(A, O.Perm.from_forward(perm.forward))
    assert _same_csr(got, ref)


def test_errors_mirror_reference():
    with pytest.raises(ValueError):
        pg.partition_graph(sp.csr_matrix((3, 4)), 2)
    with pytest.raises(ValueError):
        pg.partition_graph(sp.identity(3, format="csr"), 4)
    with pytest.raises(ValueError):
        pg.factor_blocks(sp.identity(5, format="csr"), [2, 2])
    with pytest.raises(ValueError):
        pg.ilut(sp.csr_matrix((2, 3)))
    with pytest.raises(ValueError):
        pg.ilut(sp.identity(2, format="csr"), droptol=-1.0)
    with pytest.raises(ValueError):
        pg.PslrConfig(num_subdomains=0).validate()


def test_factor_blocks_empty_system_and_bad_tiling():
    """ilu.py edge cases (pkg/tests/test_ilu.py:117-129): an empty system factors to an
    empty BlockILU; block sizes that do not tile the matrix raise ValueError."""
    import scipy.sparse as sp
    import paper_2002_00917_b200 as pg
    bf = pg.factor_blocks(sp.csr_matrix((0, 0)), [])
    assert bf.n == 0 and bf.nnz == 0
    with pytest.raises(ValueError):
        pg.factor_blocks(sp.identity(5, format="csr"), [2, 2])
