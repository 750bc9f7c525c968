"""Setup cache (paper_2002_00917_b200/setup_cache.py): a cache hit
reproduces the reordering, both block factors and the correction bit for bit, and the
device apply built from it equals the one built from scratch bit for bit."""

import numpy as np
import pytest

from conftest import have_cuda
from oracle import pslr_oracle as O


def _same_csr(A, B):
    return (A.shape == B.shape and np.array_equal(np.asarray(A.indptr, np.int64), np.asarray(B.indptr, np.int64))
            and np.array_equal(A.indices, B.indices) and np.array_equal(A.data, B.data))


def test_setup_roundtrip_bitexact(tmp_path):
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import setup_cache as SC
    from paper_2002_00917_b200.schur import _block_diag_part
    A = O.upwind3d(9, 8, 7, 0.2, 0.5)
    cfg = pg.PslrConfig(num_subdomains=6, series_degree=3, rank=4)
    system = pg.classify_and_reorder(A, pg.partition_graph(A, cfg.num_subdomains))
    b_ilu = pg.factor_blocks(system.B, system.interior_sizes, droptol=cfg.droptol)
    C0 = _block_diag_part(system.C, system.interface_sizes)
    c0_ilu = pg.factor_blocks(C0, system.interface_sizes, droptol=cfg.droptol)
    key = SC.setup_key(SC.matrix_digest(A), cfg)
    path = str(tmp_path / f"setup_{key}.npz")
    SC.save_setup(path, system, b_ilu, c0_ilu)
    ps2, b2, c2 = SC.load_setup(path, A)
    np.testing.assert_array_equal(ps2.perm.forward, system.perm.forward)
    np.testing.assert_array_equal(ps2.perm.inverse, system.perm.inverse)
    assert (ps2.p, ps2.q, ps2.num_parts) == (system.p, system.q, system.num_parts)
    for a, b in ((ps2.matrix, system.matrix), (ps2.B, system.B), (ps2.E, system.E), (ps2.F, system.F),
                 (ps2.C, system.C), (b2.L, b_ilu.L), (b2.U, b_ilu.U), (c2.L, c0_ilu.L), (c2.U, c0_ilu.U)):
        assert _same_csr(a, b)
    assert b2.pivot_repairs == b_ilu.pivot_repairs and b2.nnz == b_ilu.nnz
    # keys: any change of matrix or setup parameters misses
    A2 = A.copy()
    A2.data[0] += 1e-12
    assert SC.setup_key(SC.matrix_digest(A2), cfg) != key
    assert SC.setup_key(SC.matrix_digest(A), pg.PslrConfig(num_subdomains=6, droptol=1e-3)) != key
    assert SC.correction_key(key, cfg) != SC.correction_key(key, pg.PslrConfig(num_subdomains=6, rank=5))
    # correction round trip
    rng = np.random.default_rng(0)
    V, H, G = rng.standard_normal((system.q, 4)), rng.standard_normal((4, 4)), rng.standard_normal((4, 4))
    cp = str(tmp_path / "corr.npz")
    SC.save_correction(cp, V, H, G, 4)
    V2, H2, G2, r2 = SC.load_correction(cp)
    assert r2 == 4 and np.array_equal(V2, V) and np.array_equal(H2, H) and np.array_equal(G2, G)
    assert SC.load_setup(str(tmp_path / "missing.npz"), A) is None


@pytest.mark.gpu
@pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")
def test_build_from_cache_bitexact(tmp_path):
    import paper_2002_00917_b200 as pg
    A = O.laplacian3d(14, 13, 12, shift=0.4)
    cfg = pg.PslrConfig(num_subdomains=8, series_degree=3, rank=12)
    P1 = pg.build(A, cfg, cache_dir=str(tmp_path))
    files = sorted(p.name for p in tmp_path.iterdir())
    assert len(files) == 3 and files[0].startswith("corr_") and files[1].startswith("pack_") \
        and files[2].startswith("setup_")
    assert not P1.device.packed_reused
    P2 = pg.build(A, cfg, cache_dir=str(tmp_path))  # hit: no partition / ILUT / Arnoldi / packing
    assert P2.device.packed_reused
    P0 = pg.build(A, cfg)                           # no cache
    assert np.array_equal(P2.correction.V, P1.correction.V) and np.array_equal(P2.correction.G, P1.correction.G)
    assert P2.device.info() == {**P0.device.info(), "device_bytes": P2.device.info()["device_bytes"]}
    b = np.random.default_rng(3).standard_normal(A.shape[0])
    z0, z1, z2 = P0.apply(b), P1.apply(b), P2.apply(b)
    np.testing.assert_array_equal(z1, z0)
    np.testing.assert_array_equal(z2, z0)
    f = np.random.default_rng(4).standard_normal(P0.system.p)
    np.testing.assert_array_equal(pg.solve_B(P2.ctx, f), pg.solve_B(P0.ctx, f))
    # a different series degree reuses the setup and packed files and adds one correction file
    pg.build(A, pg.PslrConfig(num_subdomains=8, series_degree=2, rank=12), cache_dir=str(tmp_path))
    assert len(list(tmp_path.iterdir())) == 4
    # a corrupted or foreign blob is never used: the context re-packs and stays bit-exact
    pack = next(p for p in tmp_path.iterdir() if p.name.startswith("pack_"))
    pack.write_bytes(pack.read_bytes()[:-8])
    P3 = pg.build(A, cfg, cache_dir=str(tmp_path))
    assert not P3.device.packed_reused
    np.testing.assert_array_equal(P3.apply(b), z0)
    P4 = pg.build(A, cfg, cache_dir=str(tmp_path))  # P3 rewrote a good blob
    assert P4.device.packed_reused
