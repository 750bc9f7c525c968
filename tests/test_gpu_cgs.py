"""GPU: the CGS2 passes of the device Krylov loops (pslr_cgs_pass, krylov.py:75-80 /
lowrank.py:62-67) against numpy on column-major bases, ragged row counts (not multiples of
the 128/256-row tiles), widths across every columns-per-warp instance and past the
128-column fused limit:

  mode 0  h = X^T w
  mode 1  w = w - X h0 ; h = X^T w        (the shared-memory staged pass)
  mode 2  w = w - X h0 ; h[0] = w . w

The device sums in its own fixed order (deterministic, not numpy's BLAS blocking), so the
check is a tolerance: 1e-13 relative on the projected vector, 1e-12 on the dots.
"""

import numpy as np
import pytest

from conftest import have_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")]


def _run(mode, n, k, seed):
    import torch

    from paper_2002_00917_b200 import _lib, operators

    rng = np.random.default_rng(seed)
    ld = (n + 31) // 32 * 32 + 32
    X = rng.standard_normal((k, ld))
    w = rng.standard_normal(n)
    h0 = rng.standard_normal(k) * 1e-2
    Xd = torch.from_numpy(X.reshape(-1).copy()).cuda()
    wd = torch.from_numpy(w.copy()).cuda()
    hd = torch.from_numpy(h0.copy()).cuda()
    out = torch.zeros(max(k, 1), dtype=torch.float64, device="cuda")
    ws = operators.workspace(0).handle
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.fns["pslr_cgs_pass"](ws, mode, Xd.data_ptr(), ld, n, k, wd.data_ptr(), hd.data_ptr(),
                                         out.data_ptr(), st))
    torch.cuda.synchronize()
    V = X[:, :n].T  # n x k
    return V, w, h0, wd.cpu().numpy(), out.cpu().numpy()


@pytest.mark.parametrize("n", [1, 127, 1000, 100_003])
@pytest.mark.parametrize("k", [1, 3, 8, 9, 17, 33, 50, 100, 128, 130])
def test_cgs_passes_match_numpy(n, k):
    for mode in (0, 1, 2):
        V, w, h0, wdev, out = _run(mode, n, k, seed=1000 * k + n + mode)
        if mode == 0:
            ref_w, ref_h = w, V.T @ w
        else:
            ref_w = w - V @ h0
            ref_h = V.T @ ref_w if mode == 1 else np.array([ref_w @ ref_w])
        scale = np.linalg.norm(w) + np.linalg.norm(V, axis=0) @ np.abs(h0)
        assert np.linalg.norm(wdev - ref_w) <= 1e-13 * scale, (mode, n, k)
        got = out[:k] if mode != 2 else out[:1]
        hs = np.linalg.norm(ref_w) * np.linalg.norm(V, axis=0) if mode != 2 else np.array([ref_w @ ref_w])
        assert np.all(np.abs(got - ref_h) <= 1e-12 * np.maximum(hs, 1e-300)), (mode, n, k)


def test_cgs_pass_is_deterministic():
    a = _run(1, 100_003, 50, seed=7)
    b = _run(1, 100_003, 50, seed=7)
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
