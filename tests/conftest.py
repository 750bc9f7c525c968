"""Shared fixtures: golden-vector loading and the reference test-matrix helpers.

Nothing here reads /root/reference: the golden fixtures under tests/golden/
were produced from it by tests/golden/make_golden.py and committed.
"""

import json
import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

# The suite pins the bit-exact contract: the device factors are the reference's
# rows, solved in the reference's order.  The product default (PSLR_MERGE=2: level-merged
# C0 factors, exact up to round-off) is covered by tests/test_gpu_merged.py, which sets the
# mode per test (libpslr reads it when a context is created).
os.environ.setdefault("PSLR_MERGE", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def golden() -> dict:
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


def load_npz(name):
    return np.load(os.path.join(GOLDEN_DIR, name))


def csr_from(d, prefix):
    return sp.csr_matrix((d[prefix + "_data"], d[prefix + "_indices"], d[prefix + "_indptr"]),
                         shape=tuple(int(x) for x in d[prefix + "_shape"]))


def lap1d(n):
    """Reference test helper (pkg/tests/conftest.py:20-22)."""
    return sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")


def random_sparse(n, density=0.1, seed=0, diag_boost=4.0):
    """Reference test helper (pkg/tests/conftest.py:25-29)."""
    A = sp.random(n, n, density=density, random_state=seed, format="csr",
                  data_rvs=np.random.default_rng(seed).standard_normal)
    return (A + diag_boost * sp.identity(n)).tocsr()


def partition_case_matrix(name):
    """Matrices of tests/golden/make_golden.py:partition_cases, rebuilt."""
    from oracle import pslr_oracle as O
    table = {
        "lap1d6_s2": lambda: lap1d(6),
        "lap1d20_s4": lambda: lap1d(20),
        "lap3d8_s5": lambda: O.laplacian3d(8, 8, 8),
        "lap3d8_s8": lambda: O.laplacian3d(8, 8, 8),
        "rand100_s6": lambda: random_sparse(100, seed=3),
        "twopaths_s2": lambda: sp.block_diag([lap1d(3), lap1d(3)], format="csr"),
        "lap2d64_s4": lambda: O.laplacian3d(64, 64, 1, shift=2.3),
        "lap3d12_s7": lambda: O.laplacian3d(12, 12, 12, shift=0.05),
        "lap3d32_s35": lambda: O.laplacian3d(32, 32, 32, shift=0.16),
        "upw3d16_s16": lambda: O.upwind3d(16, 16, 16, 0.2, 0.5),
    }
    return table[name]()


def csr_sha(M):
    import hashlib
    M = sp.csr_matrix(M)
    h = hashlib.sha256()
    for a in (M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data):
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


SMALL_APPLY_CASES = ["lap3d6_s4_dt1e-2", "lap3d6_s4_dt0", "rand80_s4", "lap1d30_s1", "upw3d8_s4",
                     "cfg1", "crit11"]


@pytest.fixture(scope="session")
def gold():
    return golden()


def have_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
