"""Sparse-matrix plumbing for the host setup (mirrors pslr/sparse.py).

`canonical`, `Permutation` and `matvec` keep the reference's contracts
(sparse.py:26-65).  `permute_symmetric` / `extract_submatrix` produce the same
canonical CSR as the reference (sparse.py:68-89) with a vectorised gather that
is fast at the 2-4M-row configs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


def canonical(A) -> sp.csr_matrix:
    """CSR, float64, duplicates summed, indices sorted (sparse.py:26-31)."""
    M = sp.csr_matrix(A, dtype=np.float64, copy=False)
    M.sum_duplicates()
    M.sort_indices()
    return M


@dataclass(frozen=True)
class Permutation:
    """Bijection on {0..n-1}; forward maps old index -> new index (sparse.py:34-57)."""
    forward: np.ndarray
    inverse: np.ndarray

    @classmethod
    def from_forward(cls, forward) -> "Permutation":
        forward = np.asarray(forward, dtype=np.int64)
        n = forward.size
        inverse = np.empty(n, dtype=np.int64)
        if n and (forward.min() < 0 or forward.max() >= n or np.unique(forward).size != n):
            raise ValueError("forward map is not a bijection on {0..n-1}")
        inverse[forward] = np.arange(n, dtype=np.int64)
        return cls(forward=forward, inverse=inverse)

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        idx = np.arange(n, dtype=np.int64)
        return cls(forward=idx.copy(), inverse=idx.copy())

    def __len__(self):
        return self.forward.size


def matvec(A, x) -> np.ndarray:
    """y = A x with dimension checking (sparse.py:60-65)."""
    x = np.asarray(x, dtype=np.float64)
    if A.shape[1] != x.shape[0]:
        raise ValueError(f"dimension mismatch: matrix is {A.shape}, vector has {x.shape[0]}")
    return A @ x


def permute_symmetric(A, p: Permutation) -> sp.csr_matrix:
    """result[p(i), p(j)] = A[i, j] (sparse.py:68-76), as a row gather + column relabel."""
    if A.shape[0] != A.shape[1]:
        raise ValueError("matrix must be square")
    if A.shape[0] != len(p):
        raise ValueError(f"permutation over {len(p)} indices, matrix is {A.shape[0]}x{A.shape[0]}")
    A = canonical(A)
    n = A.shape[0]
    lens = np.diff(A.indptr)[p.inverse]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=indptr[1:])
    starts = A.indptr[:-1][p.inverse].astype(np.int64)
    # gather positions of every entry of the new row order
    src = np.repeat(starts - indptr[:-1], lens) + np.arange(indptr[-1], dtype=np.int64)
    indices = p.forward[A.indices[src]]
    out = sp.csr_matrix((A.data[src], indices.astype(np.int32), indptr), shape=A.shape)
    out.has_sorted_indices = False
    out.sort_indices()
    return out


def extract_submatrix(A, rows, cols) -> sp.csr_matrix:
    """result[a, b] = A[rows[a], cols[b]] for sorted in-range index sets (sparse.py:79-89)."""
    A = canonical(A)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    for name, idx, limit in (("row", rows, A.shape[0]), ("column", cols, A.shape[1])):
        if idx.size and (idx.min() < 0 or idx.max() >= limit):
            raise ValueError(f"{name} index set out of range")
        if np.any(np.diff(idx) <= 0):
            raise ValueError(f"{name} index set must be strictly increasing")

    def as_slice(idx):
        if idx.size and idx[-1] - idx[0] + 1 == idx.size:
            return slice(int(idx[0]), int(idx[-1]) + 1)
        return idx
    return canonical(A[as_slice(rows)][:, as_slice(cols)])
