"""Block ILUT factors (mirrors pslr/ilu.py).

Factorisation is setup: it stays on the host, restated in native C++
(`pslr_ilut_blocks`, csrc/setup.cpp) so that it is bit-identical to the
reference's pure-Python ilut (ilu.py:35-138) while running the independent
blocks on all host cores.  The triangular SOLVES are the hot path and run on
the GPU through the preconditioner's device context (schur.solve_B / solve_C0).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from .sparse import canonical


@dataclass
class IluFactor:
    """L unit-lower (diagonal stored explicitly, last in each row) and U upper (ilu.py:21-32)."""
    L: sp.csr_matrix
    U: sp.csr_matrix
    n: int
    pivot_repairs: int = 0

    @property
    def nnz(self) -> int:
        return self.L.nnz + self.U.nnz


@dataclass
class BlockILU:
    """Assembled block-diagonal factors of independent diagonal blocks (ilu.py:141-164)."""
    offsets: np.ndarray
    L: sp.csr_matrix
    U: sp.csr_matrix
    block_nnz: np.ndarray = field(repr=False, default=None)      # (nblocks, 2): nnz(L_b), nnz(U_b)
    block_repairs: np.ndarray = field(repr=False, default=None)  # (nblocks,)

    @property
    def n(self) -> int:
        return int(self.offsets[-1])

    @property
    def nnz(self) -> int:
        return int(self.block_nnz.sum()) if self.block_nnz is not None else self.L.nnz + self.U.nnz

    @property
    def pivot_repairs(self) -> int:
        return int(self.block_repairs.sum()) if self.block_repairs is not None else 0

    @property
    def factors(self) -> list:
        out = []
        for b in range(self.offsets.size - 1):
            lo, hi = int(self.offsets[b]), int(self.offsets[b + 1])
            out.append(IluFactor(L=self.L[lo:hi, lo:hi], U=self.U[lo:hi, lo:hi], n=hi - lo,
                                 pivot_repairs=int(self.block_repairs[b])))
        return out


def factor_blocks(A, block_sizes, droptol: float = 1e-2, fill_cap: int | None = None,
                  nthreads: int = 0) -> BlockILU:
    """ILUT of each diagonal block of A (ilu.py:167-184), blocks in parallel (C++)."""
    A = canonical(A)
    sizes = np.asarray(block_sizes, dtype=np.int64)
    if sizes.sum() != A.shape[0] or A.shape[0] != A.shape[1]:
        raise ValueError("block sizes do not tile the matrix")
    if droptol < 0:
        raise ValueError("droptol must be >= 0")
    n = A.shape[0]
    nb = sizes.size
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    if nb == 0:
        z = sp.csr_matrix((0, 0))
        return BlockILU(offsets, z, z.copy(), np.zeros((0, 2), np.int64), np.zeros(0, np.int64))
    ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    dv = np.ascontiguousarray(A.data, dtype=np.float64)
    handle = ctypes.c_void_p()
    nl, nu, rep = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.fns["pslr_ilut_blocks"](
        n, ip.ctypes.data, ix.ctypes.data, dv.ctypes.data, nb, offsets.ctypes.data, float(droptol),
        -1 if fill_cap is None else int(fill_cap), int(nthreads), ctypes.byref(handle),
        ctypes.byref(nl), ctypes.byref(nu), ctypes.byref(rep)))
    try:
        Lp = np.empty(n + 1, np.int64); Li = np.empty(nl.value, np.int32); Lx = np.empty(nl.value)
        Up = np.empty(n + 1, np.int64); Ui = np.empty(nu.value, np.int32); Ux = np.empty(nu.value)
        bnnz = np.empty((nb, 2), np.int64)
        brep = np.empty(nb, np.int64)
        _lib.check(_lib.fns["pslr_factors_fetch"](
            handle, Lp.ctypes.data, Li.ctypes.data, Lx.ctypes.data, Up.ctypes.data,
            Ui.ctypes.data, Ux.ctypes.data, bnnz.ctypes.data, brep.ctypes.data))
    finally:
        _lib.fns["pslr_factors_free"](handle)
    itype = np.int32 if max(nl.value, nu.value) < 2**31 else np.int64
    L = sp.csr_matrix((Lx, Li, Lp.astype(itype)), shape=(n, n))
    U = sp.csr_matrix((Ux, Ui, Up.astype(itype)), shape=(n, n))
    L.has_sorted_indices = True
    U.has_sorted_indices = True
    return BlockILU(offsets, L, U, bnnz, brep)


def ilut(block, droptol: float = 1e-2, fill_cap: int | None = None) -> IluFactor:
    """Incomplete LU of one square block with threshold dropping (ilu.py:35-138)."""
    A = canonical(block)
    if A.shape[0] != A.shape[1]:
        raise ValueError("block must be square")
    if droptol < 0:
        raise ValueError("droptol must be >= 0")
    n = A.shape[0]
    if n == 0:
        empty = sp.csr_matrix((0, 0))
        return IluFactor(L=empty, U=empty.copy(), n=0, pivot_repairs=0)
    bf = factor_blocks(A, [n], droptol=droptol, fill_cap=fill_cap, nthreads=1)
    return IluFactor(L=bf.L, U=bf.U, n=n, pivot_repairs=bf.pivot_repairs)


def row_norms(A) -> np.ndarray:
    """np.sqrt(A.multiply(A).sum(axis=1)) as the native ILUT computes it (ilu.py:52)."""
    A = canonical(A)
    ip = np.ascontiguousarray(A.indptr, dtype=np.int64)
    dv = np.ascontiguousarray(A.data, dtype=np.float64)
    out = np.empty(A.shape[0])
    _lib.check(_lib.fns["pslr_row_norms"](A.shape[0], ip.ctypes.data, dv.ctypes.data, out.ctypes.data))
    return out
