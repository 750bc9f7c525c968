"""Matrix-free Schur operators on the interface space (mirrors pslr/schur.py).

Splitting S = C0 - Es with Es = (C0 - C) + F B^{-1} E; the series
sum_{i<=m} (C0^{-1} Es)^i C0^{-1} and its residual operator (Es C0^{-1})^{m+1}.
Every operator here runs on the GPU (libpslr.so): one fused per-subdomain
kernel per Horner step (csrc/kernels.cu: subdomain_step_kernel).
Inputs may be numpy arrays (copied through) or float64 CUDA tensors (zero-copy);
the result has the input's type.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .device import DeviceContext
from .ilu import BlockILU, factor_blocks
from .partition import PartitionedSystem
from .sparse import canonical


@dataclass
class SchurContext:
    """Partitioned system, block factors and the device context (schur.py:26-38)."""
    system: PartitionedSystem
    b_ilu: BlockILU
    c0_ilu: BlockILU
    C0: sp.csr_matrix
    Cg: sp.csr_matrix
    device: DeviceContext = field(repr=False, default=None)

    @property
    def q(self) -> int:
        return self.system.q


def _block_diag_part(C, sizes) -> sp.csr_matrix:
    """Block-diagonal part of C for the given diagonal block sizes (schur.py:41-49)."""
    C = canonical(C)
    n = C.shape[0]
    block_of = np.repeat(np.arange(len(sizes)), sizes)
    rows = np.repeat(np.arange(n), np.diff(C.indptr))
    keep = block_of[rows] == block_of[C.indices]
    return canonical(sp.csr_matrix((C.data[keep], (rows[keep], C.indices[keep])), shape=C.shape))


def build_schur_context(ps: PartitionedSystem, droptol: float = 1e-2, fill_cap: int | None = None,
                        device=None, factors=None, packed=None, want_packed=False) -> SchurContext:
    """Factor the B_i and C_i diagonal blocks (host, native C++) and upload everything
    to the device (schur.py:52-59).  `factors` = (b_ilu, c0_ilu) from the setup cache
    skips the factorisation; `packed` (the cache's packed device format) skips the level
    analysis and chunk packing of the context."""
    C0 = _block_diag_part(ps.C, ps.interface_sizes)
    if factors is not None:
        b_ilu, c0_ilu = factors
    else:
        b_ilu = factor_blocks(ps.B, ps.interior_sizes, droptol=droptol, fill_cap=fill_cap)
        c0_ilu = factor_blocks(C0, ps.interface_sizes, droptol=droptol, fill_cap=fill_cap)
    Cg = canonical(ps.C - C0)
    dev = DeviceContext(ps, b_ilu, c0_ilu, C0, Cg, device=device, packed=packed, want_packed=want_packed)
    return SchurContext(system=ps, b_ilu=b_ilu, c0_ilu=c0_ilu, C0=C0, Cg=Cg, device=dev)


def _m(m):
    if m < 0:
        raise ValueError("series degree m must be >= 0")
    return int(m)


def solve_B(ctx: SchurContext, rhs):
    """B^{-1} rhs with the block ILUT factors (schur.py:69-70)."""
    return ctx.device.vec_op("pslr_solve_B", rhs, ctx.system.p, ctx.system.p)


def solve_C0(ctx: SchurContext, rhs):
    """C0^{-1} rhs (schur.py:73-74)."""
    return ctx.device.vec_op("pslr_solve_C0", rhs, ctx.q, ctx.q)


def apply_S(ctx: SchurContext, v):
    """S v = C v - F B^{-1} (E v) (schur.py:77-80)."""
    return ctx.device.vec_op("pslr_apply_S", v, ctx.q, ctx.q)


def apply_Es(ctx: SchurContext, v):
    """Es v = F B^{-1} (E v) - Cg v (schur.py:83-86)."""
    return ctx.device.vec_op("pslr_apply_Es", v, ctx.q, ctx.q)


def apply_neumann(ctx: SchurContext, m: int, v):
    """sum_{i=0}^{m} (C0^{-1} Es)^i C0^{-1} v by the Horner recurrence (schur.py:89-101)."""
    return ctx.device.vec_op("pslr_apply_neumann", v, ctx.q, ctx.q, _m(m))


def apply_Err(ctx: SchurContext, m: int, v):
    """(Es C0^{-1})^{m+1} v (schur.py:104-112)."""
    return ctx.device.vec_op("pslr_apply_Err", v, ctx.q, ctx.q, _m(m))


class ErrOperator:
    """op = apply_Err(ctx, m, .) as an object the device Arnoldi recognises
    (preconditioner.py:134 passes a lambda; `lowrank.arnoldi` runs on the GPU when
    handed this operator)."""

    def __init__(self, ctx: SchurContext, m: int):
        self.ctx = ctx
        self.m = _m(m)

    def __call__(self, v):
        return apply_Err(self.ctx, self.m, v)
