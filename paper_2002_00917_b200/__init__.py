"""B200-native hot path of the PSLR preconditioner (arXiv 2002.00917).

A drop-in for the reference package `pslr` on its hot path: the same
build / apply / apply_original / gmres / arnoldi / Schur-operator API
(pslr/__init__.py:11-43), with every repeated operation — the block ILU
triangular solves, the E/F/C SpMVs, the Horner power series, the rank-r
correction, the Arnoldi and GMRES Gram-Schmidt reductions — running in
hand-written sm_100a kernels (libpslr.so, reached through a C-ABI).
Partitioning, reordering and ILUT factorisation stay host setup, as in the
reference, restated in native C++ with bit-identical results.

There is no CPU fallback: importing the package requires libpslr.so, and
every hot-path operator requires a CUDA device.
"""

from ._lib import CorrectionSingularError
from .ilu import BlockILU, IluFactor, factor_blocks, ilut
from .krylov import NotSpdError, SolveReport, cg, cg_device, fgmres, gmres, gmres_device
from .lowrank import LowRankCorrection, apply_correction, arnoldi, arnoldi_device, build_correction
from .partition import PartitionedSystem, PartitionSpec, classify_and_reorder, partition_graph
from .preconditioner import FillStats, PslrConfig, PslrPreconditioner, build, with_correction
from .schur import (ErrOperator, SchurContext, apply_Err, apply_Es, apply_neumann, apply_S,
                    build_schur_context, solve_B, solve_C0)
from .sparse import Permutation, canonical, extract_submatrix, matvec, permute_symmetric
from .sweep import SWEEP_COLUMNS, sweep

__version__ = "0.1.0"

__all__ = [
    "CorrectionSingularError", "BlockILU", "IluFactor", "factor_blocks", "ilut", "NotSpdError",
    "SolveReport", "cg", "cg_device", "fgmres", "gmres", "gmres_device", "LowRankCorrection", "apply_correction",
    "arnoldi", "arnoldi_device", "build_correction", "PartitionedSystem", "PartitionSpec",
    "classify_and_reorder", "partition_graph", "FillStats", "PslrConfig", "PslrPreconditioner",
    "build", "with_correction", "ErrOperator", "SchurContext", "apply_Err", "apply_Es",
    "apply_neumann", "apply_S", "build_schur_context", "solve_B", "solve_C0", "Permutation",
    "canonical", "extract_submatrix", "matvec", "permute_symmetric", "SWEEP_COLUMNS", "sweep",
]
