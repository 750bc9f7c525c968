"""Synthetic workloads of BASELINE.json (seeded; no datasets are involved).

Generators follow pslr/problems.py (h^2-scaled 7-point operators, x fastest,
problems.py:40-73); `upwind3d` is config 3's first-order upwind
convection-diffusion, which the reference does not ship.
Each config returns the matrix plus the PslrConfig / Krylov settings.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .preconditioner import PslrConfig
from .sparse import canonical


def _axis(n: int, sub: float, diag: float, sup: float) -> sp.csr_matrix:
    return sp.diags([np.full(n - 1, sub), np.full(n, diag), np.full(n - 1, sup)], [-1, 0, 1],
                    format="csr")


def _kron3(Dx, Dy, Dz, nx, ny, nz):
    Ix, Iy, Iz = (sp.identity(k, format="csr") for k in (nx, ny, nz))
    return sp.kron(Iz, sp.kron(Iy, Dx)) + sp.kron(Iz, sp.kron(Dy, Ix)) + sp.kron(Dz, sp.kron(Iy, Ix))


def convdiff3d(nx, ny, nz, shift=0.0, gamma=(0.0, 0.0, 0.0)) -> sp.csr_matrix:
    """Centered convection-diffusion minus shift*I (problems.py:48-66)."""
    h = 1.0 / (nx + 1)
    ts = [h * g / 2.0 for g in gamma]
    A = _kron3(*(_axis(k, -1.0 + t, 2.0, -1.0 - t) for k, t in zip((nx, ny, nz), ts)), nx, ny, nz)
    if shift != 0.0:
        A = A - shift * sp.identity(nx * ny * nz)
    return canonical(A)


def laplacian3d(nx, ny, nz, shift=0.0) -> sp.csr_matrix:
    """Shifted 7-point Laplacian, diagonal 6 - shift (problems.py:69-73); nz=1 gives the
    5-point 2D operator with diagonal 4 - (shift - 2)."""
    return convdiff3d(nx, ny, nz, shift)


def upwind3d(nx, ny, nz, shift, hv) -> sp.csr_matrix:
    """7-point diffusion + first-order upwind convection, velocity (1,1,1), minus shift*I.
    Per axis: +hv on the diagonal, -hv on the upstream (i-1) neighbour; hv = h|v|/D
    (the "cell Peclet" reading recorded in DESIGN.md)."""
    A = _kron3(*(_axis(k, -1.0 - hv, 2.0 + hv, -1.0) for k in (nx, ny, nz)), nx, ny, nz)
    A = A - shift * sp.identity(nx * ny * nz)
    return canonical(A)


@dataclass(frozen=True)
class Workload:
    name: str
    grid: tuple
    kind: str            # "lap" | "upwind"
    shift: float
    s: int
    m: int
    rank: int
    restart: int
    tol: float = 1e-6
    maxit: int = 500
    flexible: bool = False
    hv: float = 0.0

    def matrix(self) -> sp.csr_matrix:
        nx, ny, nz = self.grid
        if self.kind == "upwind":
            return upwind3d(nx, ny, nz, self.shift, self.hv)
        return laplacian3d(nx, ny, nz, self.shift)

    def config(self, droptol=1e-2, seed=0) -> PslrConfig:
        return PslrConfig(num_subdomains=self.s, series_degree=self.m, rank=self.rank,
                          droptol=droptol, seed=seed)

    @property
    def n(self) -> int:
        return int(np.prod(self.grid))


# cfg4's literal shift: s2 = 0.01*4*(1-cos(pi/2049))*2049^2 on top of the 2D diagonal 4
_CFG4_S2 = 0.01 * 4 * (1 - math.cos(math.pi / 2049)) * 2049 ** 2

CONFIGS = {
    # BASELINE.json configs[0..4]; 2D grids are laplacian3d(nx, ny, 1, shift=2+s2)
    "cfg1": Workload("cfg1", (64, 64, 1), "lap", 2.3, 4, 3, 16, 50),
    "cfg2": Workload("cfg2", (64, 64, 64), "lap", 0.5, 16, 3, 32, 50),
    "cfg3": Workload("cfg3", (128, 128, 128), "upwind", 0.2, 64, 5, 64, 50, flexible=True, hv=0.5),
    "cfg4": Workload("cfg4", (2048, 2048, 1), "lap", 2.0 + _CFG4_S2, 128, 5, 128, 100),
    # weak-scaling apply sweep: 128^3 per GPU stacked in z, 32 subdomains per GPU
    "cfg5": Workload("cfg5", (128, 128, 128), "lap", 0.5, 32, 3, 64, 0),
    # converging known-answer twins (reference its 288 / 97)
    "twin_cfg2": Workload("twin_cfg2", (32, 32, 32), "lap", 0.16, 16, 3, 32, 50),
    "twin_cfg3": Workload("twin_cfg3", (32, 32, 32), "upwind", 0.2, 16, 5, 64, 50, flexible=True,
                          hv=0.5),
}


def cfg5(gpus: int = 1) -> Workload:
    """Config 5 at G GPUs: a 128 x 128 x (128 G) grid with 32 G subdomains."""
    return Workload(f"cfg5_g{gpus}", (128, 128, 128 * gpus), "lap", 0.5, 32 * gpus, 3, 64, 0)


def seeded_rhs(A, seed: int = 0) -> np.ndarray:
    """b = A x*, x* ~ N(0,1) from default_rng(seed) (cli.py:126-128)."""
    return A @ np.random.default_rng(seed).standard_normal(A.shape[0])
