"""Golden CG fixtures (krylov.py:132-174) from the REAL reference: tests/golden/cg_cases.json.

Build container only (imports /root/reference/pkg/src, absent on the GPU box):

    python tests/golden/make_golden_cg.py

Cases follow the reference's own CG call sites: the CLI's `--krylov cg` solve
(cli.py:131-143 with cli.py:138-139: reordered system, apply_A = Ap @ v, M = P.apply,
b = A x*, x* = default_rng(seed)) on SPD Laplacians, as tests/test_cli.py:66-70 runs
it (lap3d:6,6,6,0.0, s=4, rank 0), and the unpreconditioned failure contract of
tests/test_krylov.py:129-136.
"""

import json
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, "/root/reference/pkg/src")

from pslr.krylov import cg  # noqa: E402
from pslr.preconditioner import PslrConfig, build  # noqa: E402
from pslr.problems import ProblemSpec, laplacian3d  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (grid, shift, s, m, rank, tol, maxit)
    "cli_lap3d6_s4_r0": ((6, 6, 6), 0.0, 4, 3, 0, 1e-8, 500),
    "lap3d12_s8_r0_m1": ((12, 12, 12), 0.0, 8, 1, 0, 1e-8, 500),
    "lap3d12_s8_r0_m3": ((12, 12, 12), 0.0, 8, 3, 0, 1e-10, 500),
    "lap3d10_s4_r0_m3_maxit5": ((10, 10, 10), 0.0, 4, 3, 0, 1e-14, 5),
}


def main():
    out = {}
    for name, (grid, shift, s, m, rank, tol, maxit) in CASES.items():
        A = laplacian3d(ProblemSpec(*grid, shift=shift))
        P = build(A, PslrConfig(num_subdomains=s, series_degree=m, rank=rank))
        ps = P.system
        perm = ps.perm
        b = A @ np.random.default_rng(0).standard_normal(A.shape[0])
        bp = b[perm.inverse]
        Ap = ps.matrix
        x, rep = cg(lambda v: Ap @ v, P.apply, bp, tol=tol, maxit=maxit)
        out[name] = {"grid": list(grid), "shift": shift, "s": s, "m": m, "rank": rank, "tol": tol,
                     "maxit": maxit, "converged": bool(rep.converged), "iterations": int(rep.iterations),
                     "final_relres": float(rep.final_relres), "history": [float(h) for h in rep.history],
                     "x_reordered_norm": float(np.linalg.norm(x))}
        print(name, rep.converged, rep.iterations, rep.final_relres)
    # unpreconditioned failure contract (test_krylov.py:129-136)
    A1 = sp.diags([-np.ones(399), 2 * np.ones(400), -np.ones(399)], [-1, 0, 1], format="csr")
    x, rep = cg(lambda v: A1 @ v, None, np.ones(400), tol=1e-14, maxit=10)
    out["lap1d400_noprec_maxit10"] = {"converged": bool(rep.converged), "iterations": int(rep.iterations),
                                      "history": [float(h) for h in rep.history]}
    with open(os.path.join(HERE, "cg_cases.json"), "w") as fh:
        json.dump({"_generated_by": "tests/golden/make_golden_cg.py (pslr 0.1.0 reference, in place)",
                   "cases": out}, fh, indent=1)


if __name__ == "__main__":
    main()
