"""Per-level floor of the fused solve: B^{-1} on a 1D Laplacian, whose ILU factors are
bidiagonal, so every block is a chain of one-row levels (levels = rows per block).
usage: python tools/level_floor.py [n] [s]"""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph  # noqa: E402
from paper_2002_00917_b200.schur import build_schur_context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32 * 20000
s = int(sys.argv[2]) if len(sys.argv) > 2 else 32
A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
spec = partition_graph(A, s, seed=0)
system = classify_and_reorder(A, spec)
ctx = build_schur_context(system, droptol=1e-2)
info = ctx.device.info()
p = system.p
x = torch.randn(p, dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.device.vec_op("pslr_solve_B", x, p, p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    ctx.device.vec_op("pslr_solve_B", x, p, p)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
lev = info["maxdepth_LB"] + info["maxdepth_UB"]
print(f"n={n} s={s} p={p}: solve_B {ms:.3f} ms; max levels L+U {lev}; {ms * 1e6 / lev:.1f} ns/level "
      f"= {ms * 1e6 / lev * 1.965:.0f} cycles/level @1.965 GHz")
