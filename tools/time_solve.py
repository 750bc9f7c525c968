"""Time the device block solves (solve_B, solve_C0) and one Horner step on a workload.
usage: python tools/time_solve.py [cfg5|1d] ; PSLR_DBG bits select timing experiments."""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_00917_b200 import workloads  # noqa: E402
from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph  # noqa: E402
from paper_2002_00917_b200.schur import build_schur_context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
if name == "1d":
    n = 64000
    A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    s = 32
else:
    wl = workloads.CONFIGS[name]
    A, s = wl.matrix(), wl.s
system = classify_and_reorder(A, partition_graph(A, s, seed=0))
ctx = build_schur_context(system, droptol=1e-2)
info = ctx.device.info()
p, q = system.p, system.q
x = torch.randn(p, dtype=torch.float64, device="cuda")
g = torch.randn(q, dtype=torch.float64, device="cuda")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tb = timeit(lambda: ctx.device.vec_op("pslr_solve_B", x, p, p))
tc = timeit(lambda: ctx.device.vec_op("pslr_solve_C0", g, q, q)) if q else 0.0
te = timeit(lambda: ctx.device.vec_op("pslr_apply_Es", g, q, q)) if q else 0.0
lb = info["maxdepth_LB"] + info["maxdepth_UB"]
lc = info["maxdepth_LC"] + info["maxdepth_UC"]
print(f"{name} dbg={os.environ.get('PSLR_DBG', '0')}: solve_B {tb * 1e3:.1f} us ({tb * 1e6 / lb * 1.965:.0f} cyc/level, "
      f"{lb} levels); solve_C0 {tc * 1e3:.1f} us ({tc * 1e6 / max(lc, 1) * 1.965:.0f} cyc/level, {lc} levels); "
      f"apply_Es {te * 1e3:.1f} us", flush=True)
