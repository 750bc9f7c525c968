"""Per-level cycle cost of the level loop vs level width (trace build 3, PSLR_TRACE=1).
usage: PSLR_LIB=lib_variants/trace3/libpslr.so PSLR_TRACE=1 PSLR_TRACE_CTA=b python tools/trace_levels.py [cfg5] [B|C0]
Records: code 50 at the top of every level-loop step of consumer thread 0, arg = segment rows |
flags << 16 | min(w,15) << 20 | upper << 24.  A level = the steps up to one with flag bit0."""
import ctypes
import os
import sys

import numpy as np

os.environ.setdefault("PSLR_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_00917_b200 import _lib, workloads  # noqa: E402
from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph  # noqa: E402
from paper_2002_00917_b200.schur import build_schur_context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
which = sys.argv[2] if len(sys.argv) > 2 else "B"
wl = workloads.CONFIGS[name]
A, s = wl.matrix(), wl.s
system = classify_and_reorder(A, partition_graph(A, s, seed=0))
ctx = build_schur_context(system, droptol=1e-2)
n = system.p if which == "B" else system.q
op = "pslr_solve_B" if which == "B" else "pslr_solve_C0"
x = torch.randn(n, dtype=torch.float64, device="cuda")
buf = np.zeros(2 * (1 << 20), dtype=np.int64)
cnt = ctypes.c_int64()
ctx.device.vec_op(op, x, n, n)
torch.cuda.synchronize()
_lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt))
ctx.device.vec_op(op, x, n, n)
torch.cuda.synchronize()
_lib.check(_lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt)))
nn = cnt.value
ev = buf[:2 * nn].reshape(nn, 2)
codes = ev[:, 0] >> 32
args = ev[:, 0] & 0xffffffff
clk = ev[:, 1]
i50 = np.flatnonzero(codes == 50)
rows = args[i50] & 0xffff
flags = (args[i50] >> 16) & 0xf
w = (args[i50] >> 20) & 0xf
up = (args[i50] >> 24) & 1
dt = np.diff(clk[i50])
# a phase boundary: upper flag changes -> drop that step
levels = []  # (upper, rows, segments, maxw, cycles)
cur = None
for k in range(len(i50) - 1):
    if up[k + 1] != up[k] and not (flags[k] & 1):
        pass
    if cur is None:
        cur = [int(up[k]), 0, 0, 0, 0]
    cur[1] += int(rows[k]); cur[2] += 1; cur[3] = max(cur[3], int(w[k])); cur[4] += int(dt[k])
    if flags[k] & 1:
        levels.append(cur)
        cur = None
L = np.array(levels)
tot = L[:, 4].sum()
print(f"{name} {which} CTA {os.environ.get('PSLR_TRACE_CTA', '0')}: {len(L)} levels, {tot} cycles ({tot / 1.965e3:.1f} us)")
for u in (0, 1):
    M = L[L[:, 0] == u]
    if not len(M):
        continue
    print(f" {'U' if u else 'L'}: {len(M)} levels, cycles {M[:, 4].sum()} ({M[:, 4].sum() / 1.965e3:.1f} us), "
          f"mean {M[:, 4].mean():.0f} cyc/level, rows/level mean {M[:, 1].mean():.0f}")
    for lo, hi in ((1, 1), (2, 32), (33, 64), (65, 128), (129, 256), (257, 480), (481, 960), (961, 1 << 20)):
        sel = (M[:, 1] >= lo) & (M[:, 1] <= hi)
        if sel.any():
            c = M[sel, 4]
            print(f"   rows {lo:>4}-{hi:<7}: {sel.sum():4d} levels, cyc/level mean {c.mean():6.0f} median {np.median(c):6.0f} "
                  f"p90 {np.percentile(c, 90):6.0f}; segs/level {M[sel, 2].mean():.2f}; share {c.sum() / tot:.1%}")
    # least-squares cycles = a + b*rows + c*(segs-1)
    X = np.c_[np.ones(len(M)), M[:, 1], M[:, 2] - 1]
    coef, *_ = np.linalg.lstsq(X, M[:, 4].astype(float), rcond=None)
    print(f"   fit: {coef[0]:.0f} + {coef[1]:.2f}*rows + {coef[2]:.0f}*(extra segments)")
