"""Where a level-loop step of consumer thread 0 spends its cycles (trace build 3, PSLR_TRACE=1):
records 50 (step top) -> 52 (row computed) -> 53 (next operands loaded) -> 54 (header after
next read) -> next 50 (level barrier, register rotation).
usage: PSLR_LIB=lib_variants/trace3/libpslr.so PSLR_TRACE=1 PSLR_TRACE_CTA=b python tools/trace_steps.py [cfg5]"""
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
wl = workloads.CONFIGS[name]
A, s = wl.matrix(), wl.s
system = classify_and_reorder(A, partition_graph(A, s, seed=0))
ctx = build_schur_context(system, droptol=1e-2)
n = system.p
x = torch.randn(n, dtype=torch.float64, device="cuda")
buf = np.zeros(2 * (1 << 20), dtype=np.int64)
cnt = ctypes.c_int64()
for _ in range(2):
    ctx.device.vec_op("pslr_solve_B", x, n, n)
    torch.cuda.synchronize()
    _lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt))
nn = cnt.value
ev = buf[:2 * nn].reshape(nn, 2)
codes = (ev[:, 0] >> 32).astype(int)
args = ev[:, 0] & 0xffffffff
clk = ev[:, 1]
i50 = np.flatnonzero(codes == 50)
print(f"{name} CTA {os.environ.get('PSLR_TRACE_CTA', '0')}: {len(i50)} steps")
for up in (0, 1):
    rows_ = []
    for a, b in zip(i50[:-1], i50[1:]):
        if b - a != 4 or list(codes[a:b]) != [50, 52, 53, 54]:
            continue
        arg = int(args[a])
        if ((arg >> 24) & 1) != up:
            continue
        t = clk[a:b + 1]
        rows_.append((arg & 0xffff, (arg >> 16) & 0xf, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3]))
    if not rows_:
        continue
    R = np.array(rows_)
    print(f" {'U' if up else 'L'}: {len(R)} steps, rows/step mean {R[:, 0].mean():.0f}; total/step mean {R[:, 2:].sum(1).mean():.0f}")
    for nm, col in (("compute row (50->52)", 2), ("release + load next operands (52->53)", 3),
                    ("header after next / chunk wait (53->54)", 4), ("barrier + rotate (54->50)", 5)):
        c = R[:, col]
        print(f"   {nm:42s} mean {c.mean():6.0f} median {np.median(c):6.0f} p90 {np.percentile(c, 90):6.0f}")
    ce = (R[:, 1] & 8) != 0
    for lab, sel in (("chunk-end steps", ce), ("other steps", ~ce)):
        if sel.any():
            print(f"   {lab}: {sel.sum()} steps, total/step mean {R[sel, 2:].sum(1).mean():.0f}, "
                  f"53->54 mean {R[sel, 4].mean():.0f}, 52->53 mean {R[sel, 3].mean():.0f}")
