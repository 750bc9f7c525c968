"""Producer issue times vs consumer arrival times of the factor-stream chunks of one CTA
(trace build, PSLR_TRACE=1; PSLR_DBG=16 for the stream alone).
usage: PSLR_LIB=lib_variants/trace3/libpslr.so PSLR_TRACE=1 PSLR_DBG=16 python tools/trace_stream.py [cfg5]"""
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
p = system.p
x = torch.randn(p, dtype=torch.float64, device="cuda")
cap = 1 << 20
buf = np.zeros(2 * cap, dtype=np.int64)
cnt = ctypes.c_int64()
ctx.device.vec_op("pslr_solve_B", x, p, p)
torch.cuda.synchronize()
_lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt))
ctx.device.vec_op("pslr_solve_B", x, p, p)
torch.cuda.synchronize()
_lib.check(_lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt)))
base = 2 * 65536  # g_tma = trace + 2 + 2*65536 -> buf index 2*65536
issue = buf[base:base + 2 * 8192:2]
seen = buf[base + 1:base + 2 * 8192:2]
nbytes = buf[base + 2 * 8192:base + 3 * 8192]
tstart = buf[base + 4 * 8192:base + 5 * 8192]
troom = buf[base + 5 * 8192:base + 6 * 8192]
n = int(np.count_nonzero(issue))
tstart, troom, issue = tstart[:n], troom[:n], issue[:n]
print(f"loop start->room: median {np.median(troom - tstart):.0f}; room->issued: median {np.median(issue - troom):.0f}; "
      f"issued->next start: median {np.median(tstart[1:] - issue[:-1]):.0f}")
issue, seen, nbytes = issue[:n], seen[:n], nbytes[:n]
t0 = issue[0]
print(f"chunks {n}, bytes {nbytes.sum() / 1e6:.2f} MB, mean {nbytes.mean() / 1e3:.1f} KB")
di = np.diff(issue)
lat = seen - issue
print(f"issue interval cycles: mean {di.mean():.0f} median {np.median(di):.0f} p90 {np.percentile(di, 90):.0f}")
print(f"issue->seen cycles: mean {lat.mean():.0f} median {np.median(lat):.0f} p10 {np.percentile(lat, 10):.0f} p90 {np.percentile(lat, 90):.0f}")
print(f"span issue {(issue[-1] - t0) / 1.965e3:.1f} us, seen {(seen[-1] - t0) / 1.965e3:.1f} us")
for u in range(0, min(n, 40)):
    print(u, tstart[u] - t0, troom[u] - t0, issue[u] - t0, seen[u] - t0, nbytes[u])
