"""Per-step cycle breakdown of the level loop (trace build 3) on the 1D-chain floor workload.
usage: PSLR_LIB=lib_variants/trace3/libpslr.so PSLR_TRACE=1 python tools/trace_floor.py [n] [s]"""
import ctypes
import os
import sys

import numpy as np
import scipy.sparse as sp

os.environ.setdefault("PSLR_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_00917_b200 import _lib  # noqa: E402
from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph  # noqa: E402
from paper_2002_00917_b200.schur import build_schur_context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32 * 2000
s = int(sys.argv[2]) if len(sys.argv) > 2 else 32
if len(sys.argv) > 3 and sys.argv[3] == "cfg5":
    from paper_2002_00917_b200 import workloads
    A = workloads.CONFIGS["cfg5"].matrix(); s = 32
else:
    A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
system = classify_and_reorder(A, partition_graph(A, s, seed=0))
ctx = build_schur_context(system, droptol=1e-2)
p = system.p
x = torch.randn(p, dtype=torch.float64, device="cuda")
ctx.device.vec_op("pslr_solve_B", x, p, p)
torch.cuda.synchronize()
buf = np.zeros(2 * (1 << 20), dtype=np.int64)
cnt = ctypes.c_int64()
_lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt))
ctx.device.vec_op("pslr_solve_B", x, p, p)
torch.cuda.synchronize()
_lib.check(_lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt)))
nn = cnt.value
ev = buf[:2 * nn].reshape(nn, 2)
codes = ev[:, 0] >> 32
args = ev[:, 0] & 0xffffffff
clk = ev[:, 1]
# steps: 50 (top, after barrier) -> 52 (row computed) -> 53 (next ops loaded) -> 54 (header) -> 50
i50 = np.flatnonzero(codes == 50)
want_upper = int(os.environ.get("UPPER", "-1"))
d = {"compute": [], "load_ops": [], "next_hdr": [], "barrier_to_top": []}
for a, b in zip(i50[:-1], i50[1:]):
    if want_upper >= 0 and ((args[a] >> 24) & 1) != want_upper:
        continue
    seg = codes[a:b + 1]
    t = clk[a:b + 1]
    try:
        i52 = a + int(np.flatnonzero(seg == 52)[0]); i53 = a + int(np.flatnonzero(seg == 53)[0]); i54 = a + int(np.flatnonzero(seg == 54)[0])
    except IndexError:
        continue
    d["compute"].append(clk[i52] - clk[a]); d["load_ops"].append(clk[i53] - clk[i52])
    d["next_hdr"].append(clk[i54] - clk[i53]); d["barrier_to_top"].append(clk[b] - clk[i54])
for k, v in d.items():
    v = np.array(v)
    print(f"{k:>15}: mean {v.mean():7.1f} median {np.median(v):7.1f} p90 {np.percentile(v, 90):7.1f} (n={v.size})")
tot = np.diff(clk[i50])
if want_upper >= 0:
    tot = tot[((args[i50[:-1]] >> 24) & 1) == want_upper]
print(f"step total: mean {tot.mean():.1f} median {np.median(tot):.1f}")
