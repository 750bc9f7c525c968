"""TMA issue->land latency per chunk of one CTA in the stream-only experiment (trace build).
usage: PSLR_DBG=16 PSLR_TRACE=1 PSLR_TRACE_CTA=19 PSLR_LIB=lib_variants/trace1/libpslr.so python tools/tma_lat.py"""
import ctypes, os, sys
import numpy as np
os.environ.setdefault("PSLR_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
from paper_2002_00917_b200 import _lib, workloads  # noqa
from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph  # noqa
from paper_2002_00917_b200.schur import build_schur_context  # noqa
A = workloads.CONFIGS["cfg5"].matrix()
system = classify_and_reorder(A, partition_graph(A, 32, seed=0))
ctx = build_schur_context(system, droptol=1e-2)
p = system.p
x = torch.randn(p, dtype=torch.float64, device="cuda")
buf = np.zeros(2 * (1 << 20), dtype=np.int64)
cnt = ctypes.c_int64()
for it in range(3):
    _lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt))
    ctx.device.vec_op("pslr_solve_B", x, p, p)
    torch.cuda.synchronize()
_lib.check(_lib.fns["pslr_debug_trace"](ctx.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt)))
t = buf[2 * 65536 - 2 + 2: 2 * 65536 - 2 + 2 + 2 * 8192].reshape(-1, 2)  # debug_trace strips the 2-word header
t = buf[2 * 65536: 2 * 65536 + 2 * 8192].reshape(-1, 2)
ok = (t[:, 0] > 0) & (t[:, 1] > 0)
lat = (t[ok, 1] - t[ok, 0])
iss = np.diff(t[ok, 0])
by = buf[2 * 65536 + 2 * 8192: 2 * 65536 + 3 * 8192][:ok.size]
if os.environ.get("TMA_DUMP"):
    t0 = t[ok, 0].min()
    for u in range(min(120, ok.sum())):
        lw = buf[2 * 65536 + 3 * 8192 + u]
        print(f"{u:4d} issue {t[u,0]-t0:8d} land {t[u,1]-t0:8d} lastwarp {lw - t0 if lw else -1:8d} lat {t[u,1]-t[u,0]:6d} bytes {by[u]:6d}")
print(f"bytes {by[ok].sum()} mean {by[ok].mean():.0f} min {by[ok].min()} max {by[ok].max()}")
print(f"chunks {ok.sum()}: issue->land cycles mean {lat.mean():.0f} median {np.median(lat):.0f} p90 {np.percentile(lat, 90):.0f}; "
      f"issue interval mean {iss.mean():.0f}; total {(t[ok,1].max() - t[ok,0].min()) / 1.965e3:.1f} us")
