"""Time the three CGS2 passes (pslr_cgs_pass modes 0/1/2) on an n x k column-major basis.
usage: python tools/time_cgs.py [n] ; prints us per pass and the HBM fraction (8 n k bytes)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_00917_b200 import _lib, operators  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128 ** 3
ld = (n + 31) // 32 * 32
if (ld // 32) % 2 == 0:
    ld += 32
ws = operators.workspace(0).handle
st = torch.cuda.current_stream().cuda_stream
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6544.0
for k in (5, 10, 25, 50):
    X = torch.randn(k * ld, dtype=torch.float64, device="cuda")
    w = torch.randn(n, dtype=torch.float64, device="cuda")
    h0 = torch.randn(k, dtype=torch.float64, device="cuda") * 1e-3
    out = torch.empty(k, dtype=torch.float64, device="cuda")
    res = []
    for mode in (0, 1, 2):
        for _ in range(3):
            _lib.check(_lib.fns["pslr_cgs_pass"](ws, mode, X.data_ptr(), ld, n, k, w.data_ptr(), h0.data_ptr(), out.data_ptr(), st))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            _lib.check(_lib.fns["pslr_cgs_pass"](ws, mode, X.data_ptr(), ld, n, k, w.data_ptr(), h0.data_ptr(), out.data_ptr(), st))
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        res.append(f"mode{mode} {us:7.1f} us ({8 * n * k / us / 1e3 / peak:5.1%})")
    print(f"k={k:3d}: " + "  ".join(res), flush=True)
