"""Profiling driver: build one BASELINE workload and run a few PSLR applies (for ncu).
usage: python tools/prof_apply.py [cfg5] [n_applies] [nv]   (nv > 1: pslr_apply_multi calls)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
napply = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = workloads.CONFIGS[name]
P = pg.build(wl.matrix(), wl.config())
print({k: v for k, v in P.device.info().items()}, flush=True)
b = torch.from_numpy(np.random.default_rng(0).standard_normal(P.system.n)).cuda()
nv = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if nv > 1:
    from paper_2002_00917_b200 import _lib
    P.device.ensure_correction(P.correction)
    B = torch.from_numpy(np.random.default_rng(0).standard_normal((nv, P.system.n))).cuda()
    Z = torch.empty_like(B)
    for _ in range(napply):
        _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, wl.m, nv, B.data_ptr(), Z.data_ptr(),
                                                P.device.stream()))
    z = Z
else:
    for _ in range(napply):
        z = P.apply(b)
torch.cuda.synchronize()
print("done", float(z.norm()))
