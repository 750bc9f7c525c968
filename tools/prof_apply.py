"""Profiling driver: build one BASELINE workload and run a few PSLR applies (for ncu).
usage: python tools/prof_apply.py [cfg5] [n_applies]"""
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
for _ in range(napply):
    z = P.apply(b)
torch.cuda.synchronize()
print("done", float(z.norm()))
