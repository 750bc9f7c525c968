"""Profiling driver: cfg5 build + one device GMRES(50) of `maxit` iterations (for ncu)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import workloads  # noqa: E402
from paper_2002_00917_b200.krylov import gmres_device  # noqa: E402

maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 60
wl = workloads.CONFIGS["cfg5"]
P = pg.build(wl.matrix(), wl.config())
b = torch.from_numpy(P.system.matrix @ np.random.default_rng(0).standard_normal(P.system.n)).cuda()
gmres_device(P, b, tol=1e-6, maxit=5, restart=50)
torch.cuda.synchronize()
t = time.perf_counter()
x, rep = gmres_device(P, b, tol=1e-6, maxit=maxit, restart=50)
torch.cuda.synchronize()
print(f"gmres {rep.iterations} its {time.perf_counter() - t:.3f} s, {1e3 * (time.perf_counter() - t) / rep.iterations:.3f} ms/it")
