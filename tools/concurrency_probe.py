"""Aggregate apply throughput with K independent contexts on K streams (the apply sweep's
1000 applies are independent; one step-kernel launch occupies only s = 32 of 148 SMs)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import _lib, workloads  # noqa: E402
from paper_2002_00917_b200.device import DeviceContext  # noqa: E402

wl = workloads.CONFIGS["cfg5"]
P = pg.build(wl.matrix(), wl.config())
n, m = P.system.n, wl.m
ctxs = [P.device]
for _ in range(int(sys.argv[1]) - 1 if len(sys.argv) > 1 else 3):
    d = DeviceContext(P.system, P.ctx.b_ilu, P.ctx.c0_ilu, P.ctx.C0, P.ctx.Cg)
    d.set_correction(torch.as_tensor(np.ascontiguousarray(P.correction.V), device="cuda"), P.correction.G)
    ctxs.append(d)
K = len(ctxs)
streams = [torch.cuda.Stream() for _ in range(K)]
rng = np.random.default_rng(0)
vecs = [torch.from_numpy(rng.standard_normal(n)).cuda() for _ in range(8)]
outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(K)]
fn = _lib.fns["pslr_apply"]


def run(steps):
    main = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s in streams:
        s.wait_stream(main)
    for k in range(steps):
        j = k % K
        _lib.check(fn(ctxs[j].handle, m, vecs[k % 8].data_ptr(), outs[j].data_ptr(), streams[j].cuda_stream))
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


run(8)
for steps in (200,):
    ms = run(steps)
    print(f"K={K}: {ms / steps:.3f} ms per apply (aggregate over {steps} applies)")
# correctness: every context gives the same bits
z = [None] * K
for j in range(K):
    _lib.check(fn(ctxs[j].handle, m, vecs[0].data_ptr(), outs[j].data_ptr(), streams[j].cuda_stream))
torch.cuda.synchronize()
print("identical across contexts:", all(torch.equal(outs[0], outs[j]) for j in range(K)))
