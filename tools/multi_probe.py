"""Aggregate apply throughput: K streams (clone contexts) x NV vectors per call."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import _lib, workloads  # noqa: E402

wl = workloads.CONFIGS["cfg5"]
P = pg.build(wl.matrix(), wl.config())
P.device.ensure_correction(P.correction)
n, m = P.system.n, wl.m
B = torch.as_tensor(np.random.default_rng(0).standard_normal((8, n)), device="cuda").contiguous()
fn = _lib.fns["pslr_apply_multi"]
for K, NV in [(1, 1), (1, 2), (4, 2), (6, 2), (8, 2), (8, 1)]:
    devs = [P.device] + [P.device.clone() for _ in range(K - 1)]
    streams = [torch.cuda.Stream() for _ in range(K)]
    Z = [torch.empty((NV, n), dtype=torch.float64, device="cuda") for _ in range(K)]

    def run(calls):
        main = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s in streams:
            s.wait_stream(main)
        for k in range(calls):
            j = k % K
            v0 = (k * NV) % (8 - NV + 1)
            _lib.check(fn(devs[j].handle, m, NV, B[v0].data_ptr(), Z[j].data_ptr(), streams[j].cuda_stream))
        for s in streams:
            main.wait_stream(s)
        e1.record(main)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    run(2 * K)
    calls = max(40, 200 // NV)
    ms = run(calls)
    print(f"K={K} NV={NV}: {ms / (calls * NV):.4f} ms per apply (aggregate), {ms / calls:.3f} ms per call", flush=True)
    del devs
