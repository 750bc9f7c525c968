"""Level-merged factors (PSLR_MERGE) vs the reference's factors: single-stream apply time,
solve_B / solve_C0 times and the merged apply's relative error against the exact one.
usage: python tools/merge_ab.py [cfg5 cfg2 ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import _lib, workloads  # noqa: E402


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name in (sys.argv[1:] or ["cfg5"]):
    wl = workloads.CONFIGS[name]
    A = wl.matrix()
    res = {}
    for mode in (os.environ.get("MODES", "0,1,2,3").split(",")):
        os.environ["PSLR_MERGE"] = mode
        P = pg.build(A, wl.config(), device=0)
        dev = P.device
        info = dev.info()
        n, p, q, m = P.system.n, P.system.p, P.system.q, wl.m
        b = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
        z = torch.empty(n, dtype=torch.float64, device="cuda")
        fn = _lib.fns["pslr_apply"]
        s = torch.cuda.current_stream().cuda_stream
        t = timeit(lambda: _lib.check(fn(dev.handle, m, b.data_ptr(), z.data_ptr(), s)))
        torch.cuda.synchronize()
        x = torch.randn(p, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
        g = torch.randn(q, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
        tb = timeit(lambda: dev.vec_op("pslr_solve_B", x, p, p))
        tc = timeit(lambda: dev.vec_op("pslr_solve_C0", g, q, q))
        res[mode] = (z.clone(), dev.vec_op("pslr_solve_B", x, p, p).clone(), dev.vec_op("pslr_solve_C0", g, q, q).clone())
        z0, xb0, yc0 = res[next(iter(res))]
        rel = lambda a, c: float(torch.linalg.norm(a - c) / torch.linalg.norm(c))  # noqa: E731
        print(f"{name} merge={mode}: apply {t * 1e3:.1f} us, solve_B {tb * 1e3:.1f} us, solve_C0 {tc * 1e3:.1f} us | "
              f"depth LB {info['maxdepth_LB']} UB {info['maxdepth_UB']} LC {info['maxdepth_LC']} UC {info['maxdepth_UC']} | "
              f"rel vs first mode: apply {rel(z, z0):.2e} solve_B {rel(res[mode][1], xb0):.2e} "
              f"solve_C0 {rel(res[mode][2], yc0):.2e}", flush=True)
        del P, dev
        torch.cuda.empty_cache()
