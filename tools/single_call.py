"""Time one P.apply(numpy) call on cfg5 (the reference API's end to end) for pinned-chunk sizes."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import device, workloads  # noqa: E402

wl = workloads.CONFIGS["cfg5"]
P = pg.build(wl.matrix(), wl.config())
b = np.random.default_rng(0).standard_normal(P.system.n)
for chunk in [int(c) for c in (sys.argv[1:] or ["262144"])]:
    device._PIN_CHUNK = chunk
    for _ in range(3):
        P.apply(b)
    t0 = time.perf_counter()
    for _ in range(20):
        P.apply(b)
    print(f"chunk {chunk}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per P.apply(numpy)", flush=True)
