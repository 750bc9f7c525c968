"""Time the rank-r correction (pslr_apply_correction: V^T y, G, y + V u) on cfg5 with CUDA
events (single stream), for A/B of library variants (PSLR_LIB)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import workloads  # noqa: E402

wl = workloads.CONFIGS["cfg5"]
P = pg.build(wl.matrix(), wl.config())
q = P.system.q
y = torch.from_numpy(np.random.default_rng(0).standard_normal(q)).cuda()
for _ in range(5):
    pg.apply_correction(P.correction, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    out = pg.apply_correction(P.correction, y)
e1.record()
torch.cuda.synchronize()
print(f"correction: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us per call ({os.environ.get('PSLR_LIB', 'default')})")
