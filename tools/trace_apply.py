"""Timeline of CTA 0 of the fused step kernel over one PSLR apply (PSLR_TRACE=1).
usage: PSLR_TRACE=1 python tools/trace_apply.py [cfg5]"""
import ctypes
import os
import sys

import numpy as np

os.environ.setdefault("PSLR_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00917_b200 as pg  # noqa: E402
from paper_2002_00917_b200 import _lib, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
wl = workloads.CONFIGS[name]
P = pg.build(wl.matrix(), wl.config())
print(P.device.info(), flush=True)
b = torch.from_numpy(np.random.default_rng(0).standard_normal(P.system.n)).cuda()
P.apply(b)
torch.cuda.synchronize()
buf = np.zeros(2 * (1 << 20), dtype=np.int64)  # == 2*trace_cap: whole buffer
cnt = ctypes.c_int64()
_lib.fns["pslr_debug_trace"](P.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt))  # reset
P.apply(b)
torch.cuda.synchronize()
_lib.check(_lib.fns["pslr_debug_trace"](P.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt)))
n = cnt.value
ev = buf[:2 * n].reshape(n, 2)
ev = ev[ev[:, 1] != 0]
n = ev.shape[0]
codes = ev[:, 0] >> 32
args = ev[:, 0] & 0xffffffff
ts = ev[:, 1] - ev[0, 1]
# per-level timeline: a level = time between consecutive level-end barrier releases (41)
rel = np.flatnonzero(codes == 41)
arr = np.flatnonzero(codes == 40)
if rel.size > 2:
    lv = np.diff(ts[rel])
    rows = np.zeros(arr.size - 1, dtype=np.int64)
    ws = args[arr[1:]]
    wait = ts[rel] - ts[arr]
    print(f"levels {rel.size}: level us mean {lv.mean() / 1e3:.3f} median {np.median(lv) / 1e3:.3f} "
          f"p90 {np.percentile(lv, 90) / 1e3:.3f}; barrier wait (thread0) mean {wait.mean() / 1e3:.3f}")
    for lo, hi in ((0, 64), (64, 256), (256, 520)):
        sel = (rows >= lo) & (rows < hi)
        if sel.any():
            print(f"   rows [{lo},{hi}): n={sel.sum()} level us mean {lv[sel].mean() / 1e3:.3f}")
    print("   first 40 levels (us, rows, w):",
          [(round(lv[i] / 1e3, 2), int(rows[i]), int(ws[i])) for i in range(min(40, lv.size))])
names = {1: "start", 3: "prepass", 10: "phase0", 11: "phase1", 12: "phase2", 13: "phase3",
         20: "chunk_ready", 21: "chunk_done", 30: "iface"}
# summarise per launch: split at code 1
starts = np.flatnonzero(codes == 1)
for li, s0 in enumerate(starts):
    s1 = starts[li + 1] if li + 1 < len(starts) else n
    c, a, t = codes[s0:s1], args[s0:s1], ts[s0:s1]
    t = t - t[0]
    print(f"--- launch {li}: {t[-1] / 1e3:.1f} us, chunks {a[0]}")
    wait = 0.0
    work = 0.0
    last_done = None
    for i in range(len(c)):
        if c[i] in (10, 11, 12, 13, 3, 30):
            print(f"   {names[c[i]]:>8} at {t[i] / 1e3:8.1f} us")
        if c[i] == 20:
            prev = t[i - 1]
            wait += t[i] - prev
        if c[i] == 21:
            work += t[i] - t[i - 1]
    print(f"   chunk wait total {wait / 1e3:.1f} us, chunk work total {work / 1e3:.1f} us")
    ready = [(a[i], t[i]) for i in range(len(c)) if c[i] == 20]
    done = [(a[i], t[i]) for i in range(len(c)) if c[i] == 21]
    if ready:
        w = [done[i][1] - ready[i][1] for i in range(min(len(ready), len(done)))]
        print(f"   per-chunk work us: mean {np.mean(w) / 1e3:.2f} max {np.max(w) / 1e3:.2f}; "
              f"first 10: {[round(x / 1e3, 2) for x in w[:10]]}")
# fine-grained clock64 events 50..53 (thread 0): header -> rhs -> fold done -> stores done
sel = np.isin(codes, [50, 51, 52, 53])
if sel.any():
    c5, a5 = codes[sel], args[sel]
    d = {}
    for i in range(len(c5) - 1):
        if c5[i + 1] == c5[i] + 1:
            d.setdefault(int(c5[i]), []).append((int(a5[i + 1]) - int(a5[i])) & 0x7fffffff)
    for k in sorted(d):
        v = np.array(d[k])
        print(f"clock {k}->{k + 1}: n={v.size} median {np.median(v):.0f} mean {v.mean():.0f} p90 {np.percentile(v, 90):.0f} cycles")
# per-CTA cycle counters of the level loop (thread 0): header->rhs, fold, stores, barrier wait
cyc = buf[2 * (1 << 20) - 8 * 4096:].reshape(4096, 8)[:P.system.num_parts]
segs = cyc[:, 4].astype(float)
if segs.sum() > 0:
    for i, nm in enumerate(["hdr->rhs", "fold", "stores", "barrier"]):
        per = cyc[:, i] / np.maximum(segs, 1)
        print(f"cycles/level-segment {nm:>9}: mean over CTAs {per.mean():8.1f}  min {per.min():8.1f} max {per.max():8.1f}")
    print("level-ending segments per CTA (both applies):", int(segs.mean()))
# distribution of per-chunk waits (launch with most chunks)
best = None
for li, s0 in enumerate(starts):
    s1 = starts[li + 1] if li + 1 < len(starts) else n
    cnt_c = int(np.sum(codes[s0:s1] == 20))
    if best is None or cnt_c > best[2]:
        best = (s0, s1, cnt_c)
if best and best[2] > 0:
    s0, s1, _ = best
    c, a, t = codes[s0:s1], args[s0:s1], ts[s0:s1]
    waits = []
    prev = None
    for i in range(len(c)):
        if c[i] in (21, 10, 11, 12, 13):
            prev = t[i]
        if c[i] == 20 and prev is not None:
            waits.append((t[i] - prev, int(a[i])))
    w = np.array([x[0] for x in waits]) / 1e3
    print(f"chunk waits: n={w.size} median {np.median(w):.2f} p90 {np.percentile(w, 90):.2f} max {w.max():.2f} us; "
          f"sum {w.sum():.1f}; waits > 1us: {(w > 1).sum()} totalling {w[w > 1].sum():.1f} us")
    print("   largest:", sorted(waits, reverse=True)[:8])
# producer counters (the producer thread): idle cycles, total cycles, iterations
if segs.sum() > 0 or cyc[:, 7].sum() > 0:
    tot = cyc[:, 7].astype(float)
    print(f"producer: total cycles/CTA {tot.mean():.0f}, idle {cyc[:, 5].mean() / max(tot.mean(), 1):.2%}, "
          f"iterations/CTA {cyc[:, 4].mean():.0f}")

# PSLR_PROBE build: thread-0 cycle totals of the level loop's parts (rows 2048+b)
pr = buf[2 * (1 << 20) - 8 * 4096:].reshape(4096, 8)[2048:2048 + P.system.num_parts].astype(float)
if pr.sum() > 0:
    names_p = ["loop+hdr", "rhs(+div)", "fold", "stores", "->barrier", "barrier", "chunk tail", "chunk wait"]
    tot = pr.sum(axis=1).mean()
    print(f"probe (thread 0, both applies, mean over CTAs): total {tot:.0f} cycles")
    for i, nm in enumerate(names_p):
        print(f"   {nm:>10}: {pr[:, i].mean():12.0f} cycles ({pr[:, i].mean() / tot:6.1%})")
lat = buf[2 * (1 << 20) - 8 * 4096:].reshape(4096, 8)[3072:3072 + P.system.num_parts].astype(float)
if lat[:, 2].sum() > 0:
    n_ = lat[:, 2].sum()
    print(f"latency probes: dependent LDS {lat[:, 0].sum() / n_ / 16:.1f} cycles, dependent DADD {lat[:, 1].sum() / n_ / 16:.1f} cycles (n={n_:.0f})")
if lat[:, 3].sum() > 0:
    m = lat.mean(axis=0)
    print(f"thread 0 per CTA: rows {m[3]:.0f}, entries {m[4]:.0f} (w/row {m[4] / max(m[3], 1):.1f}), levels {m[5]:.0f}, segments {m[6]:.0f}")
    if pr.sum() > 0:
        pm = pr.mean(axis=0)
        print(f"   fold cycles/row {pm[2] / m[3]:.0f}, per entry {pm[2] / max(m[4], 1):.1f}; rhs cycles/row {pm[1] / m[3]:.0f}; "
              f"stores/row {pm[3] / m[3]:.0f}; hdr/segment {pm[0] / m[6]:.0f}; barrier/level {pm[5] / m[5]:.0f}")
