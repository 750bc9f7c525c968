"""Timeline of CTA 0 of the fused step kernel over one PSLR apply (PSLR_TRACE=1).
usage: PSLR_TRACE=1 python tools/trace_apply.py [cfg5] [nv]   (nv=2: one pslr_apply_multi call)"""
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
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1
b = torch.from_numpy(np.random.default_rng(0).standard_normal(P.system.n)).cuda()
if nv > 1:
    P.device.ensure_correction(P.correction)
    B2 = torch.from_numpy(np.random.default_rng(0).standard_normal((nv, P.system.n))).cuda()
    Z2 = torch.empty_like(B2)

    class _Multi:
        def apply(self, _b):
            _lib.check(_lib.fns["pslr_apply_multi"](P.device.handle, wl.m, nv, B2.data_ptr(), Z2.data_ptr(),
                                                    P.device.stream()))
    P_run = _Multi()
else:
    P_run = P
P_run.apply(b)
torch.cuda.synchronize()
buf = np.zeros(2 * (1 << 20), dtype=np.int64)  # == 2*trace_cap: whole buffer
cnt = ctypes.c_int64()
_lib.fns["pslr_debug_trace"](P.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt))  # reset
P_run.apply(b)
torch.cuda.synchronize()
_lib.check(_lib.fns["pslr_debug_trace"](P.device.handle, buf.ctypes.data, buf.size, ctypes.byref(cnt)))
n = cnt.value
ev = buf[:2 * n].reshape(n, 2)
ev = ev[ev[:, 1] != 0]
n = ev.shape[0]
codes = ev[:, 0] >> 32
args = ev[:, 0] & 0xffffffff
ts = ev[:, 1] - ev[0, 1]
# per launch: phase boundaries, level durations (between level-barrier releases, 41),
# chunk waits (19 -> 20: the consumer blocked on a chunk that had not landed)
names = {1: "start", 3: "prepass", 10: "phase0", 11: "phase1", 12: "phase2", 13: "phase3", 30: "iface"}
starts = np.flatnonzero(codes == 1)
for li, s0 in enumerate(starts):
    s1 = starts[li + 1] if li + 1 < len(starts) else n
    c, a, t = codes[s0:s1], args[s0:s1], ts[s0:s1]
    t = t - t[0]
    print(f"--- launch {li}: {t[-1] / 1e3:.1f} us, chunks {a[0]}")
    for i in range(len(c)):
        if c[i] in names and c[i] != 1:
            print(f"   {names[c[i]]:>8} at {t[i] / 1e3:8.1f} us")
    rel = t[c == 41]
    if rel.size > 2:
        lv = np.diff(rel) / 1e3
        print(f"   levels {rel.size}: mean {lv.mean():.3f} us, median {np.median(lv):.3f}, p90 {np.percentile(lv, 90):.3f}, "
              f"sum {lv.sum():.1f} us")
    i19 = np.flatnonzero(c == 19)
    w = [t[i + 1] - t[i] for i in i19 if i + 1 < len(c) and c[i + 1] == 20]
    if w:
        w = np.array(w) / 1e3
        print(f"   chunk transitions {len(w)}: waits sum {w.sum():.1f} us, mean {w.mean():.3f}, max {w.max():.2f}; "
              f"> 0.2 us: {(w > 0.2).sum()}")
# producer counters (the producer thread): idle cycles, total cycles, iterations
cyc = buf[2 * (1 << 20) - 8 * 4096:].reshape(4096, 8)[:P.system.num_parts]
if cyc[:, 7].sum() > 0:
    tot = cyc[:, 7].astype(float)
    print(f"producer: total cycles/CTA {tot.mean():.0f}, idle {cyc[:, 5].mean() / max(tot.mean(), 1):.2%}, "
          f"iterations/CTA {cyc[:, 4].mean():.0f}")

pr = buf[2 * (1 << 20) - 8 * 4096:].reshape(4096, 8)[2048:2048 + P.system.num_parts].astype(float)
if pr[:, 4].sum() > 0:
    m = pr.mean(axis=0)
    tot = m[0] + m[1] + m[2] + m[3]
    print(f"thread 0 level loop (one apply, mean over CTAs): {tot:.0f} cycles; steps {m[4]:.0f}, levels {m[5]:.0f}, chunks {m[6]:.0f}")
    for i, nm in enumerate(["chunk wait", "fold", "publish+next", "barrier"]):
        print(f"   {nm:>13}: {m[i]:11.0f} cycles ({m[i] / tot:6.1%}); per level {m[i] / max(m[5], 1):7.1f}, per step {m[i] / max(m[4], 1):7.1f}")
# PSLR_TRACE_BUILD=3: per-step clock64 records (code 50, arg = level_end | chunk_done<<1 |
# G<<2 | nrows<<8) of CTA 0: level durations in cycles by phase, rows and width
i50 = np.flatnonzero(codes == 50)
if i50.size:
    clk = ev[:, 1]
    pstarts = {int(i): int(codes[i]) for i in np.flatnonzero((codes >= 10) & (codes <= 13))}
    phase_of = np.zeros(n, dtype=np.int64)
    cur = -1
    for i in range(n):
        if i in pstarts:
            cur = pstarts[i] - 10
        phase_of[i] = cur
    stats = {}
    prev_end = None
    lv_rows, lv_g, lv_chunks, lv_segs = 0, 0, 0, 0
    for i in i50:
        a = int(args[i])
        if prev_end is None or phase_of[i] != phase_of[prev_end] or (i - prev_end) > 64:
            prev_end = i  # first step of a phase: no start reference
            lv_rows = lv_g = lv_chunks = lv_segs = 0
            continue
        lv_rows += (a >> 8) & 0xffff
        lv_g = max(lv_g, (a >> 2) & 0x3f)
        lv_chunks += (a >> 1) & 1
        lv_segs += 1
        if a & 1:
            dur = int(clk[i] - clk[prev_end])
            key = int(phase_of[i])
            stats.setdefault(key, []).append((dur, lv_rows, lv_g, lv_chunks, lv_segs))
            prev_end = i
            lv_rows = lv_g = lv_chunks = lv_segs = 0
    for k, v in sorted(stats.items()):
        v = np.array(v, dtype=np.float64)
        print(f"phase {k}: levels {len(v)}, cycles/level mean {v[:, 0].mean():.0f} median {np.median(v[:, 0]):.0f}; "
              f"rows/level {v[:, 1].mean():.0f}, segs/level {v[:, 4].mean():.2f}, chunk ends/level {v[:, 3].mean():.2f}")
        for lo, hi in ((0, 33), (33, 129), (129, 257), (257, 513), (513, 100000)):
            sel = (v[:, 1] >= lo) & (v[:, 1] < hi)
            if sel.any():
                print(f"    rows [{lo},{hi}): n={sel.sum():4d} cycles {v[sel, 0].mean():7.0f}  G {v[sel, 2].mean():.2f} "
                      f"segs {v[sel, 4].mean():.2f} chunk-ends {v[sel, 3].mean():.2f}")
i51 = np.flatnonzero(codes == 51)
if i51.size:
    w = args[i51].astype(np.int64)
    print(f"chunk transitions (CTA 0, trace build 3): n={w.size}, wait cycles mean {w.mean():.0f} median "
          f"{np.median(w):.0f} p90 {np.percentile(w, 90):.0f}; > 200 cycles: {(w > 200).mean():.1%}, "
          f"sum {w.sum() / 1.965e3:.1f} us")
    for k in sorted(set(phase_of[i51].tolist())):
        sel = phase_of[i51] == k
        print(f"   phase {k}: n={sel.sum()}, mean {w[sel].mean():.0f}, sum {w[sel].sum() / 1.965e3:.1f} us")
# per-CTA phase stamps, the last launch of each kind (trace builds): which block is critical
kinds = {2: "first_step", 3: "correction_c0", 11: "correction_c0 (C0 launch)", 4: "horner_step (B launch)",
         12: "horner_step (C0 launch)", 5: "last_step"}
names_s = ["start", "prepass", "L_B", "U_B", "L_C0", "U_C0", "end", "iface"]
area = buf[2 * (1 << 20) - 8 * 4096:].reshape(4096, 8)
dump = {}
for tag, kname in kinds.items():
    cs = area[1024 + 64 * tag:1024 + 64 * tag + P.system.num_parts].astype(np.float64)
    if cs[:, 0].sum() <= 0:
        continue
    dump[kname] = cs
    t0 = cs[:, 0].min()
    end = (cs[:, 6] - t0) / 1e3
    print("%s, per CTA (us from the first CTA start): end min %.1f median %.1f max %.1f (CTA %d)"
          % (kname, end.min(), np.median(end), end.max(), int(end.argmax())))
    order = np.argsort(-end)[:4]
    for b in order:
        row = cs[b]
        seg = []
        marks = sorted([(i, row[i]) for i in range(8) if row[i] >= row[0] > 0], key=lambda m: m[1])
        for (i, tv), (j, tn) in zip(marks, marks[1:]):
            seg.append(f"{names_s[i]} {(tn - tv) / 1e3:.1f}")
        wt = area[3072 + 64 * tag + b]
        wtxt = f"  | chunk waits {wt[0] / 1.965e3:.1f} us over {int(wt[1])} transitions ({int(wt[2])} > 200 cyc)" if wt[1] else ""
        print(f"   CTA {b:3d}: start {(row[0] - t0) / 1e3:6.1f} end {(row[6] - t0) / 1e3:6.1f}  |  " + ", ".join(seg) + wtxt)
out = os.environ.get("TRACE_DUMP")
if out:
    np.savez(out, **dump)
