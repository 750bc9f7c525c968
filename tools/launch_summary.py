"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum CSV), optionally only
after the last launch of a marker kernel (e.g. the end of the preconditioner build)."""
import collections
import csv
import sys

path = sys.argv[1]
after = sys.argv[2] if len(sys.argv) > 2 else None
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
seq = [(r[ik].split("(")[0].replace("void ", ""), float(r[iv].replace(",", ""))) for r in data]
if after:
    last = max(i for i, (n, _) in enumerate(seq) if n.startswith(after))
    seq = seq[last + 1:]
tot, cnt = collections.defaultdict(float), collections.Counter()
for name, v in seq:
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:45s} {cnt[k]:6d} {tot[k] / 1e3:10.1f} us  avg {tot[k] / cnt[k] / 1e3:8.2f}  {tot[k] / T * 100:5.1f}%")
if iters:
    print(f"{T / 1e3 / iters:.1f} us per iteration ({iters})")
for k in sorted(tot):
    if k.startswith("cgs_pass"):
        print(k, [round(v / 1e3, 1) for n, v in seq if n == k][-50:])
