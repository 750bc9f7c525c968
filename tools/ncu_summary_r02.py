"""Summarise the round's ncu launch lists (tools/round_profile.sh) into profiles/ncu_summary.json:
per-launch time + DRAM bytes of one cfg5 apply with one vector (pslr_apply) and one call with
two vectors (pslr_apply_multi), the Horner-step launch's DRAM bytes (bench.py roofline
`traffic` / `frac_physical`), and the bench command's own launch list shares.
usage: python tools/ncu_summary_r02.py <launches_nv1.csv> <launches_nv2.csv> <bench_launches.csv> <tag>"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    I, K, M, U, V = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    L = {}
    for r in rows[hi + 1:]:
        if len(r) <= V:
            continue
        d = L.setdefault(int(r[I]), {"kernel": r[K].split("(")[0].replace("void ", "").replace("pslr::", "")})
        d[r[M]] = float(r[V].replace(",", "")) * SCALE.get(r[U], 1)
    return [L[k] for k in sorted(L)]


def last_call(L, first_kernel):
    """The launches of the last apply call: from the last `first_kernel` launch on."""
    i = max(j for j, d in enumerate(L) if d["kernel"].startswith(first_kernel))
    return [d for d in L[i:] if not d["kernel"].startswith("at::")]


def call_summary(call):
    out = []
    for d in call:
        out.append({"kernel": d["kernel"], "us": d["gpu__time_duration.sum"] / 1e3,
                     "dram_MB": (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / 1e6})
    return out


def main(nv1, nv2, bench, tag):
    L1, L2 = load(nv1), load(nv2)
    c1, c2 = last_call(L1, "permute_f_kernel"), last_call(L2, "permute2_kernel")
    # a Horner step = pre_step_kernel + the B launch + iface_kernel + the C0 launch (split
    # interface phase; one fused step launch before round 2's split)
    groups = []
    for i, d in enumerate(c1):
        if d["kernel"].startswith("pre_step_kernel") and i + 3 < len(c1) and \
                c1[i + 3]["kernel"].startswith("subdomain_step_kernel<1, 0") and \
                c1[i + 2]["kernel"].startswith("iface_kernel"):
            groups.append(c1[i:i + 4])
    if not groups:
        groups = [[d] for d in c1 if d["kernel"].startswith("subdomain_step_kernel<1, 1")][1:4]
    hb = sum(sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in g) for g in groups) / len(groups)
    ht = sum(sum(d["gpu__time_duration.sum"] for d in g) for g in groups) / len(groups)
    summ = {"round": tag,
            "horner_step_dram_bytes": hb,
            "horner_step_us_ncu": ht / 1e3,
            "apply1_call_dram_bytes": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in c1),
            "apply1_call_us_ncu": sum(d["gpu__time_duration.sum"] for d in c1) / 1e3,
            "apply2_call_dram_bytes": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in c2),
            "apply2_call_us_ncu": sum(d["gpu__time_duration.sum"] for d in c2) / 1e3,
            "apply1_launches": call_summary(c1), "apply2_launches": call_summary(c2),
            "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                    "--clock-control none: serialised, cold-cache launches (tools/round_profile.sh)"}
    if bench and os.path.exists(bench):
        rows = [r for r in csv.reader(open(bench)) if r]
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hi]
        K, M, V = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        per = {}
        for r in rows[hi + 1:]:
            if len(r) > V and r[M] == "gpu__time_duration.sum":
                per.setdefault(r[K].split("(")[0].replace("void ", "").replace("pslr::", ""), []).append(
                    float(r[V].replace(",", "")))
        tot = sum(sum(v) for v in per.values())
        summ["bench_launch_list"] = {k: {"launches": len(v), "total_ns": sum(v), "share": sum(v) / tot}
                                     for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}
    json.dump(summ, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in summ.items() if not k.endswith("launches") and k != "bench_launch_list"},
                     indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4], sys.argv[4] if len(sys.argv) > 4 else "r02")
