"""Summarise ncu captures into profiles/: per-kernel launch list shares and the
dominant kernel's DRAM traffic / throughput (run here, on the .ncu-rep / csv files)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append(d)
    return res


def main(rep, launches_csv, tag):
    summ = {"round": tag}
    if launches_csv and os.path.exists(launches_csv):
        rows = [r for r in csv.reader(open(launches_csv)) if r]
        hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hdr_i]
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        per = {}
        for r in rows[hdr_i + 1:]:
            if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
                continue
            name = r[ki].split("(")[0].replace("pslr::", "")
            v = float(r[vi].replace(",", ""))
            per.setdefault(name, []).append(v)
        tot = sum(sum(v) for v in per.values())
        summ["launch_list"] = {k: {"launches": len(v), "total_ns": sum(v), "share": sum(v) / tot,
                                   "mean_ns": sum(v) / len(v)} for k, v in per.items()}
    if rep and os.path.exists(rep):
        m = raw_metrics(rep)
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                "smsp__issue_active.avg.per_cycle_active", "launch__registers_per_thread",
                "smsp__inst_executed.sum"]
        caps = []
        for d in m:
            caps.append({k: d.get(k) for k in keys} | {"kernel": d.get("Kernel Name", "")[:60]})
        summ["full_capture"] = caps
        # per launch DRAM bytes of the dominant (step) kernel, in bytes
        def to_bytes(v, unit):
            f = float(v.replace(",", ""))
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        units = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                               text=True).stdout.splitlines()
        urow = list(csv.reader(units))[1]
        hdr = list(csv.reader(units))[0]
        u = dict(zip(hdr, urow))
        tr = []
        for d in m:
            if "subdomain_step" in d.get("Kernel Name", ""):
                tr.append(to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
                          + to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]))
        if tr:
            summ["horner_step_dram_bytes"] = sum(tr) / len(tr)
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    json.dump(summ, open(path, "w"), indent=1, default=str)
    print(json.dumps({k: v for k, v in summ.items() if k != "full_capture"}, indent=1, default=str)[:3000])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None, sys.argv[2] if len(sys.argv) > 2 else None,
         sys.argv[3] if len(sys.argv) > 3 else "r01")
