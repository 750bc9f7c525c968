"""Golden sweep CSVs (cli.py:200-266, `pslr sweep`) from the REAL reference:
tests/golden/sweep_cases.json.  Build container only (imports /root/reference/pkg/src):

    python tests/golden/make_golden_sweep.py

Cases: the reference CLI tests' sweeps (pkg/tests/test_cli.py:97-124 on lap3d:6,6,6,0.0)
and acceptance criterion 07's series-degree sweep at 32^3 (test_acceptance.py:153-166:
shift 0.16, s=35, rank 15, seed 2, m = 0..5; reference its [309,190,167,148,127,121]),
run through the CLI's sweep driver (one partition + ILU shared across m, one Arnoldi
truncated per rank).
"""

import json
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")

from pslr.cli import main  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    "cli_m_sweep": ["--problem", "lap3d:6,6,6,0.0", "--s", "4", "--rank", "6", "--axis", "m",
                    "--values", "0,1,2"],
    "cli_rank_sweep": ["--problem", "lap3d:6,6,6,0.0", "--s", "4", "--axis", "rank",
                       "--values", "0,4,8"],
    "cli_s_sweep": ["--problem", "lap3d:6,6,6,0.0", "--rank", "4", "--axis", "s", "--values", "2,4"],
    "lap3d12_rank_sweep_gmres20": ["--problem", "lap3d:12,12,12,0.3", "--s", "8", "--restart", "20",
                                   "--axis", "rank", "--values", "0,2,8,16"],
    "crit07_m_sweep": ["--problem", "lap3d:32,32,32,0.16", "--s", "35", "--rank", "15", "--seed", "2",
                       "--axis", "m", "--values", "0,1,2,3,4,5"],
}


def run(args):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "sweep.csv")
        code = main(["sweep", *args, "--out", out])
        text = open(out).read()
    lines = text.strip().splitlines()
    hdr = lines[0].split(",")
    rows = [dict(zip(hdr, ln.split(","))) for ln in lines[1:]]
    return code, rows


def main_():
    out = {}
    for name, args in CASES.items():
        code, rows = run(args)
        keep = [{k: r[k] for k in ("axis", "value", "its", "converged", "fill_ilu", "fill_lowrank",
                                   "fill_total", "final_relres")} for r in rows]
        out[name] = {"args": args, "exit": code, "rows": keep}
        print(name, code, [(r["value"], r["its"], r["converged"]) for r in keep], flush=True)
    with open(os.path.join(HERE, "sweep_cases.json"), "w") as fh:
        json.dump({"_generated_by": "tests/golden/make_golden_sweep.py (pslr 0.1.0 reference CLI, in place)",
                   "cases": out}, fh, indent=1)


if __name__ == "__main__":
    main_()
