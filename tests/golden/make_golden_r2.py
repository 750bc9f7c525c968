"""Round-2 golden fixtures from the REAL reference (build container only; imports the
read-only /root/reference/pkg/src):

  * setup identity at the BASELINE configs (SURVEY §8f rank 1 acceptance: "identical L/U
    and assignment on cfg1-5"): SHA-256 of the reordered matrix, the partition
    assignment, the permutation and every factor the reference's setup produces for
    cfg2, cfg3, cfg5 and cfg4 -> golden.json["setup_sha"];
  * the cfg4 twin (2D 256^2, shift 2 + 0.197392, s=16, m=5, r=128, GMRES(100),
    tol 1e-6, maxit 500; the reference fails at 500 with relres 9.21e-5): its correction
    (V, H, G), the first two GMRES cycles' residual history and the outcome ->
    golden.json["gmres"]["twin_cfg4"], apply_twin_cfg4.npz.

    python tests/golden/make_golden_r2.py [setup|twin4|all]
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402  (puts /root/reference/pkg/src on sys.path)
from pslr.partition import classify_and_reorder, partition_graph  # noqa: E402
from pslr.preconditioner import PslrConfig, build  # noqa: E402
from pslr.problems import ProblemSpec, laplacian3d  # noqa: E402
from pslr.schur import build_schur_context  # noqa: E402

S2 = 0.01 * 4 * (1 - math.cos(math.pi / 2049)) * 2049 ** 2  # cfg4's literal shift

CONFIGS = {  # (matrix, s) as BASELINE.json / paper_2002_00917_b200/workloads.py define them
    "cfg2": (lambda: laplacian3d(ProblemSpec(64, 64, 64, shift=0.5)), 16),
    "cfg3": (lambda: MG.upwind3d(128, 128, 128, 0.2, 0.5), 64),
    "cfg5": (lambda: laplacian3d(ProblemSpec(128, 128, 128, shift=0.5)), 32),
    "cfg4": (lambda: laplacian3d(ProblemSpec(2048, 2048, 1, shift=2.0 + S2)), 128),
}


def load():
    path = os.path.join(HERE, "golden.json")
    return path, json.load(open(path))


def setup_sha(names):
    path, golden = load()
    out = golden.setdefault("setup_sha", {})
    for name in names:
        mk, s = CONFIGS[name]
        t0 = time.perf_counter()
        A = mk()
        spec = partition_graph(A, s, seed=0)
        ps = classify_and_reorder(A, spec)
        t1 = time.perf_counter()
        ctx = build_schur_context(ps, droptol=1e-2)
        t2 = time.perf_counter()
        out[name] = {"s": s, "n": int(ps.n), "p": int(ps.p), "q": int(ps.q),
                     "A_sha": MG.csr_sha(A), "assignment_sha": MG.sha(spec.assignment.astype(np.int64)),
                     "forward_sha": MG.sha(ps.perm.forward.astype(np.int64)),
                     "matrix_sha": MG.csr_sha(ps.matrix),
                     "LB_sha": MG.csr_sha(ctx.b_ilu.L), "UB_sha": MG.csr_sha(ctx.b_ilu.U),
                     "LC_sha": MG.csr_sha(ctx.c0_ilu.L), "UC_sha": MG.csr_sha(ctx.c0_ilu.U),
                     "Cg_sha": MG.csr_sha(ctx.Cg),
                     "nnz_LB": int(ctx.b_ilu.L.nnz), "nnz_UB": int(ctx.b_ilu.U.nnz),
                     "secs_partition": t1 - t0, "secs_ilut": t2 - t1}
        print(name, out[name], flush=True)
        path, g2 = load()  # re-read: another generator may have written meanwhile
        g2.setdefault("setup_sha", {})[name] = out[name]
        json.dump(g2, open(path, "w"), indent=1, sort_keys=True)


def twin4():
    A = laplacian3d(ProblemSpec(256, 256, 1, shift=2.0 + S2))
    t0 = time.perf_counter()
    P = build(A, PslrConfig(num_subdomains=16, series_degree=5, rank=128, droptol=1e-2, seed=0))
    t1 = time.perf_counter()
    ps, ctx, lr = P.system, P.ctx, P.correction
    rep, secs = MG.solve_reordered(A, P, tol=1e-6, maxit=500, restart=100)
    out = {"V": lr.V, "H": lr.H, "G": lr.G}
    MG.csr_parts("A", A, out)
    np.savez_compressed(os.path.join(HERE, "apply_twin_cfg4.npz"), **out)
    path, golden = load()
    golden.setdefault("apply", {})["twin_cfg4"] = {
        "s": 16, "m": 5, "rank": 128, "droptol": 1e-2, "seed": 0, "n": int(ps.n), "p": int(ps.p),
        "q": int(ps.q), "achieved_rank": int(lr.rank), "shift": 2.0 + S2,
        "LB_sha": MG.csr_sha(ctx.b_ilu.L), "UB_sha": MG.csr_sha(ctx.b_ilu.U),
        "LC_sha": MG.csr_sha(ctx.c0_ilu.L), "UC_sha": MG.csr_sha(ctx.c0_ilu.U),
        "matrix_sha": MG.csr_sha(ps.matrix), "secs": t1 - t0}
    golden.setdefault("gmres", {})["twin_cfg4"] = {
        "converged": rep.converged, "iterations": rep.iterations, "final_relres": rep.final_relres,
        "history_first_cycles": rep.history[:201], "secs": secs, "restart": 100, "tol": 1e-6, "maxit": 500}
    json.dump(golden, open(path, "w"), indent=1, sort_keys=True)
    print("twin4", rep.converged, rep.iterations, rep.final_relres, secs, flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("twin4", "all"):
        twin4()
    if which in ("setup", "all"):
        setup_sha(sys.argv[2:] if len(sys.argv) > 2 else ["cfg2", "cfg3", "cfg5", "cfg4"])
