"""Parameter sweeps on the device path (cli.py:186-266, `pslr sweep`).

One CSV row per axis value, the reference's columns (cli.py:196-197).  As in the
reference driver, the m and rank sweeps reuse ONE partition and ONE set of ILU factors
— here also one device context, so the factors are packed and uploaded once — and the
rank sweep reuses ONE device Arnoldi run at the largest rank, truncated per row
(V[:, :r], H[:r, :r]; the Arnoldi basis of a smaller rank is exactly that prefix).  The s
sweep rebuilds per value.  Each row solves b = A x*, x* = default_rng(seed) (cli.py:126-128)
on the reordered system with the device GMRES or CG (cli.py:131-143).
"""

from __future__ import annotations

import time

import numpy as np

from .krylov import cg_device, gmres_device
from .lowrank import arnoldi_device, build_correction
from .partition import classify_and_reorder, partition_graph
from .preconditioner import PslrConfig, PslrPreconditioner, _fill_stats, build
from .schur import build_schur_context
from .sparse import canonical

SWEEP_COLUMNS = ["axis", "value", "its", "converged", "fill_ilu", "fill_lowrank",
                 "fill_total", "final_relres", "p_t", "i_t", "t_t"]


def _solve(A, P, seed, krylov, tol, maxit, restart):
    """cli._solve_with (cli.py:131-143) with the device accelerators."""
    b = A @ np.random.default_rng(seed).standard_normal(A.shape[0])
    bp = b[P.system.perm.inverse]
    if krylov == "cg":
        zp, rep = cg_device(P, bp, tol=tol, maxit=maxit)
    else:
        zp, rep = gmres_device(P, bp, tol=tol, maxit=maxit, restart=restart)
    return zp[P.system.perm.forward], rep


def _bind(ctx, system, m, Vd, H, A, order_t, build_t):
    corr = build_correction(Vd.cpu().numpy(), H)
    ctx.device.set_correction(Vd if corr.rank else None, corr.G if corr.rank else None)
    ctx.device._bound = corr
    corr.device = ctx.device
    stats = _fill_stats(A, ctx, corr, order_time=order_t, build_time=build_t)
    return PslrPreconditioner(system=system, ctx=ctx, series_degree=m, correction=corr, stats=stats)


def sweep(A, axis: str, values, s: int = 8, m: int = 3, rank: int = 15, droptol: float = 1e-2,
          seed: int = 0, krylov: str = "gmres", tol: float = 1e-8, maxit: int = 500,
          restart: int = 0, device=None):
    """cmd_sweep (cli.py:200-266).  Returns (rows, csv_text); each row is a dict with the
    SWEEP_COLUMNS keys plus the report."""
    if axis not in ("s", "m", "rank"):
        raise ValueError("sweep axis must be one of s, m, rank")
    values = [int(v) for v in values]
    if not values:
        raise ValueError("sweep needs at least one axis value")
    A = canonical(A)
    rows = []
    if axis == "s":
        for sv in values:
            P = build(A, PslrConfig(num_subdomains=sv, series_degree=m, rank=rank, droptol=droptol,
                                    seed=seed), device=device)
            _, rep = _solve(A, P, seed, krylov, tol, maxit, restart)
            rows.append((sv, P, rep))
    else:
        t0 = time.perf_counter()
        system = classify_and_reorder(A, partition_graph(A, s, seed=seed))
        t1 = time.perf_counter()
        ctx = build_schur_context(system, droptol=droptol, device=device)
        order_t, ilu_t = t1 - t0, time.perf_counter() - t1
        if axis == "m":
            for mv in values:
                t0 = time.perf_counter()
                Vd, H, _ = arnoldi_device(ctx, mv, min(rank, system.q), seed=seed)
                P = _bind(ctx, system, mv, Vd, H, A, order_t, ilu_t + time.perf_counter() - t0)
                _, rep = _solve(A, P, seed, krylov, tol, maxit, restart)
                rows.append((mv, P, rep))
        else:
            t0 = time.perf_counter()
            Vd, H, r = arnoldi_device(ctx, m, min(max(values), system.q), seed=seed)
            arnoldi_t = time.perf_counter() - t0
            for rv in values:
                rr = min(rv, r)
                t0 = time.perf_counter()
                P = _bind(ctx, system, m, Vd[:, :rr].contiguous(), np.ascontiguousarray(H[:rr, :rr]), A,
                          order_t, ilu_t + arnoldi_t + time.perf_counter() - t0)
                _, rep = _solve(A, P, seed, krylov, tol, maxit, restart)
                rows.append((rv, P, rep))
    out = []
    lines = [",".join(SWEEP_COLUMNS)]
    for value, P, rep in rows:
        st = P.stats
        row = {"axis": axis, "value": value, "its": rep.iterations, "converged": rep.converged,
               "fill_ilu": st.fill_ilu, "fill_lowrank": st.fill_lowrank, "fill_total": st.fill_total,
               "final_relres": rep.final_relres, "p_t": st.build_time_s, "i_t": rep.time_s,
               "t_t": st.build_time_s + rep.time_s, "report": rep}
        out.append(row)
        lines.append(",".join(str(x) for x in [
            axis, value, rep.iterations, rep.converged, f"{st.fill_ilu:.6f}", f"{st.fill_lowrank:.6f}",
            f"{st.fill_total:.6f}", f"{rep.final_relres:.6e}", f"{st.build_time_s:.6f}",
            f"{rep.time_s:.6f}", f"{st.build_time_s + rep.time_s:.6f}"]))
    return out, "\n".join(lines) + "\n"
