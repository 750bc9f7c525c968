#!/usr/bin/env python
"""bench.py — PSLR preconditioner-apply throughput on B200 (BASELINE.json metric).

Workload (N=1): BASELINE config 5, the preconditioner-apply sweep — a 128^3 block of the
3D 7-point Laplacian (diagonal 6, shift 0.5), 32 subdomains, m=3, rank 64, fp64, applied
to seeded N(0,1) vectors (8 pre-generated, cycled).  One step = one PSLR apply
(Alg. 3.2, preconditioner.py:79-93) of one vector.  The sweep's applies are independent
and a step launch occupies one SM per subdomain (32 of 148), so K = 8 applies are in
flight (one stream and pslr_ctx_clone context each; every apply is bit-identical to the
single-stream one); the single-stream latency (what one GMRES iteration sees) is
reported beside it in config.single_stream.  Under torchrun each rank applies its
own 128^3 slab of ONE coupled global problem (grid 128 x 128 x 128N, s = 32N; subdomain
sharding with NCCL halo exchanges, weak scaling; see run_sharded and DESIGN.md §Multi-GPU).

  value   : algorithmic GB/s over all ranks = N * bytes_apply * K / max-over-ranks time
  e2e     : same metric through the C-ABI host-buffer call (pslr_apply_host: pinned H2D
            copy of b, apply, D2H copy of z inside the timed region)
  roofline: the dominant kernel (the fused Horner-step launch) vs the measured HBM copy peak
  cpu_baseline: the oracle port (scipy/numpy restatement) timed on this box's host cores

`--impl reference` times the reference CPU path (the oracle port, since the Python
reference cannot travel to the GPU box) on the same config and prints the same line.
"""

import os

_NCPU = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, str(_NCPU))
# the JSON line must be the only stdout output: NCCL's own log lines go to stderr
os.environ.setdefault("NCCL_DEBUG", "WARN")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
# ... and so does anything else a library prints to fd 1 (NCCL's version banner ignores
# NCCL_DEBUG_FILE on some builds): fd 1 is pointed at stderr, the JSON line goes to a
# duplicate of the original stdout
_JSON_FD = os.dup(1)
os.dup2(2, 1)
_JSON_OUT = os.fdopen(_JSON_FD, "w")


def emit(line):
    _JSON_OUT.write(__import__("json").dumps(line) + "\n")
    _JSON_OUT.flush()

import argparse  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
DATASHEET_HBM_GBS = 8000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="pslr", choices=["pslr", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="steps of the host-buffer (e2e) leg; 0 = the same as --steps")
    ap.add_argument("--cpu-applies", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=0,
                    help="independent apply calls in flight per GPU (0 = auto: 4 * (SMs // subdomains), "
                         "<= 16; <= 8 on the sharded path)")
    ap.add_argument("--nv", type=int, default=2,
                    help="right-hand sides per apply call in the N=1 sweep (pslr_apply_multi: the "
                         "vectors share one launch sequence); 1 = pslr_apply")
    ap.add_argument("--gmres-maxit", type=int, default=500,
                    help="N=1: also time one device GMRES solve (SURVEY §8d time-to-solution); 0 = skip")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (multi-GPU) path even at N=1 (testing the NCCL path)")
    args = ap.parse_args()
    if args.e2e_steps <= 0:
        args.e2e_steps = args.steps
    return args


def auto_streams(sm_count, s, cap=16):
    """Independent applies in flight: a step launch holds one SM per subdomain and its
    CTAs finish unevenly, so several launches per SM-set keep the SMs busy (measured on
    cfg5, two vectors per call: K = 6 / 7 / 8 / 9-12 / 16 / 24 -> 0.382 / 0.367 / 0.363 /
    0.41-0.49 / 0.363 / 0.364 ms per apply; K = 16 also hides the host copies of the e2e
    leg best: 4.27 vs 4.03 TB/s at K = 8).  The sharded path caps it at 8: every pipeline
    there owns an NCCL communicator."""
    return max(1, min(cap, 4 * (sm_count // max(1, s))))


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def workload(name, world):
    from paper_2002_00917_b200 import workloads
    return workloads.CONFIGS[name]


def algorithmic_bytes(info, m, r, n):
    """compulsory bytes of one apply (12 B per stored nonzero per use, V twice,
    b read + z written)."""
    nz = lambda k: info["nnz_" + k]  # noqa: E731
    mat = ((m + 2) * (nz("LB") + nz("UB")) + (m + 1) * (nz("LC") + nz("UC"))
           + (m + 1) * (nz("E") + nz("F")) + m * nz("Cg"))
    return 12 * mat + 16 * info["q"] * r + 16 * n


def horner_launch_bytes(info):
    """Algorithmic bytes of one fused Horner-step launch: E, B^{-1} (L,U), F, Cg, C0^{-1} (L,U)
    once each, y and c read, y written."""
    nz = lambda k: info["nnz_" + k]  # noqa: E731
    return 12 * (nz("LB") + nz("UB") + nz("LC") + nz("UC") + nz("E") + nz("F") + nz("Cg")) \
        + 24 * info["q"]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/pslr_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def oracle_apply_seconds(A, wl, corr_state, n_applies):
    """The reference's CPU apply (oracle port: scipy spsolve_triangular / csr @ / BLAS) on
    this box's host cores.  Setup via the oracle's C restatement of ILUT + bisection."""
    from oracle import pslr_oracle as O
    t0 = time.perf_counter()
    assign = O.partition_c(A, wl.s)
    ps = O.classify_and_reorder(A, assign, wl.s)
    ctx = O.schur_context(ps, droptol=1e-2, use_c=True)
    setup_s = time.perf_counter() - t0
    V, H, G = corr_state(ps.q)
    P = O.Preconditioner(ps, ctx, wl.m, O.Correction(V, H, G, V.shape[1]))
    rng = np.random.default_rng(0)
    vecs = [rng.standard_normal(ps.n) for _ in range(2)]
    P.apply(vecs[0])  # warm-up
    times = []
    for k in range(n_applies):
        t = time.perf_counter()
        P.apply(vecs[k % 2])
        times.append(time.perf_counter() - t)
    return float(np.median(times)), setup_s, ps, ctx


def _seeded_correction(q, r=64, seed=0):
    """Timing-only correction state for the reference arm (its cost does not depend on
    the values): seeded orthonormal V, small Hessenberg H, G = (I-H)^{-1} - I."""
    from oracle import pslr_oracle as O
    rng = np.random.default_rng(seed)
    V, _ = np.linalg.qr(rng.standard_normal((q, r)))
    H = np.triu(rng.standard_normal((r, r)) * 0.01, -1)
    corr = O.build_correction(V, H)
    return corr.V, corr.H, corr.G


def oracle_bytes(ctx, ps, m, r):
    info = {"nnz_LB": ctx.b_ilu.L.nnz, "nnz_UB": ctx.b_ilu.U.nnz, "nnz_LC": ctx.c0_ilu.L.nnz,
            "nnz_UC": ctx.c0_ilu.U.nnz, "nnz_E": ps.E.nnz, "nnz_F": ps.F.nnz, "nnz_Cg": ctx.Cg.nnz,
            "q": ps.q}
    return algorithmic_bytes(info, m, r, ps.n)


def run_reference(args):
    wl = workload(args.config, 1)
    A = wl.matrix()
    n_app = max(1, min(args.steps, args.cpu_applies))
    sec, setup_s, ps, ctx = oracle_apply_seconds(A, wl, lambda q: _seeded_correction(q, wl.rank), n_app)
    bytes_apply = oracle_bytes(ctx, ps, wl.m, wl.rank)
    value = bytes_apply / sec / 1e9
    line = {
        "impl": "reference", "metric": "PSLR apply GB/s", "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": n_app, "warmup": 1, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{wl.name}: 3D 7-point Laplacian 128^3 shift 0.5, s={wl.s}, "
                               f"m={wl.m}, rank={wl.rank}", "n": int(A.shape[0]),
                   "bytes_per_apply": int(bytes_apply)},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": _NCPU, "kind": "port",
                         "sample": f"{n_app} applies (median) of the {args.steps} requested, after 1 "
                                   "warm-up; oracle/pslr_oracle.py (scipy spsolve_triangular + csr @ "
                                   "+ BLAS, SpTRSV/SpMV single-threaded); setup via oracle C "
                                   f"restatement in {setup_s:.1f}s (untimed); timing-only seeded "
                                   "orthonormal V"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def run_sharded(args, rank, world, local):
    """N > 1: config 5 as one coupled problem sharded over the ranks:
    the 128 x 128 x (128 N) grid, s = 32 N subdomains, rank g owns subdomains
    [32 g, 32 (g+1)) (a 128^3 slab).  Per apply: m halo exchanges for C_g and one
    r-double allreduce (NCCL), everything else rank-local.  Weak scaling: per-GPU work is
    one 128^3 slab at every N."""
    import torch
    import torch.distributed as dist
    from paper_2002_00917_b200 import shard, workloads
    from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dist.barrier()
    base = workloads.CONFIGS[args.config]
    nx, ny, nz = base.grid
    t0 = time.perf_counter()
    A = workloads.laplacian3d(nx, ny, nz * world, base.shift)
    s_glob = base.s * world
    cfg = __import__("paper_2002_00917_b200").PslrConfig(num_subdomains=s_glob, series_degree=base.m,
                                                         rank=base.rank, droptol=1e-2, seed=0)
    # the global reordering is the same on every rank: rank 0 computes it (or finds it in
    # the setup cache) and the others load it (setup_cache.py; content-keyed, so a stale
    # file can never be picked up)
    from paper_2002_00917_b200 import setup_cache as SC
    order_path = os.path.join(SC.cache_dir() or "/tmp/pslr_setup_cache",
                              f"order_{SC.setup_key(SC.matrix_digest(A), cfg)}.npz")
    hit = SC.load_setup(order_path, A, need_factors=False) if rank == 0 else None
    if rank == 0 and hit is None:
        ps = classify_and_reorder(A, partition_graph(A, s_glob, seed=0))
        SC.save_setup(order_path, ps)
    elif rank == 0:
        ps = hit[0]
    dist.barrier()
    if rank != 0:
        ps = SC.load_setup(order_path, A, need_factors=False)[0]
    P = shard.build_sharded(ps, cfg, device=local)
    # K independent sharded applies in flight (as at N=1): pipeline j has its own clone
    # context, stream and process group (its NCCL communicator), so every group sees its
    # collectives in the same order on all ranks
    K = args.streams if args.streams > 0 else auto_streams(P.ops.dev.info()["sm_count"], base.s, cap=8)
    pipes, streams = [P], [torch.cuda.current_stream()]
    for _ in range(K - 1):
        g = dist.new_group(list(range(world)))
        ops_j = P.ops.clone()
        pipes.append(shard.ShardedPreconditioner(P.plan, ops_j, shard.Halo(P.plan, ops_j.device, g),
                                                 P.series_degree, P.correction))
        streams.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    plan, ops = P.plan, P.ops
    info = ops.dev.info()
    m, r = base.m, int(P.correction.rank)
    bytes_local = algorithmic_bytes(info, m, r, plan.n_loc)
    tb = torch.tensor([float(bytes_local)], device="cuda", dtype=torch.float64)
    dist.all_reduce(tb)
    bytes_apply = float(tb.item())
    rows = torch.as_tensor(shard.local_rows(plan, ps.p), device="cuda")
    rng = np.random.default_rng(0)
    vecs = []
    for _ in range(8):
        g = torch.as_tensor(rng.standard_normal(ps.n), device="cuda")
        vecs.append(g[rows].contiguous())
    stream = torch.cuda.current_stream()
    # NV right-hand sides per pipeline call (ShardedPreconditioner.apply2: one launch
    # sequence, one halo per Horner step and one allreduce for both vectors)
    NV = 2 if args.nv >= 2 else 1
    pairs = [torch.stack([vecs[2 * i], vecs[2 * i + 1]]).contiguous() for i in range(4)]
    calls = -(-args.steps // NV)
    args.steps = calls * NV

    def sweep_step(k, fn=None):
        j = k % K
        with torch.cuda.stream(streams[j]):
            if NV == 2:
                out = pipes[j].apply2(pairs[k % 4] if fn is None else fn(j))
            else:
                out = pipes[j].apply(vecs[k % 8] if fn is None else fn(j))
        return out

    def sweep(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in streams[1:]:
            st.wait_stream(stream)
        for k in range(steps):
            sweep_step(k)
        for st in streams[1:]:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for k in range(max(3, args.warmup) * K):
        sweep_step(k)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    ms = sweep(calls)
    dist.barrier()
    clk = clocks.stop()
    tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    value = bytes_apply * args.steps / (ms / 1e3) / 1e9
    # e2e: host (pinned) b -> device, sharded apply, z -> host, every step
    bhs = [(pairs[j % 4] if NV == 2 else vecs[j % 8]).cpu().pin_memory() for j in range(K)]
    zhs = [torch.empty_like(bhs[0]).pin_memory() for _ in range(K)]
    e2e_calls = -(-args.e2e_steps // NV)
    args.e2e_steps = e2e_calls * NV

    def e2e_step(k):
        j = k % K
        with torch.cuda.stream(streams[j]):
            bd = bhs[j].to("cuda", non_blocking=True)
            zhs[j].copy_(pipes[j].apply2(bd) if NV == 2 else pipes[j].apply(bd), non_blocking=True)

    for k in range(3 * K):
        e2e_step(k)
    dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for st in streams[1:]:
        st.wait_stream(stream)
    for k in range(e2e_calls):
        e2e_step(k)
    for st in streams[1:]:
        stream.wait_stream(st)
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3)
    tt = torch.tensor([ms_e2e], device="cuda", dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_e2e = float(tt.item())
    # GMRES time-to-solution of the coupled N-GPU system: b = A x*, x*
    # seeded; shard.sharded_gmres (one sharded apply + halo'd A-SpMV + three allreduced CGS2
    # passes per iteration), wall time max over ranks
    solve = None
    if args.gmres_maxit > 0:
        xs = np.random.default_rng(0).standard_normal(ps.n)
        b_loc = torch.as_tensor((ps.matrix @ xs), device="cuda")[rows].contiguous()
        rs = base.restart if base.restart > 0 else 50
        torch.cuda.synchronize()
        dist.barrier()
        t0s = time.perf_counter()
        _, conv, its, rel, _ = shard.sharded_gmres(P, b_loc, tol=base.tol, maxit=args.gmres_maxit,
                                                   restart=rs)
        torch.cuda.synchronize()
        tsol = torch.tensor([time.perf_counter() - t0s], device="cuda", dtype=torch.float64)
        dist.all_reduce(tsol, op=dist.ReduceOp.MAX)
        ts = float(tsol.item())
        solve = {"solver": "GMRES", "restart": rs, "tol": base.tol, "maxit": args.gmres_maxit,
                 "iterations": its, "converged": conv, "final_relres": rel, "time_s": ts,
                 "ms_per_iteration": ts * 1e3 / max(its, 1), "timing": "wall clock, max over ranks"}
    peak, peak_src = hbm_peak()
    per_gpu = bytes_local / (ms / args.steps / 1e3) / 1e9
    nghost = torch.tensor([float(plan.nghost)], device="cuda", dtype=torch.float64)
    dist.all_reduce(nghost, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {
            "metric": "PSLR apply GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{base.name} sharded: 3D 7-point Laplacian {nx}x{ny}x{nz * world} "
                                   f"shift {base.shift}, s={s_glob} ({base.s} per GPU), m={m}, rank={r}; "
                                   "one step = one PSLR apply of the global system",
                       "n": int(ps.n), "n_per_gpu_rank0": int(plan.n_loc),
                       "bytes_per_apply": int(bytes_apply),
                       "parallelism": f"subdomain sharding x{world} (NCCL: {m} halo exchanges + 1 "
                                      f"allreduce({r}) per apply; max ghosts/rank {int(nghost.item())}); "
                                      f"{K} independent apply calls in flight per GPU (stream + clone + NCCL group "
                                      f"each), {NV} right-hand sides per call",
                       "concurrency": K, "vectors_per_call": NV,
                       "l2": "no flush: each apply streams %.2f GB per GPU (> 126 MB L2)" % (bytes_local / 1e9),
                       "build_s": round(build_s, 2)},
            "roofline": {"bound": "hbm", "kernel": "whole sharded apply on rank 0 (all launches + halo)",
                         "achieved": per_gpu, "peak": peak, "unit": "GB/s", "frac": per_gpu / peak,
                         "traffic": None, "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": {"value": bytes_apply * args.e2e_steps / (ms_e2e / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * int(plan.n_loc), "d2h_bytes_per_step": 8 * int(plan.n_loc),
                    "ms_per_step": ms_e2e / args.e2e_steps},
            "gpu_launches": ((m + 7) * args.steps if NV == 1 else (m + 11) * calls),
            "solve": solve,
            "clocks": clk,
        }
        emit(line)
    dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    if world > 1 or args.sharded:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        return run_sharded(args, rank, world, local)
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = workload(args.config, world)
    A = wl.matrix()
    t0 = time.perf_counter()
    P = pg.build(A, wl.config(), device=local)
    build_s = time.perf_counter() - t0
    dev = P.device
    info = dev.info()
    n, m, r = P.system.n, wl.m, P.correction.rank
    bytes_apply = algorithmic_bytes(info, m, r, n)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    rng = np.random.default_rng(0)
    vecs = [torch.from_numpy(rng.standard_normal(n)).cuda() for _ in range(8)]
    vmat = torch.stack(vecs).contiguous()
    outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    fn = _lib.fns["pslr_apply"]
    fm = _lib.fns["pslr_apply_multi"]
    h = dev.handle
    # The sweep's applies are independent and one step launch occupies only s of the
    # SMs: K apply calls run concurrently, each on its own stream with its own clone
    # context (shared factors / correction, private scratch; pslr_ctx_clone), and each
    # call carries NV right-hand sides through one launch sequence (pslr_apply_multi: the
    # factors stream once for both vectors).  Every vector's result is the single-vector
    # apply bit for bit (tests/test_gpu_parity.py::test_clones_...,
    # ::test_apply_multi_bitexact).
    K = args.streams if args.streams > 0 else auto_streams(info["sm_count"], P.system.num_parts)
    NV = max(1, min(args.nv, 8))
    calls = -(-args.steps // NV)
    args.steps = calls * NV  # one step = one vector's apply
    devs = [dev] + [dev.clone() for _ in range(K - 1)]
    streams = [stream] + [torch.cuda.Stream() for _ in range(K - 1)]
    souts = [[torch.empty((NV, n), dtype=torch.float64, device="cuda") for _ in range(2)] for _ in range(K)]

    def step(k, kk=None):
        j = k % K if kk is None else kk
        if NV == 1 or kk is not None:
            _lib.check(fn(devs[j].handle, m, vecs[k % 8].data_ptr(), souts[j][(k // K) % 2].data_ptr(),
                          streams[j].cuda_stream))
        else:
            v0 = (k * NV) % (8 - NV + 1)
            _lib.check(fm(devs[j].handle, m, NV, vmat[v0].data_ptr(), souts[j][(k // K) % 2].data_ptr(),
                          streams[j].cuda_stream))

    def sweep(steps, kk=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in streams[1:]:
            st.wait_stream(stream)
        for k in range(steps):
            step(k, kk)
        for st in streams[1:]:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for k in range(max(3, args.warmup) * K):
        step(k)
    torch.cuda.synchronize()
    # single-stream latency of one apply (what a GMRES iteration sees), for the record
    ms_single = sweep(max(10, args.steps // 10), kk=0) / max(10, args.steps // 10)
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES") else local
    clocks = ClockSampler(gpu_index)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms = sweep(calls)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    if dist:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    value = world * bytes_apply * args.steps / (ms / 1e3) / 1e9

    # per-launch durations (events between launches; measurement pass, not the timed one)
    cap = 64
    lms = np.zeros(cap)
    lkind = np.zeros(cap, dtype=np.int32)
    nl = __import__("ctypes").c_int64()
    per_kind = {}
    for k in range(5):
        _lib.check(_lib.fns["pslr_apply_profiled"](h, m, vecs[k % 8].data_ptr(), outs[0].data_ptr(),
                                                   sptr, lms.ctypes.data, lkind.ctypes.data, cap,
                                                   __import__("ctypes").byref(nl)))
        for i in range(min(nl.value, cap)):
            per_kind.setdefault(int(lkind[i]), []).append(float(lms[i]))
    launches_per_apply = int(nl.value)
    kind_names = {1: "correction_core", 2: "first_step", 3: "correction_c0", 4: "horner_step",
                  5: "last_step", 6: "permute_f", 0: "step"}
    launch_ms = {kind_names.get(k, str(k)): float(np.mean(v)) for k, v in per_kind.items()}
    horner_ms = launch_ms.get("horner_step")
    peak, peak_src = hbm_peak()
    hb = horner_launch_bytes(info)
    achieved = hb / (horner_ms / 1e3) / 1e9 if horner_ms else None
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof_json):
        try:
            traffic = json.load(open(prof_json)).get("horner_step_dram_bytes")
        except Exception:
            traffic = None

    # e2e through the C-ABI host-buffer call (pinned host memory: b H2D, apply, z D2H
    # inside the timed region every step), the same K applies in flight
    bhs = [torch.from_numpy(rng.standard_normal((NV, n))).pin_memory() for _ in range(K)]
    zhs = [torch.empty((NV, n), dtype=torch.float64).pin_memory() for _ in range(K)]
    fh = _lib.fns["pslr_apply_multi_host_async"]
    e2e_calls = -(-args.e2e_steps // NV)
    args.e2e_steps = e2e_calls * NV

    def e2e_step(k):
        j = k % K
        _lib.check(fh(devs[j].handle, m, NV, bhs[j].data_ptr(), zhs[j].data_ptr(), streams[j].cuda_stream))

    for k in range(3 * K):
        e2e_step(k)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for st in streams[1:]:
        st.wait_stream(stream)
    for k in range(e2e_calls):
        e2e_step(k)
    for st in streams[1:]:
        stream.wait_stream(st)
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3)
    if dist:
        tt = torch.tensor([ms_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_e2e = float(tt.item())
    e2e_value = world * bytes_apply * args.e2e_steps / (ms_e2e / 1e3) / 1e9

    # GMRES time-to-solution: b = A x*, x* seeded; the device solve with the
    # reference's control flow (krylov.py:35-129); algorithmic bytes per iteration j of a
    # cycle = apply + A-SpMV + CGS2 (3 passes over j+1 basis vectors: the projections fuse
    # with the following dot / norm) + 16 n
    solve = None
    if args.gmres_maxit > 0:
        from paper_2002_00917_b200.krylov import gmres_device
        xs = np.random.default_rng(0).standard_normal(n)
        bg = torch.from_numpy(P.system.matrix @ xs).cuda()
        torch.cuda.synchronize()
        rs = wl.restart if wl.restart > 0 else 50  # cfg5 names no solver: GMRES(50)
        xg, rep = gmres_device(P, bg, tol=wl.tol, maxit=args.gmres_maxit, restart=rs,
                               flexible=wl.flexible)
        torch.cuda.synchronize()
        spmv_b = 12 * info["nnz_A"] + 16 * n
        gb = sum(bytes_apply + spmv_b + 8 * n * ((k % rs) + 1) * 3 + 16 * n for k in range(rep.iterations))
        solve = {"solver": "FGMRES" if wl.flexible else "GMRES", "restart": rs, "tol": wl.tol,
                 "maxit": args.gmres_maxit, "iterations": rep.iterations, "converged": rep.converged,
                 "final_relres": rep.final_relres, "time_s": rep.time_s,
                 "ms_per_iteration": rep.time_s * 1e3 / max(rep.iterations, 1),
                 "GB_per_s": gb / rep.time_s / 1e9 if rep.time_s > 0 else None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        V, H, G = P.correction.V, P.correction.H, P.correction.G
        sec, setup_s, ps_o, ctx_o = oracle_apply_seconds(A, wl, lambda q: (V, H, G), args.cpu_applies)
        cpu = {"value": bytes_apply / sec / 1e9, "unit": "GB/s", "cores": _NCPU, "kind": "port",
               "ms_per_apply": sec * 1e3,
               "sample": f"{args.cpu_applies} applies (median) after 1 warm-up of the same cfg5 "
                         "instance, oracle/pslr_oracle.py (scipy spsolve_triangular + csr @ + BLAS; "
                         "SpTRSV/SpMV single-threaded), correction state = this run's V,H,G"}
    if rank == 0:
        line = {
            "metric": "PSLR apply GB/s", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{wl.name}: 3D 7-point Laplacian 128^3 per GPU, shift 0.5, "
                                   f"s={wl.s}, m={m}, rank={r}; one step = one PSLR apply",
                       "n_per_gpu": n, "bytes_per_apply": int(bytes_apply),
                       "parallelism": f"{K} independent apply calls in flight (one stream + clone "
                                      f"context each), {NV} right-hand sides per call",
                       "concurrency": K, "vectors_per_call": NV,
                       "single_stream": {"ms_per_apply": ms_single,
                                         "value": bytes_apply / (ms_single / 1e3) / 1e9},
                       "l2": "no flush: each apply streams %.2f GB (> 126 MB L2)" % (bytes_apply / 1e9),
                       "build_s": round(build_s, 2)},
            "roofline": {"bound": "hbm", "kernel": "subdomain_step_kernel (Horner step)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "peak_source": peak_src,
                         "frac_of_datasheet_8TBs": achieved / DATASHEET_HBM_GBS if achieved else None,
                         "bytes_per_launch": int(hb), "launch_ms": launch_ms,
                         "apply_frac": (bytes_apply / (ms_per_step / 1e3) / 1e9) / peak,
                         "apply_frac_single_stream": (bytes_apply / (ms_single / 1e3) / 1e9) / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * n, "ms_per_step": ms_e2e / args.e2e_steps},
            "gpu_launches": (launches_per_apply + (0 if NV == 1 else (3 if r > 0 else 1))) * calls,
            "solve": solve,
            "clocks": clk,
            "levels": {k: info[k] for k in ("maxdepth_LB", "maxdepth_UB", "maxdepth_LC", "maxdepth_UC")},
        }
        emit(line)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
