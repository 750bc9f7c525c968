#!/usr/bin/env python
"""bench.py — PSLR preconditioner-apply throughput on B200 (BASELINE.json metric:
"PSLR apply GB/s (% HBM roofline) & GMRES time-to-solution at 1/2/4/8 B200").

Workload (config.workload, identical in both arms): BASELINE config 5, the apply sweep —
per GPU a 128^3 block of the 3D 7-point Laplacian (diagonal 6, shift 0.5), 32 subdomains
per GPU, m=3, rank 64, fp64; at N GPUs the global grid is 128 x 128 x 128N with 32N
subdomains (weak scaling).  One step = one PSLR apply (Alg. 3.2, preconditioner.py:79-93)
of one seeded N(0,1) vector (8 pre-generated, cycled; synthetic data).

  value    : algorithmic GB/s of the whole job = N * bytes_apply * steps / max-over-ranks
             device time (SURVEY §8d compulsory bytes: 12 B per stored nonzero per use, V
             twice, b and z once).  The sweep's applies are independent: K calls are in
             flight per GPU (one stream + pslr_ctx_clone context each), each call carries
             two right-hand sides through one launch sequence (pslr_apply_multi), so the
             factors stream once per two vectors — `value` is algorithmic throughput, the
             physical HBM traffic is reported beside it (roofline.sweep).
  e2e      : the same metric through the C-ABI host-buffer call (pinned H2D of b, apply,
             D2H of z inside the timed region, every step), plus e2e.single_call: one
             P.apply(numpy) call, the reference API a user calls.
  roofline : the dominant kernel (the fused Horner-step launch, one vector, single
             stream), the same definition at every N: algorithmic bytes per launch / its
             CUDA-event duration on rank 0; `frac_physical` uses the ncu DRAM bytes of that
             launch (profiles/ncu_summary.json).
  solves   : GMRES / FGMRES time-to-solution on cfg5 and on the BASELINE solver
             configs 2 and 3 (reference outcome beside each).
  cpu_baseline: the oracle port (scipy/numpy restatement of the reference) timed on this
             box's host cores on a bounded sample.

`--impl reference` times the reference's CPU implementation (the oracle port: the Python
reference cannot travel to the GPU box) on the same config and prints the same line; it
never imports this package.  `--gpus N` without a torchrun environment launches N ranks
itself (torch.distributed.run, 127.0.0.1).
"""

import os

_NCPU = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, str(_NCPU))
# the JSON line must be the only stdout output: NCCL's own log lines go to stderr
os.environ.setdefault("NCCL_DEBUG", "WARN")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
# ... and so does anything else a library prints to fd 1: fd 1 is pointed at stderr, the
# JSON line goes to a duplicate of the original stdout
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
PROFILE_PATH = os.path.join(ROOT, "profiles", "ncu_summary.json")
FALLBACK_HBM_GBS = 6650.0
DATASHEET_HBM_GBS = 8000.0
METRIC = "PSLR apply GB/s"
# config 5 per GPU (BASELINE.json configs[4]); defined here so the reference arm needs no
# import of the package under test
CFG5 = {"grid": (128, 128, 128), "shift": 0.5, "s": 32, "m": 3, "rank": 64}
REF_STEP_CAP = 30  # reference arm: at most this many timed applies (~2 s each on CPU)


def workload_string(n_gpus):
    g = n_gpus
    return (f"cfg5 (BASELINE configs[4]) weak-scaled to {g} GPU(s): 3D 7-point Laplacian, diagonal 6, "
            f"shift 0.5, grid 128x128x{128 * g} ({g} x 128^3 per-GPU slabs), s={32 * g} (32 per GPU), "
            f"m=3, rank=64, fp64; one step = one PSLR apply of one seeded N(0,1) vector")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="pslr", choices=["pslr", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="steps of the host-buffer (e2e) leg; 0 = the same as --steps")
    ap.add_argument("--cpu-applies", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=0,
                    help="independent apply calls in flight per GPU (0 = auto)")
    ap.add_argument("--nv", type=int, default=2,
                    help="right-hand sides per apply call (pslr_apply_multi); 1 = pslr_apply")
    ap.add_argument("--gmres-maxit", type=int, default=500,
                    help="maxit of the time-to-solution solves (SURVEY §8d); 0 = skip them")
    ap.add_argument("--solves", default="cfg5,cfg2,cfg3",
                    help="configs whose GMRES/FGMRES time-to-solution is measured (N=1)")
    ap.add_argument("--comm", default="native", choices=["native", "torch"],
                    help="N>1 data plane: native = libpslr's stream-ordered NCCL halo/allreduce "
                         "(pslr_comm_init); torch = torch.distributed process groups from Python")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (multi-GPU) path even at N=1 (testing the NCCL path)")
    args = ap.parse_args()
    if args.e2e_steps <= 0:
        args.e2e_steps = args.steps
    return args


def auto_streams(sm_count, s, calls, cap=16):
    """Independent apply calls in flight: a step launch holds one SM per subdomain and its
    CTAs finish unevenly, so several launches per SM-set keep the SMs busy (cfg5, two
    vectors per call: K = 6 / 8 / 16 -> 0.382 / 0.363 / 0.363 ms per apply, round 1).  At
    most half the timed calls, so the timed region holds at least two waves."""
    return max(1, min(cap, 4 * (sm_count // max(1, s)), calls // 2))


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def profile_summary():
    try:
        with open(PROFILE_PATH) as fh:
            return json.load(fh)
    except Exception:
        return {}


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
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
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


# ------------------------------------------------------------------ CPU arms (oracle)
def oracle_preconditioner(corr_state):
    """The reference's CPU apply (oracle port: scipy spsolve_triangular / csr @ / BLAS) on
    cfg5, setup through the oracle's C restatement of the reference's bisection + ILUT.
    corr_state(q) -> (V, H, G).  Imports only oracle/ (never the package under test)."""
    from oracle import pslr_oracle as O
    t0 = time.perf_counter()
    A = O.laplacian3d(*CFG5["grid"], shift=CFG5["shift"])
    assign = O.partition_c(A, CFG5["s"])
    ps = O.classify_and_reorder(A, assign, CFG5["s"])
    ctx = O.schur_context(ps, droptol=1e-2, use_c=True)
    V, H, G = corr_state(ps.q)
    P = O.Preconditioner(ps, ctx, CFG5["m"], O.Correction(V, H, G, V.shape[1]))
    info = {"nnz_LB": ctx.b_ilu.L.nnz, "nnz_UB": ctx.b_ilu.U.nnz, "nnz_LC": ctx.c0_ilu.L.nnz,
            "nnz_UC": ctx.c0_ilu.U.nnz, "nnz_E": ps.E.nnz, "nnz_F": ps.F.nnz, "nnz_Cg": ctx.Cg.nnz,
            "q": ps.q}
    return P, ps, algorithmic_bytes(info, CFG5["m"], V.shape[1], ps.n), time.perf_counter() - t0


def time_oracle_applies(P, n, steps, warmup):
    rng = np.random.default_rng(0)
    vecs = [rng.standard_normal(n) for _ in range(2)]
    for k in range(warmup):
        P.apply(vecs[k % 2])
    t0 = time.perf_counter()
    for k in range(steps):
        P.apply(vecs[k % 2])
    return (time.perf_counter() - t0) / steps


def _seeded_correction(q, r=64, seed=0):
    """Timing-only correction state for the reference arm (its cost does not depend on
    the values): seeded orthonormal V, small Hessenberg H, G = (I-H)^{-1} - I."""
    from oracle import pslr_oracle as O
    rng = np.random.default_rng(seed)
    V, _ = np.linalg.qr(rng.standard_normal((q, r)))
    H = np.triu(rng.standard_normal((r, r)) * 0.01, -1)
    corr = O.build_correction(V, H)
    return corr.V, corr.H, corr.G


def run_reference(args, world):
    steps = max(1, min(args.steps, REF_STEP_CAP))
    warmup = max(1, min(args.warmup, 1))
    P, ps, bytes_apply, setup_s = oracle_preconditioner(lambda q: _seeded_correction(q, CFG5["rank"]))
    sec = time_oracle_applies(P, ps.n, steps, warmup)
    value = bytes_apply / sec / 1e9  # one 128^3 slab per apply; the job at N GPUs = N slabs
    emit({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_string(world), "n_per_gpu": int(ps.n),
                   "bytes_per_apply_per_gpu": int(bytes_apply)},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": _NCPU, "kind": "port",
                         "sample": f"{steps} applies (of the {args.steps} requested; capped at "
                                   f"{REF_STEP_CAP} ~2 s applies) after {warmup} warm-up, one 128^3 "
                                   "slab, oracle/pslr_oracle.py (the reference's algorithm on scipy "
                                   "spsolve_triangular + csr @ + BLAS; SpTRSV/SpMV single-threaded, "
                                   f"BLAS on {_NCPU} threads); setup via the oracle's C restatement in "
                                   f"{setup_s:.1f} s (untimed); timing-only seeded orthonormal V"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


# ------------------------------------------------------------------ N = 1
def run_single(args):
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib, workloads

    torch.cuda.set_device(0)
    wl = workloads.CONFIGS["cfg5"]
    A = wl.matrix()
    t0 = time.perf_counter()
    P = pg.build(A, wl.config(), device=0)
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
    NV = max(1, min(args.nv, 8))
    calls = -(-args.steps // NV)
    args.steps = calls * NV  # one step = one vector's apply
    K = args.streams if args.streams > 0 else auto_streams(info["sm_count"], P.system.num_parts, calls)
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

    warm = max(3, args.warmup)
    for k in range(warm * K):
        step(k)
    torch.cuda.synchronize()
    # single-stream latency of one apply (what a GMRES iteration sees)
    ns = max(10, min(100, args.steps // 10))
    ms_single = sweep(ns, kk=0) / ns
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    ms = sweep(calls)
    clk = clocks.stop()
    ms_per_step = ms / args.steps
    value = bytes_apply * args.steps / (ms / 1e3) / 1e9

    # per-launch durations (events between launches on the launching stream)
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

    # e2e through the C-ABI host-buffer call (pinned host memory: b H2D, apply, z D2H
    # inside the timed region every step), the same K calls in flight
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
    e2e_value = bytes_apply * args.e2e_steps / (ms_e2e / 1e3) / 1e9
    # the reference API a user calls: P.apply(numpy) (pageable copies, synchronous)
    bnp = rng.standard_normal(n)
    for _ in range(3):
        P.apply(bnp)
    t0 = time.perf_counter()
    nsc = 10
    for _ in range(nsc):
        P.apply(bnp)
    sc_s = (time.perf_counter() - t0) / nsc
    for d in devs[1:]:
        del d
    devs = [dev]

    solves = run_solves(args, P, A, wl, info, bytes_apply) if args.gmres_maxit > 0 else []

    cpu = None
    if not args.no_cpu_baseline:
        V, H, G = P.correction.V, P.correction.H, P.correction.G
        Po, pso, bytes_o, setup_s = oracle_preconditioner(lambda q: (V, H, G))
        sec = time_oracle_applies(Po, pso.n, args.cpu_applies, 1)
        cpu = {"value": bytes_apply / sec / 1e9, "unit": "GB/s", "cores": _NCPU, "kind": "port",
               "ms_per_apply": sec * 1e3,
               "sample": f"{args.cpu_applies} applies after 1 warm-up of the same cfg5 instance, "
                         "oracle/pslr_oracle.py (scipy spsolve_triangular + csr @ + BLAS; SpTRSV/SpMV "
                         f"single-threaded, BLAS on {_NCPU} threads), correction state = this run's V,H,G"}

    peak, peak_src = hbm_peak()
    prof = profile_summary()
    horner_ms = launch_ms.get("horner_step")
    hb = horner_launch_bytes(info)
    achieved = hb / (horner_ms / 1e3) / 1e9 if horner_ms else None
    traffic = prof.get("horner_step_dram_bytes")
    phys = traffic / (horner_ms / 1e3) / 1e9 if (traffic and horner_ms) else None
    call_dram = prof.get("apply2_call_dram_bytes") if NV == 2 else prof.get("apply1_call_dram_bytes")
    sweep_phys = (call_dram * calls / (ms / 1e3) / 1e9) if call_dram else None
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": warm, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_string(1), "n_per_gpu": n, "bytes_per_apply": int(bytes_apply),
                   "parallelism": f"{K} independent apply calls in flight (one stream + clone "
                                  f"context each), {NV} right-hand sides per call",
                   "concurrency": K, "vectors_per_call": NV, "calls": calls,
                   "single_stream": {"ms_per_apply": ms_single,
                                     "value": bytes_apply / (ms_single / 1e3) / 1e9,
                                     "frac": bytes_apply / (ms_single / 1e3) / 1e9 / peak},
                   "l2": "no flush: each apply streams %.2f GB (> 126 MB L2)" % (bytes_apply / 1e9),
                   "build_s": round(build_s, 2)},
        "roofline": {"bound": "hbm", "kernel": "subdomain_step_kernel (Horner step, one vector, single stream)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": traffic,
                     "frac_physical": phys / peak if phys else None,
                     "peak_source": peak_src,
                     "frac_of_datasheet_8TBs": achieved / DATASHEET_HBM_GBS if achieved else None,
                     "bytes_per_launch": int(hb), "launch_ms": launch_ms,
                     "sweep": {"algorithmic_frac": value / peak,
                               "physical_GBps": sweep_phys,
                               "physical_frac": sweep_phys / peak if sweep_phys else None,
                               "note": "value counts 12 B per factor nonzero per vector; a two-vector "
                                       "call streams the factors once (physical = ncu DRAM bytes per "
                                       "call, profiles/ncu_summary.json)"}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": ms_e2e / args.e2e_steps,
                "single_call": {"api": "PslrPreconditioner.apply(numpy)", "ms": sc_s * 1e3,
                                "value": bytes_apply / sc_s / 1e9}},
        # per call: the profiled launch groups (+ the two-vector permute/deinterleave, the
        # correction's second kernel) + one all-SM pre-step kernel per Horner and last step
        # + the split interface phase (an iface kernel per first/correction/Horner step and
        # a second step launch per correction/Horner step)
        "gpu_launches": (launches_per_apply + (0 if NV == 1 else (3 if r > 0 else 1))
                         + ((m + 1) if os.environ.get("PSLR_EY_ALLSM", "1") != "0" else 0)
                         + ((2 + 2 * m + 1) if os.environ.get("PSLR_SPLIT_IFACE", "1") != "0" else 0)) * calls,
        "solves": solves,
        "clocks": clk,
        "levels": {k: info[k] for k in ("maxdepth_LB", "maxdepth_UB", "maxdepth_LC", "maxdepth_UC")},
    }
    emit(line)


REFERENCE_SOLVE = {  # the reference's outcome on the same solve
    "cfg5": None,
    "cfg2": {"converged": False, "iterations": 500, "final_relres": 1.556e-5, "time_s": 232.6,
             "source": "SURVEY.md §6 (reference GMRES(50), 8-core Xeon)"},
    "cfg3": {"converged": False, "iterations": 500, "final_relres": 1.55e-3, "time_s": 2682.0,
             "source": "SURVEY.md §6 (reference GMRES(50) as the FGMRES oracle)"},
}


def run_solves(args, P5, A5, wl5, info5, bytes5):
    """GMRES / FGMRES time-to-solution: b = A x*, x* = default_rng(0), zero
    guess, the device solve with the reference's control flow (krylov.py:35-129)."""
    import torch
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import workloads
    from paper_2002_00917_b200.krylov import gmres_device
    out = []
    for name in [s for s in args.solves.split(",") if s]:
        if name == "cfg5":
            P, A, wl, info, bytes_apply = P5, A5, wl5, info5, bytes5
        else:
            wl = workloads.CONFIGS[name]
            A = wl.matrix()
            P = pg.build(A, wl.config(), device=0)
            info = P.device.info()
            bytes_apply = algorithmic_bytes(info, wl.m, P.correction.rank, P.system.n)
        n = P.system.n
        xs = np.random.default_rng(0).standard_normal(n)
        bg = torch.from_numpy(P.system.matrix @ xs).cuda()
        torch.cuda.synchronize()
        rs = wl.restart if wl.restart > 0 else 50  # cfg5 names no solver: GMRES(50)
        xg, rep = gmres_device(P, bg, tol=wl.tol, maxit=args.gmres_maxit, restart=rs, flexible=wl.flexible)
        torch.cuda.synchronize()
        true_rel = float(torch.linalg.norm(bg - torch.as_tensor(P.system.matrix @ xg.cpu().numpy(),
                                                                device="cuda")) / torch.linalg.norm(bg))
        spmv_b = 12 * info["nnz_A"] + 16 * n
        gb = sum(bytes_apply + spmv_b + 8 * n * ((k % rs) + 1) * 3 + 16 * n for k in range(rep.iterations))
        out.append({"config": name, "solver": "FGMRES" if wl.flexible else "GMRES", "restart": rs,
                    "tol": wl.tol, "maxit": args.gmres_maxit, "n": n, "iterations": rep.iterations,
                    "converged": rep.converged, "final_relres": rep.final_relres, "true_relres": true_rel,
                    "time_s": rep.time_s, "ms_per_iteration": rep.time_s * 1e3 / max(rep.iterations, 1),
                    "GB_per_s": gb / rep.time_s / 1e9 if rep.time_s > 0 else None,
                    "reference": REFERENCE_SOLVE.get(name)})
        if P is not P5:
            del P
    return out


# ------------------------------------------------------------------ N > 1
def run_sharded(args, rank, world, local):
    """N > 1 (or --sharded): config 5 as one coupled problem sharded over the ranks (SURVEY
    §8d.5, §8e): the 128 x 128 x (128 N) grid, s = 32 N subdomains, rank g owns subdomains
    [32 g, 32 (g+1)) (a 128^3 slab).  Per apply: m halo exchanges for C_g and one
    r-double allreduce, everything else rank-local.  --comm native (default): every
    pipeline's context owns an NCCL communicator inside libpslr (pslr_comm_init +
    pslr_ctx_set_halo) and runs pslr_apply_multi with the halos / allreduce stream-ordered
    in the library; --comm torch: shard.py's Python orchestration over torch.distributed."""
    import ctypes
    import torch
    import torch.distributed as dist
    import paper_2002_00917_b200 as pg
    from paper_2002_00917_b200 import _lib, shard, workloads
    from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph
    from paper_2002_00917_b200 import setup_cache as SC

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dist.barrier()
    base = workloads.CONFIGS["cfg5"]
    nx, ny, nz = base.grid
    t0 = time.perf_counter()
    A = workloads.laplacian3d(nx, ny, nz * world, base.shift)
    s_glob = base.s * world
    cfg = pg.PslrConfig(num_subdomains=s_glob, series_degree=base.m, rank=base.rank, droptol=1e-2, seed=0)
    # the global reordering is the same on every rank: rank 0 computes it (or finds it in
    # the content-keyed setup cache) and the others load it
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
    plan, ops = P.plan, P.ops
    info = ops.dev.info()
    m, r = base.m, int(P.correction.rank)
    NV = 2 if args.nv >= 2 else 1
    calls = -(-args.steps // NV)
    args.steps = calls * NV
    K = args.streams if args.streams > 0 else auto_streams(info["sm_count"], base.s, calls, cap=8)
    stream = torch.cuda.current_stream()
    rows = torch.as_tensor(shard.local_rows(plan, ps.p), device="cuda")
    rng = np.random.default_rng(0)
    vecs = []
    for _ in range(8):
        g = torch.as_tensor(rng.standard_normal(ps.n), device="cuda")
        vecs.append(g[rows].contiguous())
    pairs = [torch.stack([vecs[2 * i], vecs[2 * i + 1]]).contiguous() for i in range(4)]
    streams = [stream] + [torch.cuda.Stream() for _ in range(K - 1)]
    outs = [torch.empty((NV, plan.n_loc), dtype=torch.float64, device="cuda") for _ in range(K)]
    if args.comm == "native":
        # K contexts (the built one + clones sharing its factors and correction), each with
        # its own communicator: pipeline j's collectives are issued in the same order on
        # every rank, stream-ordered inside libpslr
        ctxs = [ops.dev] + [ops.dev.clone() for _ in range(K - 1)]
        for c in ctxs:
            obj = [shard.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            shard.attach_nccl_ctx(c, plan, obj[0])
        fm = _lib.fns["pslr_apply_multi"]
        fa = _lib.fns["pslr_apply"]

        def sweep_step(k):
            j = k % K
            src = pairs[k % 4] if NV == 2 else vecs[k % 8]
            f = fm if NV == 2 else None
            if NV == 2:
                _lib.check(f(ctxs[j].handle, m, 2, src.data_ptr(), outs[j].data_ptr(), streams[j].cuda_stream))
            else:
                _lib.check(fa(ctxs[j].handle, m, src.data_ptr(), outs[j].data_ptr(), streams[j].cuda_stream))
    else:
        pipes = [P]
        for _ in range(K - 1):
            grp = dist.new_group(list(range(world)))
            ops_j = ops.clone()
            pipes.append(shard.ShardedPreconditioner(plan, ops_j, shard.Halo(plan, ops_j.device, grp),
                                                     P.series_degree, P.correction))

        def sweep_step(k):
            j = k % K
            with torch.cuda.stream(streams[j]):
                outs[j] = pipes[j].apply2(pairs[k % 4]) if NV == 2 else pipes[j].apply(vecs[k % 8])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    bytes_local = algorithmic_bytes(info, m, r, plan.n_loc)
    tb = torch.tensor([float(bytes_local)], device="cuda", dtype=torch.float64)
    dist.all_reduce(tb)
    bytes_apply = float(tb.item())

    def sweep(ncalls):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in streams[1:]:
            st.wait_stream(stream)
        for k in range(ncalls):
            sweep_step(k)
        for st in streams[1:]:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    warm = max(3, args.warmup)
    sweep(warm * K)
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
    zhs = [torch.empty((NV, plan.n_loc), dtype=torch.float64).pin_memory() for _ in range(K)]
    e2e_calls = -(-args.e2e_steps // NV)
    args.e2e_steps = e2e_calls * NV
    dbufs = [torch.empty((NV, plan.n_loc), dtype=torch.float64, device="cuda") for _ in range(K)]
    saved = (pairs, vecs)

    def e2e_step(k):
        j = k % K
        with torch.cuda.stream(streams[j]):
            dbufs[j].copy_(bhs[j], non_blocking=True)
        if args.comm == "native":
            if NV == 2:
                _lib.check(fm(ctxs[j].handle, m, 2, dbufs[j].data_ptr(), outs[j].data_ptr(), streams[j].cuda_stream))
            else:
                _lib.check(fa(ctxs[j].handle, m, dbufs[j].data_ptr(), outs[j].data_ptr(), streams[j].cuda_stream))
            res = outs[j]
        else:
            with torch.cuda.stream(streams[j]):
                res = pipes[j].apply2(dbufs[j]) if NV == 2 else pipes[j].apply(dbufs[j][0])
        with torch.cuda.stream(streams[j]):
            zhs[j].copy_(res.reshape(zhs[j].shape), non_blocking=True)

    for k in range(2 * K):
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
    del saved
    # the dominant kernel, same definition as N = 1: one Horner-step launch (one vector,
    # single stream) on rank 0's context, CUDA events around it on its stream
    y_ext = ops.zeros(ops.q + ops.ng)
    y_ext[:ops.q] = 1e-3
    c_ext = ops.zeros(ops.q + ops.ng)
    for _ in range(3):
        ops.horner(y_ext, c_ext)
    torch.cuda.synchronize()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record()
    nh = 10
    for _ in range(nh):
        ops.horner(y_ext, c_ext)
    e5.record()
    torch.cuda.synchronize()
    horner_ms = e4.elapsed_time(e5) / nh
    # GMRES time-to-solution of the coupled N-GPU system
    solve = None
    if args.gmres_maxit > 0:
        xs = np.random.default_rng(0).standard_normal(ps.n)
        b_loc = torch.as_tensor((ps.matrix @ xs), device="cuda")[rows].contiguous()
        rs = 50
        torch.cuda.synchronize()
        dist.barrier()
        t0s = time.perf_counter()
        if args.comm == "native":  # the in-library solve: pslr_gmres on the communicator-owning context
            xl = torch.empty_like(b_loc)
            hist = np.zeros(args.gmres_maxit + 1)
            its_, conv_, rel_, hl_ = ctypes.c_int64(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int64()
            _lib.check(_lib.fns["pslr_gmres"](ctxs[0].handle, m, b_loc.data_ptr(), xl.data_ptr(), float(base.tol),
                                              int(args.gmres_maxit), rs, 1, 0, ctypes.byref(its_),
                                              ctypes.byref(conv_), ctypes.byref(rel_), hist.ctypes.data,
                                              ctypes.byref(hl_), stream.cuda_stream))
            conv, its, rel = bool(conv_.value), int(its_.value), float(rel_.value)
        else:
            _, conv, its, rel, _ = shard.sharded_gmres(P, b_loc, tol=base.tol, maxit=args.gmres_maxit, restart=rs)
        torch.cuda.synchronize()
        tsol = torch.tensor([time.perf_counter() - t0s], device="cuda", dtype=torch.float64)
        dist.all_reduce(tsol, op=dist.ReduceOp.MAX)
        ts = float(tsol.item())
        solve = {"config": f"cfg5 x{world}", "solver": "GMRES", "restart": rs, "tol": base.tol,
                 "maxit": args.gmres_maxit, "iterations": its, "converged": conv, "final_relres": rel,
                 "time_s": ts, "ms_per_iteration": ts * 1e3 / max(its, 1),
                 "timing": "wall clock, max over ranks"}
    peak, peak_src = hbm_peak()
    prof = profile_summary()
    hb = horner_launch_bytes(info)
    achieved = hb / (horner_ms / 1e3) / 1e9
    traffic = prof.get("horner_step_dram_bytes")
    nghost = torch.tensor([float(plan.nghost)], device="cuda", dtype=torch.float64)
    dist.all_reduce(nghost, op=dist.ReduceOp.MAX)
    if rank == 0:
        emit({
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_string(world), "n": int(ps.n), "n_per_gpu_rank0": int(plan.n_loc),
                       "bytes_per_apply": int(bytes_apply),
                       "parallelism": f"subdomain sharding x{world} ({args.comm} data plane: {m} halo "
                                      f"exchanges + 1 allreduce({r}) per apply; max ghosts/rank "
                                      f"{int(nghost.item())}); {K} independent apply calls in flight per GPU, "
                                      f"{NV} right-hand sides per call",
                       "concurrency": K, "vectors_per_call": NV, "calls": calls, "comm": args.comm,
                       "l2": "no flush: each apply streams %.2f GB per GPU (> 126 MB L2)" % (bytes_local / 1e9),
                       "build_s": round(build_s, 2)},
            "roofline": {"bound": "hbm", "kernel": "subdomain_step_kernel (Horner step, one vector, single "
                                                   "stream, rank 0)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": peak_src, "bytes_per_launch": int(hb),
                         "launch_ms": {"horner_step": horner_ms},
                         "sweep": {"algorithmic_frac": value / world / peak}},
            "cpu_baseline": None,
            "e2e": {"value": bytes_apply * args.e2e_steps / (ms_e2e / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * int(plan.n_loc), "d2h_bytes_per_step": 8 * int(plan.n_loc),
                    "ms_per_step": ms_e2e / args.e2e_steps},
            "gpu_launches": ((m + 7) * args.steps if NV == 1 else (m + 11) * calls),
            "solves": [solve] if solve else [],
            "clocks": clk,
        })
    dist.destroy_process_group()


def spawn(args):
    """--gpus N without a torchrun environment: launch N ranks on this node."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    proc = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=None, text=True)
    for line in proc.stdout.splitlines():
        if line.startswith("{"):
            _JSON_OUT.write(line + "\n")
    _JSON_OUT.flush()
    return proc.returncode


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         "(torch.distributed.run --nproc-per-node N), or omit WORLD_SIZE and let "
                         "bench.py spawn them")
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, world)
        return
    if world > 1 or args.sharded:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        return run_sharded(args, rank, world, local)
    return run_single(args)


if __name__ == "__main__":
    main()
