"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container only (it imports the read-only reference package
from /root/reference/pkg/src; that tree does not exist on the GPU box):

    python tests/golden/make_golden.py            # all cases
    python tests/golden/make_golden.py small      # just the small cases

Every fixture is produced by calling the reference's own public API
(pslr.partition / pslr.ilu / pslr.schur / pslr.lowrank / pslr.preconditioner /
pslr.krylov) on seeded synthetic inputs.  The committed .npz / .json files are
what the oracle (oracle/pslr_oracle.py) and the product's host setup are pinned
against in tests/test_oracle_golden.py and tests/test_setup_bitexact.py.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from pslr.ilu import block_solve, factor_blocks, ilut  # noqa: E402
from pslr.krylov import gmres  # noqa: E402
from pslr.lowrank import apply_correction, arnoldi, build_correction  # noqa: E402
from pslr.partition import classify_and_reorder, partition_graph  # noqa: E402
from pslr.preconditioner import PslrConfig, build  # noqa: E402
from pslr.problems import ProblemSpec, laplacian3d  # noqa: E402
from pslr.schur import (apply_Err, apply_Es, apply_neumann, build_schur_context,  # noqa: E402
                        solve_B, solve_C0)

HERE = os.path.dirname(os.path.abspath(__file__))


def lap1d(n):
    return sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")


def random_sparse(n, density=0.1, seed=0, diag_boost=4.0):
    # same construction as the reference test helper (pkg/tests/conftest.py:25-29)
    A = sp.random(n, n, density=density, random_state=seed, format="csr",
                  data_rvs=np.random.default_rng(seed).standard_normal)
    return (A + diag_boost * sp.identity(n)).tocsr()


def upwind3d(nx, ny, nz, shift, hv):
    """Our cfg3 generator (absent from the reference):
    h^2-scaled 7-point diffusion + first-order upwind convection, velocity (1,1,1).
    Per axis: +hv on the diagonal, -hv on the upstream (i-1) neighbour."""
    def axis(n):
        return sp.diags([np.full(n - 1, -1.0 - hv), np.full(n, 2.0 + hv), np.full(n - 1, -1.0)],
                        [-1, 0, 1], format="csr")
    Ix, Iy, Iz = (sp.identity(k, format="csr") for k in (nx, ny, nz))
    A = sp.kron(Iz, sp.kron(Iy, axis(nx))) + sp.kron(Iz, sp.kron(axis(ny), Ix)) \
        + sp.kron(axis(nz), sp.kron(Iy, Ix))
    A = A - shift * sp.identity(nx * ny * nz)
    A = sp.csr_matrix(A, dtype=np.float64)
    A.sum_duplicates()
    A.sort_indices()
    return A


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def csr_parts(prefix, M, out):
    M = sp.csr_matrix(M)
    out[prefix + "_indptr"] = M.indptr.astype(np.int64)
    out[prefix + "_indices"] = M.indices.astype(np.int32)
    out[prefix + "_data"] = M.data.astype(np.float64)
    out[prefix + "_shape"] = np.array(M.shape, dtype=np.int64)


def csr_sha(M):
    M = sp.csr_matrix(M)
    return sha(M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data)


def ilut_cases():
    out, meta = {}, {}
    cases = [
        ("rand40_dt0", random_sparse(40, density=0.2, seed=0), 0.0, None),
        ("rand60_dt0", random_sparse(60, density=0.15, seed=4), 0.0, None),
        ("rand60_dt1e-3", random_sparse(60, density=0.15, seed=4), 1e-3, None),
        ("rand60_dt1e-1", random_sparse(60, density=0.15, seed=4), 1e-1, None),
        ("rand25_dt1e-2", random_sparse(25, seed=1), 1e-2, None),
        ("rand30_dt0.5", random_sparse(30, seed=3), 0.5, None),
        ("rand50_cap3", random_sparse(50, density=0.4, seed=5), 0.0, 3),
        ("rand80_cap2_dt1e-3", random_sparse(80, density=0.3, seed=9), 1e-3, 2),
        ("antidiag2", sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]])), 1e-2, None),
        ("zero3", sp.csr_matrix((3, 3)), 1e-2, None),
        ("lap1d8_dt0", lap1d(8), 0.0, None),
        ("lap3d5_dt1e-2", laplacian3d(ProblemSpec(5, 5, 5, shift=0.3)), 1e-2, None),
    ]
    for name, A, dt, cap in cases:
        f = ilut(A, droptol=dt, fill_cap=cap)
        csr_parts(name + "_A", A, out)
        csr_parts(name + "_L", f.L, out)
        csr_parts(name + "_U", f.U, out)
        meta[name] = {"droptol": dt, "fill_cap": cap, "pivot_repairs": f.pivot_repairs,
                      "nnz": int(f.nnz)}
    np.savez_compressed(os.path.join(HERE, "ilut_cases.npz"), **out)
    return meta


def partition_cases():
    out, meta = {}, {}
    cases = [
        ("lap1d6_s2", lap1d(6), 2),
        ("lap1d20_s4", lap1d(20), 4),
        ("lap3d8_s5", laplacian3d(ProblemSpec(8, 8, 8)), 5),
        ("lap3d8_s8", laplacian3d(ProblemSpec(8, 8, 8)), 8),
        ("rand100_s6", random_sparse(100, seed=3), 6),
        ("twopaths_s2", sp.block_diag([lap1d(3), lap1d(3)], format="csr"), 2),
        ("lap2d64_s4", laplacian3d(ProblemSpec(64, 64, 1, shift=2.3)), 4),
        ("lap3d12_s7", laplacian3d(ProblemSpec(12, 12, 12, shift=0.05)), 7),
        ("lap3d32_s35", laplacian3d(ProblemSpec(32, 32, 32, shift=0.16)), 35),
        ("upw3d16_s16", upwind3d(16, 16, 16, 0.2, 0.5), 16),
    ]
    for name, A, s in cases:
        spec = partition_graph(A, s)
        ps = classify_and_reorder(A, spec)
        out[name + "_assignment"] = spec.assignment.astype(np.int16)
        out[name + "_forward"] = ps.perm.forward.astype(np.int32)
        meta[name] = {"s": s, "n": int(A.shape[0]), "p": ps.p, "q": ps.q,
                      "interior_sizes": ps.interior_sizes.tolist(),
                      "interface_sizes": ps.interface_sizes.tolist(),
                      "matrix_sha": csr_sha(ps.matrix), "B_sha": csr_sha(ps.B),
                      "E_sha": csr_sha(ps.E), "F_sha": csr_sha(ps.F), "C_sha": csr_sha(ps.C)}
    np.savez_compressed(os.path.join(HERE, "partition_cases.npz"), **out)
    return meta


def apply_case(name, A, s, m, r, droptol, seed=0, vec_seed=1, store_factors=True):
    """Build with the reference, then record every hot-path operator output."""
    t0 = time.perf_counter()
    cfg = PslrConfig(num_subdomains=s, series_degree=m, rank=r, droptol=droptol, seed=seed)
    P = build(A, cfg)
    ps, ctx, lr = P.system, P.ctx, P.correction
    rng = np.random.default_rng(vec_seed)
    b = rng.standard_normal(ps.n)
    v = rng.standard_normal(ps.q)
    f = rng.standard_normal(ps.p)
    out = {"b": b, "v": v, "f": f,
           "apply": P.apply(b), "apply_original": P.apply_original(b),
           "solve_B": solve_B(ctx, f), "solve_C0": solve_C0(ctx, v),
           "apply_Es": apply_Es(ctx, v) if ps.q else np.zeros(0),
           "apply_neumann": apply_neumann(ctx, m, v) if ps.q else np.zeros(0),
           "apply_Err": apply_Err(ctx, m, v) if ps.q else np.zeros(0),
           "apply_correction": apply_correction(lr, v) if ps.q else np.zeros(0),
           "V": lr.V, "H": lr.H, "G": lr.G,
           "assignment": partition_graph(A, s).assignment.astype(np.int16),
           "forward": ps.perm.forward.astype(np.int32),
           "interior_sizes": ps.interior_sizes, "interface_sizes": ps.interface_sizes}
    csr_parts("A", A, out)
    if store_factors:
        csr_parts("LB", ctx.b_ilu.L, out)
        csr_parts("UB", ctx.b_ilu.U, out)
        csr_parts("LC", ctx.c0_ilu.L, out)
        csr_parts("UC", ctx.c0_ilu.U, out)
    np.savez_compressed(os.path.join(HERE, f"apply_{name}.npz"), **out)
    meta = {"s": s, "m": m, "rank": r, "droptol": droptol, "seed": seed, "vec_seed": vec_seed,
            "n": ps.n, "p": ps.p, "q": ps.q, "achieved_rank": lr.rank,
            "nnz_LB": int(ctx.b_ilu.L.nnz), "nnz_UB": int(ctx.b_ilu.U.nnz),
            "nnz_LC": int(ctx.c0_ilu.L.nnz), "nnz_UC": int(ctx.c0_ilu.U.nnz),
            "nnz_E": int(ps.E.nnz), "nnz_F": int(ps.F.nnz), "nnz_Cg": int(ctx.Cg.nnz),
            "LB_sha": csr_sha(ctx.b_ilu.L), "UB_sha": csr_sha(ctx.b_ilu.U),
            "LC_sha": csr_sha(ctx.c0_ilu.L), "UC_sha": csr_sha(ctx.c0_ilu.U),
            "Cg_sha": csr_sha(ctx.Cg), "matrix_sha": csr_sha(ps.matrix),
            "stats": json.loads(P.stats.to_json()), "secs": time.perf_counter() - t0}
    return P, meta


def solve_reordered(A, P, tol, maxit, restart, seed=0):
    """cli._solve_with (pkg/src/pslr/cli.py:131-143): reordered space, Ap @ v."""
    b = A @ np.random.default_rng(seed).standard_normal(A.shape[0])
    perm = P.system.perm
    Ap = P.system.matrix
    bp = b[perm.inverse]
    t0 = time.perf_counter()
    _, rep = gmres(lambda v: Ap @ v, P.apply, bp, tol=tol, maxit=maxit, restart=restart)
    return rep, time.perf_counter() - t0


def solve_original(A, P, tol, maxit, restart, seed):
    """Acceptance-test driver (pkg/tests/test_acceptance.py:39-44): original space."""
    b = A @ np.random.default_rng(seed).standard_normal(A.shape[0])
    _, rep = gmres(lambda v: A @ v, P.apply_original, b, tol=tol, maxit=maxit, restart=restart)
    return rep


def main(which="all"):
    golden = {}
    path = os.path.join(HERE, "golden.json")
    if os.path.exists(path):
        golden = json.load(open(path))
    golden["_generated_by"] = "tests/golden/make_golden.py against /root/reference/pkg/src (pslr 0.1.0)"
    golden["ilut"] = ilut_cases()
    golden["partition"] = partition_cases()
    apply_meta = golden.setdefault("apply", {})
    gm = golden.setdefault("gmres", {})

    # small operator cases (dense-checkable), incl. exact factors and a nonsymmetric matrix
    for name, A, s, m, r, dt in [
        ("lap3d6_s4_dt1e-2", laplacian3d(ProblemSpec(6, 6, 6, shift=0.3)), 4, 2, 8, 1e-2),
        ("lap3d6_s4_dt0", laplacian3d(ProblemSpec(6, 6, 6)), 4, 3, 6, 0.0),
        ("rand80_s4", random_sparse(80, density=0.08, seed=5), 4, 1, 5, 1e-2),
        ("lap1d30_s1", lap1d(30), 1, 3, 15, 0.0),
        ("upw3d8_s4", upwind3d(8, 8, 8, 0.2, 0.5), 4, 5, 10, 1e-2),
    ]:
        P, meta = apply_case(name, A, s, m, r, dt)
        apply_meta[name] = meta
    # cfg1 as BASELINE states it (2D 64^2, L - 0.3I == laplacian3d(64,64,1, shift=2.3))
    A1 = laplacian3d(ProblemSpec(64, 64, 1, shift=2.3))
    P1, meta = apply_case("cfg1", A1, 4, 3, 16, 1e-2)
    apply_meta["cfg1"] = meta
    rep, secs = solve_reordered(A1, P1, tol=1e-6, maxit=500, restart=50)
    gm["cfg1_gmres50"] = {"converged": rep.converged, "iterations": rep.iterations,
                          "final_relres": rep.final_relres, "history_first_cycle": rep.history[:51],
                          "secs": secs}
    # criterion 11 (12^3 shift 0.05, s=6, r=10, defaults m=3, full GMRES tol 1e-8): 13 its
    A11 = laplacian3d(ProblemSpec(12, 12, 12, shift=0.05))
    P11, meta = apply_case("crit11", A11, 6, 3, 10, 1e-2)
    apply_meta["crit11"] = meta
    rep, secs = solve_reordered(A11, P11, tol=1e-8, maxit=500, restart=0)
    gm["crit11"] = {"converged": rep.converged, "iterations": rep.iterations,
                    "final_relres": rep.final_relres, "secs": secs}
    json.dump(golden, open(path, "w"), indent=1, sort_keys=True)
    if which == "small":
        return

    # criterion 07 instance (32^3 shift 0.16, s=35, r=15, seed 2): its per m (full GMRES, tol 1e-8)
    A7 = laplacian3d(ProblemSpec(32, 32, 32, shift=0.16))
    crit7 = {}
    for m in (3, 5):
        P7, meta = apply_case(f"crit07_m{m}", A7, 35, m, 15, 1e-2, seed=2, store_factors=False)
        apply_meta[f"crit07_m{m}"] = meta
        rep = solve_original(A7, P7, tol=1e-8, maxit=500, restart=0, seed=2)
        crit7[str(m)] = {"converged": rep.converged, "iterations": rep.iterations}
        rep2, secs = solve_reordered(A7, P7, tol=1e-8, maxit=500, restart=0, seed=2)
        crit7[f"{m}_reordered"] = {"converged": rep2.converged, "iterations": rep2.iterations,
                                   "secs": secs}
    gm["crit07"] = crit7
    json.dump(golden, open(path, "w"), indent=1, sort_keys=True)

    # converging twins: cfg2 twin and cfg3 twin, GMRES(50) tol 1e-6, seed 0
    A2 = laplacian3d(ProblemSpec(32, 32, 32, shift=0.16))
    P2, meta = apply_case("twin_cfg2", A2, 16, 3, 32, 1e-2, store_factors=False)
    apply_meta["twin_cfg2"] = meta
    rep, secs = solve_reordered(A2, P2, tol=1e-6, maxit=500, restart=50)
    gm["twin_cfg2"] = {"converged": rep.converged, "iterations": rep.iterations,
                       "final_relres": rep.final_relres, "secs": secs}
    json.dump(golden, open(path, "w"), indent=1, sort_keys=True)
    A3 = upwind3d(32, 32, 32, 0.2, 0.5)
    P3, meta = apply_case("twin_cfg3", A3, 16, 5, 64, 1e-2, store_factors=False)
    apply_meta["twin_cfg3"] = meta
    rep, secs = solve_reordered(A3, P3, tol=1e-6, maxit=500, restart=50)
    gm["twin_cfg3"] = {"converged": rep.converged, "iterations": rep.iterations,
                       "final_relres": rep.final_relres, "secs": secs}
    json.dump(golden, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
