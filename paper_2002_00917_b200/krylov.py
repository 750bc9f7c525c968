"""Right-preconditioned restarted GMRES / FGMRES and preconditioned CG (mirrors pslr/krylov.py).

When the operator pair is a PSLR preconditioner's own (A = P.matvec,
M = P.apply — the pairing cli._solve_with uses, cli.py:131-143 — or their
original-space versions), the whole solve runs on the device: pslr_gmres
drives the apply, the A-SpMV and the CGS2 kernels with the reference's exact
control flow (krylov.py:55-127), only the (cycle+1)-sized Givens/least-squares
bookkeeping is scalar host code; pslr_cg does the same for CG (krylov.py:132-174).  Arbitrary Python callables keep the
reference's generic contract.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib


NotSpdError = _lib.NotSpdError  # krylov.py:18-19 (raised by the device CG through its status code)


@dataclass
class SolveReport:
    """krylov.py:22-28."""
    converged: bool
    iterations: int
    final_relres: float
    history: list = field(default_factory=list)  # relative residuals, history[0] = 1.0
    time_s: float = 0.0


def _identity(v):
    return v


def _bound(fn, name):
    """The PslrPreconditioner a bound method `fn` belongs to, if it is P.<name>."""
    from .preconditioner import PslrPreconditioner
    owner = getattr(fn, "__self__", None)
    if isinstance(owner, PslrPreconditioner) and getattr(fn, "__func__", None) is \
            getattr(PslrPreconditioner, name):
        return owner
    return None


def gmres(apply_A, apply_M, b, tol: float = 1e-8, maxit: int = 500, restart: int = 0,
          flexible: bool = False):
    """Solve A x = b with right preconditioning (krylov.py:35-129). restart=0: full GMRES.
    flexible=True: FGMRES (Z_j = M v_j kept, x += Z y).  Returns (x, SolveReport)."""
    P = _bound(apply_M, "apply")
    if P is not None and _bound(apply_A, "matvec") is P:
        return gmres_device(P, b, tol, maxit, restart, flexible)
    P = _bound(apply_M, "apply_original")
    if P is not None and _bound(apply_A, "matvec_original") is P:
        perm = P.system.perm
        x, rep = gmres_device(P, np.asarray(b, dtype=np.float64)[perm.inverse], tol, maxit,
                              restart, flexible)
        return x[perm.forward], rep
    return _gmres_generic(apply_A, apply_M, b, tol, maxit, restart, flexible)


def fgmres(apply_A, apply_M, b, tol: float = 1e-8, maxit: int = 500, restart: int = 0):
    """Flexible GMRES (config 3's accelerator; absent from the reference)."""
    return gmres(apply_A, apply_M, b, tol, maxit, restart, flexible=True)


def gmres_device(P, b, tol: float = 1e-8, maxit: int = 500, restart: int = 0,
                 flexible: bool = False, precond: bool = True):
    """The device solve (pslr_gmres) in P's reordered space; b numpy or CUDA tensor."""
    from .device import torch_mod
    t = torch_mod()
    dev = P.device
    dev.ensure_correction(P.correction)
    n = P.system.n
    is_tensor = hasattr(b, "data_ptr")
    if is_tensor:
        bd = b.contiguous()
    else:
        b = np.asarray(b, dtype=np.float64)
        if b.shape[0] != n:
            raise ValueError(f"vector has length {b.shape[0]}, system is {n}-dimensional")
        bd = t.from_numpy(np.ascontiguousarray(b)).to(dev.dev)
    xd = t.empty(n, dtype=t.float64, device=dev.dev)
    hist = np.zeros(int(maxit) + 1)
    its, conv, rel, hlen = ctypes.c_int64(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int64()
    t0 = time.perf_counter()
    _lib.check(_lib.fns["pslr_gmres"](
        dev.handle, int(P.series_degree), bd.data_ptr(), xd.data_ptr(), float(tol), int(maxit),
        int(restart), 1 if precond else 0, 1 if flexible else 0, ctypes.byref(its),
        ctypes.byref(conv), ctypes.byref(rel), hist.ctypes.data, ctypes.byref(hlen), dev.stream()))
    elapsed = time.perf_counter() - t0
    rep = SolveReport(bool(conv.value), int(its.value), float(rel.value),
                      hist[:hlen.value].tolist(), elapsed)
    return (xd if is_tensor else xd.cpu().numpy()), rep


def cg(apply_A, apply_M, b, tol: float = 1e-8, maxit: int = 500):
    """Preconditioned conjugate gradient for SPD systems, zero initial guess (krylov.py:132-174).
    On a PSLR preconditioner's own operator pair (the CLI's `--krylov cg`, cli.py:138-139)
    the whole loop runs on the device (pslr_cg)."""
    P = _bound(apply_M, "apply")
    if P is not None and _bound(apply_A, "matvec") is P:
        return cg_device(P, b, tol, maxit)
    P = _bound(apply_M, "apply_original")
    if P is not None and _bound(apply_A, "matvec_original") is P:
        perm = P.system.perm
        x, rep = cg_device(P, np.asarray(b, dtype=np.float64)[perm.inverse], tol, maxit)
        return x[perm.forward], rep
    return _cg_generic(apply_A, apply_M, b, tol, maxit)


def cg_device(P, b, tol: float = 1e-8, maxit: int = 500, precond: bool = True):
    """The device CG (pslr_cg) in P's reordered space; b numpy or CUDA tensor."""
    from .device import torch_mod
    t = torch_mod()
    dev = P.device
    dev.ensure_correction(P.correction)
    n = P.system.n
    is_tensor = hasattr(b, "data_ptr")
    if is_tensor:
        bd = b.contiguous()
    else:
        b = np.asarray(b, dtype=np.float64)
        if b.shape[0] != n:
            raise ValueError(f"vector has length {b.shape[0]}, system is {n}-dimensional")
        bd = t.from_numpy(np.ascontiguousarray(b)).to(dev.dev)
    xd = t.empty(n, dtype=t.float64, device=dev.dev)
    hist = np.zeros(max(int(maxit), 0) + 1)
    its, conv, rel, hlen = ctypes.c_int64(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int64()
    t0 = time.perf_counter()
    _lib.check(_lib.fns["pslr_cg"](
        dev.handle, int(P.series_degree), bd.data_ptr(), xd.data_ptr(), float(tol), int(maxit),
        1 if precond else 0, ctypes.byref(its), ctypes.byref(conv), ctypes.byref(rel),
        hist.ctypes.data, ctypes.byref(hlen), dev.stream()))
    elapsed = time.perf_counter() - t0
    rep = SolveReport(bool(conv.value), int(its.value), float(rel.value),
                      hist[:hlen.value].tolist(), elapsed)
    return (xd if is_tensor else xd.cpu().numpy()), rep


def _cg_generic(apply_A, apply_M, b, tol, maxit):
    """The reference recurrence for arbitrary callables (krylov.py:132-174)."""
    if apply_M is None:
        apply_M = _identity
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    t0 = time.perf_counter()
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), SolveReport(True, 0, 0.0, [1.0], time.perf_counter() - t0)
    x = np.zeros(n)
    r = b.copy()
    z = np.asarray(apply_M(r), dtype=np.float64)
    p = z.copy()
    rz = r @ z
    history = [1.0]
    converged = False
    relres = 1.0
    it = 0
    for it in range(1, maxit + 1):
        Ap = np.asarray(apply_A(p), dtype=np.float64)
        pAp = p @ Ap
        if pAp <= 0.0:
            raise NotSpdError("matrix not SPD: non-positive curvature encountered")
        alpha = rz / pAp
        x = x + alpha * p
        r = r - alpha * Ap
        relres = np.linalg.norm(r) / bnorm
        history.append(relres)
        if relres <= tol:
            converged = True
            break
        z = np.asarray(apply_M(r), dtype=np.float64)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    iterations = it if converged else maxit
    if not converged:
        history.extend([relres] * (maxit + 1 - len(history)))
    return x, SolveReport(converged, iterations, relres, history, time.perf_counter() - t0)


def _gmres_generic(apply_A, apply_M, b, tol, maxit, restart, flexible):
    """The reference recurrence for arbitrary callables (krylov.py:35-129)."""
    if apply_M is None:
        apply_M = _identity
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    t0 = time.perf_counter()
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), SolveReport(True, 0, 0.0, [1.0], time.perf_counter() - t0)
    x = np.zeros(n)
    history = [1.0]
    total = 0
    converged = False
    relres = 1.0
    while total < maxit and not converged:
        r = b - np.asarray(apply_A(x))
        beta = np.linalg.norm(r)
        relres = beta / bnorm
        if relres <= tol:
            converged = True
            break
        cycle = maxit - total if restart <= 0 else min(restart, maxit - total)
        V = np.zeros((n, cycle + 1))
        Z = np.zeros((n, cycle)) if flexible else None
        Hcol = np.zeros((cycle + 1, cycle))
        cs = np.zeros(cycle)
        sn = np.zeros(cycle)
        g = np.zeros(cycle + 1)
        g[0] = beta
        V[:, 0] = r / beta
        j = 0
        breakdown = False
        while j < cycle:
            mv = np.asarray(apply_M(V[:, j]))
            if flexible:
                Z[:, j] = mv
            w = np.asarray(apply_A(mv), dtype=np.float64)
            h = V[:, :j + 1].T @ w
            w = w - V[:, :j + 1] @ h
            h2 = V[:, :j + 1].T @ w
            w = w - V[:, :j + 1] @ h2
            h = h + h2
            hnext = np.linalg.norm(w)
            if not (np.all(np.isfinite(h)) and np.isfinite(hnext)):
                raise ArithmeticError("GMRES diverged: non-finite values in the recurrence")
            Hcol[:j + 1, j] = h
            Hcol[j + 1, j] = hnext
            for i in range(j):
                tmp = cs[i] * Hcol[i, j] + sn[i] * Hcol[i + 1, j]
                Hcol[i + 1, j] = -sn[i] * Hcol[i, j] + cs[i] * Hcol[i + 1, j]
                Hcol[i, j] = tmp
            denom = np.hypot(Hcol[j, j], hnext)
            if denom == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = Hcol[j, j] / denom, hnext / denom
            Hcol[j, j] = denom
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            j += 1
            est = abs(g[j]) / bnorm
            history.append(est)
            if hnext <= 1e-14 * beta:
                breakdown = True
                break
            if est <= tol:
                break
            if j < cycle:
                V[:, j] = w / hnext
        if j > 0:
            y = np.zeros(j)
            for i in range(j - 1, -1, -1):
                y[i] = (g[i] - Hcol[i, i + 1:j] @ y[i + 1:j]) / Hcol[i, i]
            x = x + (Z[:, :j] @ y if flexible else np.asarray(apply_M(V[:, :j] @ y)))
        relres = np.linalg.norm(b - np.asarray(apply_A(x))) / bnorm
        history[-1] = relres
        if relres <= tol:
            converged = True
        elif breakdown:
            break
    if not converged and total < maxit and not np.isfinite(relres):
        raise ArithmeticError("GMRES diverged: non-finite residual")
    iterations = total if converged else maxit
    if not converged:
        history.extend([relres] * (maxit + 1 - len(history)))
    return x, SolveReport(converged, iterations, relres, history, time.perf_counter() - t0)
