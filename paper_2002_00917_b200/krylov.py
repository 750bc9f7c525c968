"""Right-preconditioned restarted GMRES / FGMRES and preconditioned CG (mirrors pslr/krylov.py).

Every solve runs on the device with the reference's exact control flow
(krylov.py:35-174): the Krylov basis, the CGS2 projections and norms are libpslr
kernels, only the (cycle+1)-sized Givens / least-squares scalars are host code.

  * A PSLR preconditioner's own operator pair (A = P.matvec, M = P.apply — the pairing
    cli._solve_with uses, cli.py:131-143 — or their original-space versions) runs
    entirely inside libpslr (pslr_gmres / pslr_cg);
  * any other apply_A / apply_M (the reference accepts arbitrary callables) reaches the
    same device loop as an operator callback (pslr_gmres_op / pslr_cg_op,
    operators.py): P's operators and scipy sparse matrices stay on the device, other
    callables are called on host vectors.
There is no host Krylov loop and no CPU fallback: without a CUDA device every solve raises.
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
    return _solve_ops("gmres", apply_A, apply_M, b, tol, maxit, restart, flexible)


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
    return _solve_ops("cg", apply_A, apply_M, b, tol, maxit)


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


def _solve_ops(kind, apply_A, apply_M, b, tol, maxit, restart=0, flexible=False):
    """The device loop for any operator pair (pslr_gmres_op / pslr_cg_op).  The context is
    the preconditioner's when M is P.apply (its apply runs inside libpslr), else a
    device workspace; A is a device operator callback (operators.py)."""
    from . import operators as ops_
    from .device import require_cuda
    t = require_cuda()
    is_tensor = hasattr(b, "data_ptr")
    P = _bound(apply_M, "apply")
    if P is not None:
        dev, handle, m, precond = P.device.dev, P.device.handle, int(P.series_degree), 1
        P.device.ensure_correction(P.correction)
        M_op = None
    else:
        owner = getattr(apply_M, "__self__", None) or getattr(apply_A, "__self__", None)
        odev = getattr(owner, "device", None)
        dev = odev.dev if hasattr(odev, "dev") else (b.device if is_tensor else
                                                     t.device("cuda", t.cuda.current_device()))
        handle, m, precond = ops_.workspace(dev.index if dev.index is not None else 0).handle, 0, 0
        M_op = None
    if is_tensor:
        bd = b.to(device=dev, dtype=t.float64).contiguous()
    else:
        bn = np.asarray(b, dtype=np.float64)
        if bn.ndim != 1:
            raise ValueError("right-hand side must be a vector")
        bd = t.from_numpy(np.ascontiguousarray(bn)).to(dev)
    n = int(bd.shape[0])
    if P is not None and n != P.system.n:
        raise ValueError(f"vector has length {n}, system is {P.system.n}-dimensional")
    A_op = ops_.make_operator(apply_A, n, dev)
    if P is None and apply_M is not None:
        M_op = ops_.make_operator(apply_M, n, dev)
    xd = t.empty(n, dtype=t.float64, device=dev)
    hist = np.zeros(max(int(maxit), 0) + 1)
    its, conv, rel, hlen = ctypes.c_int64(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int64()
    st = t.cuda.current_stream(dev).cuda_stream
    Mf = M_op.cfunc if M_op is not None else ops_.null_fn()
    t0 = time.perf_counter()
    with t.cuda.device(dev):
        if kind == "gmres":
            rc = _lib.fns["pslr_gmres_op"](handle, m, n, A_op.cfunc, None, Mf, None, precond, bd.data_ptr(),
                                           xd.data_ptr(), float(tol), int(maxit), int(restart),
                                           1 if flexible else 0, ctypes.byref(its), ctypes.byref(conv),
                                           ctypes.byref(rel), hist.ctypes.data, ctypes.byref(hlen), st)
        else:
            rc = _lib.fns["pslr_cg_op"](handle, m, n, A_op.cfunc, None, Mf, None, precond, bd.data_ptr(),
                                        xd.data_ptr(), float(tol), int(maxit), ctypes.byref(its),
                                        ctypes.byref(conv), ctypes.byref(rel), hist.ctypes.data,
                                        ctypes.byref(hlen), st)
    A_op.check(rc)
    if M_op is not None:
        M_op.check(rc)
    _lib.check(rc)
    elapsed = time.perf_counter() - t0
    rep = SolveReport(bool(conv.value), int(its.value), float(rel.value), hist[:hlen.value].tolist(), elapsed)
    return (xd if is_tensor else xd.cpu().numpy()), rep
