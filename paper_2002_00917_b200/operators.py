"""Operators for the generic Krylov drivers (krylov.py / lowrank.py with arbitrary
apply_A / apply_M / op, as the reference's gmres, cg and arnoldi accept).

The Krylov state (basis, CGS2 projections, norms, Givens) always lives on the device
(libpslr.so's pslr_gmres_op / pslr_cg_op / pslr_arnoldi_op).  An operator reaches it as a
C callback (include/pslr.h `pslr_vec_fn`):

  * the preconditioner's own operators (P.matvec, P.apply, their original-space forms)
    run on the device, no host round trip;
  * a scipy sparse matrix is uploaded once and applied by libpslr's CSR SpMV kernel
    (scipy csr_matvec order: bit-identical to A @ v);
  * any other callable or scipy LinearOperator is the reference's contract — a function
    of host vectors — so its input is copied to the host and its output back (the only
    host work per iteration is the user's own function).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_workspaces: dict = {}


def workspace(device: int):
    """A `pslr_workspace_create` context (device scratch only) per CUDA device."""
    ws = _workspaces.get(device)
    if ws is None:
        from .device import require_cuda
        t = require_cuda()
        h = ctypes.c_void_p()
        with t.cuda.device(device):
            _lib.check(_lib.fns["pslr_workspace_create"](ctypes.byref(h), int(device)))
        ws = _Handle(h)
        _workspaces[device] = ws
    return ws


class _Handle:
    def __init__(self, h):
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.fns["pslr_ctx_destroy"](h)
            except Exception:
                pass


class _DevArray:
    """A device pointer as a torch tensor (zero copy, __cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def as_tensor(ptr: int, n: int, device):
    from .device import torch_mod
    return torch_mod().as_tensor(_DevArray(ptr, n), device=device)


class Operator:
    """A linear operator on device n-vectors behind a pslr_vec_fn callback.  Exceptions
    raised inside are kept and re-raised by `check` after the driver returns."""

    def __init__(self, fn_dev, n: int, device):
        self.n, self.device = n, device
        self.error = None
        self._fn = fn_dev  # (x_tensor, y_tensor) -> None, on the current stream

        def cb(user, x, y, stream):
            try:
                self._fn(as_tensor(x, n, device), as_tensor(y, n, device))
                return 0
            except BaseException as exc:  # noqa: BLE001  (re-raised by check())
                self.error = exc
                return 1

        self.cfunc = _lib.VEC_FN(cb)

    def check(self, rc: int):
        if rc == _lib.PSLR_ECALLBACK and self.error is not None:
            err, self.error = self.error, None
            raise err


def _host_fn(apply, n):
    """The reference contract: apply maps host float64 vectors to host vectors."""
    from .device import torch_mod
    t = torch_mod()
    try:
        import scipy.sparse.linalg as spla
        f = apply.matvec if isinstance(apply, spla.LinearOperator) else apply
    except ImportError:  # pragma: no cover
        f = apply

    def run(x, y):
        t.cuda.current_stream(x.device).synchronize()
        out = np.asarray(f(x.cpu().numpy()), dtype=np.float64).reshape(-1)
        if out.shape[0] != n:
            raise ValueError(f"operator returned a vector of length {out.shape[0]}, expected {n}")
        y.copy_(t.from_numpy(np.ascontiguousarray(out)), non_blocking=False)
    return run


class _CsrOnDevice:
    """A scipy sparse matrix uploaded once (int32 indices, fp64 values)."""

    def __init__(self, M, device):
        import scipy.sparse as sp
        from .device import torch_mod
        t = torch_mod()
        M = sp.csr_matrix(M, dtype=np.float64)  # entry order kept: csr_matvec's summation order
        self.shape = M.shape
        self.indptr = t.as_tensor(M.indptr.astype(np.int32), device=device)
        self.indices = t.as_tensor(M.indices.astype(np.int32), device=device)
        self.data = t.as_tensor(M.data.astype(np.float64), device=device)

    def __call__(self, x, y):
        from .device import torch_mod
        st = torch_mod().cuda.current_stream(x.device).cuda_stream
        _lib.check(_lib.fns["pslr_csr_spmv"](self.shape[0], self.shape[1], self.indptr.data_ptr(),
                                             self.indices.data_ptr(), self.data.data_ptr(), x.data_ptr(),
                                             y.data_ptr(), st))


def is_sparse_matrix(obj) -> bool:
    try:
        import scipy.sparse as sp
        return sp.issparse(obj)
    except Exception:
        return False


def make_operator(apply, n: int, device) -> Operator:
    """Operator for apply_A / apply_M / op (see the module docstring)."""
    from .preconditioner import PslrPreconditioner
    owner = getattr(apply, "__self__", None)
    name = getattr(getattr(apply, "__func__", None), "__name__", None)
    if isinstance(owner, PslrPreconditioner) and name in ("apply", "apply_original", "matvec",
                                                          "matvec_original"):
        bound = getattr(owner, name)  # device tensors in, device tensors out

        def dev_fn(x, y):
            y.copy_(bound(x))
        return Operator(dev_fn, n, device)
    if is_sparse_matrix(apply):
        if apply.shape != (n, n):
            raise ValueError(f"operator has shape {apply.shape}, system is {n}-dimensional")
        return Operator(_CsrOnDevice(apply, device), n, device)  # uploaded once per solve
    if not callable(apply) and not hasattr(apply, "matvec"):
        raise TypeError("operator must be callable, a scipy sparse matrix or a LinearOperator")
    return Operator(_host_fn(apply, n), n, device)


def null_fn():
    return _lib.VEC_FN()
