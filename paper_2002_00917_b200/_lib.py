"""ctypes binding of libpslr.so (the C-ABI declared in include/pslr.h).

The library is built in-tree (paper_2002_00917_b200/lib/libpslr.so, see
`__graft_entry__.build()` / `make -C paper_2002_00917_b200/csrc`).  There is
no fallback: if the library is missing or cannot be loaded, importing this
module raises ImportError, and every device operator raises when no CUDA
device is present.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSLR_LIB: an alternative build of the same library (timing experiments, tools/)
LIB_PATH = os.environ.get("PSLR_LIB") or os.path.join(_HERE, "lib", "libpslr.so")

PSLR_OK, PSLR_EDIM, PSLR_ENONFINITE, PSLR_ESINGULAR, PSLR_ECUDA, PSLR_EINVAL, PSLR_ENOMEM, \
    PSLR_ENCCL, PSLR_ENOTSPD, PSLR_ECALLBACK = range(10)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libpslr.so not found at {LIB_PATH}: build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")

lib = ctypes.CDLL(LIB_PATH)

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
P = ctypes.c_void_p
# pslr_vec_fn: int (*)(void* user, const double* x_dev, double* y_dev, void* stream)
VEC_FN = ctypes.CFUNCTYPE(c_int, P, P, P, P)


class Csr(ctypes.Structure):
    _fields_ = [("nrows", c_i64), ("ncols", c_i64), ("nnz", c_i64),
                ("indptr", P), ("indices", P), ("data", P)]


class System(ctypes.Structure):
    _fields_ = [("n", c_i64), ("p", c_i64), ("q", c_i64), ("s", c_i64),
                ("interior_offsets", P), ("interface_offsets", P),
                ("LB", Csr), ("UB", Csr), ("LC", Csr), ("UC", Csr),
                ("E", Csr), ("F", Csr), ("C", Csr), ("C0", Csr), ("Cg", Csr), ("A", Csr)]


class CtxInfo(ctypes.Structure):
    _fields_ = [(k, c_i64) for k in (
        "n", "p", "q", "s", "rank",
        "levels_LB", "levels_UB", "levels_LC", "levels_UC",
        "maxdepth_LB", "maxdepth_UB", "maxdepth_LC", "maxdepth_UC",
        "nnz_LB", "nnz_UB", "nnz_LC", "nnz_UC", "nnz_E", "nnz_F", "nnz_C", "nnz_C0", "nnz_Cg",
        "nnz_A", "device_bytes", "sm_count", "ring_slots", "stages", "far_deps", "reach", "nghost")]


def _sig(name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


# every symbol declared in include/pslr.h (tests/test_abi.py checks the list against the header)
EXPORTS = {
    "pslr_last_error": (ctypes.c_char_p,),
    "pslr_abi_version": (c_int,),
    "pslr_partition_bisect": (c_int, c_i64, P, P, c_i64, P),
    "pslr_ilut_blocks": (c_int, c_i64, P, P, P, c_i64, P, c_dbl, c_i64, c_int,
                         ctypes.POINTER(P), ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                         ctypes.POINTER(c_i64)),
    "pslr_factors_fetch": (c_int, P, P, P, P, P, P, P, P, P),
    "pslr_factors_free": (None, P),
    "pslr_row_norms": (c_int, c_i64, P, P, P),
    "pslr_ctx_create": (c_int, ctypes.POINTER(P), c_int, ctypes.POINTER(System)),
    "pslr_ctx_create_packed": (c_int, ctypes.POINTER(P), c_int, ctypes.POINTER(System), P, c_i64,
                               ctypes.POINTER(P), ctypes.POINTER(c_i64), ctypes.POINTER(c_int)),
    "pslr_blob_free": (None, P),
    "pslr_ctx_destroy": (None, P),
    "pslr_ctx_info": (c_int, P, ctypes.POINTER(CtxInfo)),
    "pslr_ctx_set_correction": (c_int, P, c_i64, P, P),
    "pslr_ctx_set_correction_device": (c_int, P, c_i64, P, P),
    "pslr_solve_B": (c_int, P, P, P, P),
    "pslr_solve_C0": (c_int, P, P, P, P),
    "pslr_apply_S": (c_int, P, P, P, P),
    "pslr_apply_Es": (c_int, P, P, P, P),
    "pslr_apply_neumann": (c_int, P, c_i64, P, P, P),
    "pslr_apply_Err": (c_int, P, c_i64, P, P, P),
    "pslr_apply_correction": (c_int, P, P, P, P),
    "pslr_apply": (c_int, P, c_i64, P, P, P),
    "pslr_spmv": (c_int, P, c_int, P, P, P),
    "pslr_apply_host": (c_int, P, c_i64, P, P, P),
    "pslr_apply_host_async": (c_int, P, c_i64, P, P, P),
    "pslr_apply_multi": (c_int, P, c_i64, c_i64, P, P, P),
    "pslr_apply_multi_host_async": (c_int, P, c_i64, c_i64, P, P, P),
    "pslr_ctx_clone": (c_int, P, ctypes.POINTER(P)),
    "pslr_apply_first": (c_int, P, P, P, P, P),
    "pslr_apply_mid": (c_int, P, P, P, P, P),
    "pslr_apply_horner": (c_int, P, P, P, P, P),
    "pslr_halo_pending": (c_int, P, P),
    "pslr_apply_last": (c_int, P, P, P, P, P),
    "pslr_apply2_first": (c_int, P, P, P, P, P),
    "pslr_apply2_mid": (c_int, P, P, P, P, P),
    "pslr_apply2_horner": (c_int, P, P, P, P, P),
    "pslr_apply2_last": (c_int, P, P, P, P, P),
    "pslr_apply_es_step": (c_int, P, P, P, c_int, P),
    "pslr_apply_profiled": (c_int, P, c_i64, P, P, P, P, P, c_i64, ctypes.POINTER(c_i64)),
    "pslr_debug_trace": (c_int, P, P, c_i64, ctypes.POINTER(c_i64)),
    "pslr_arnoldi": (c_int, P, c_i64, c_i64, P, P, P, ctypes.POINTER(c_i64), P),
    "pslr_gmres": (c_int, P, c_i64, P, P, c_dbl, c_i64, c_i64, c_int, c_int,
                   ctypes.POINTER(c_i64), ctypes.POINTER(c_int), ctypes.POINTER(c_dbl), P,
                   ctypes.POINTER(c_i64), P),
    "pslr_comm_unique_id": (c_int, P),
    "pslr_comm_init": (c_int, P, P, c_int, c_int),
    "pslr_ctx_set_halo": (c_int, P, c_int, P, P, P),
    "pslr_cgs_pass": (c_int, P, c_int, P, c_i64, c_i64, c_i64, P, P, P, P),
    "pslr_cg": (c_int, P, c_i64, P, P, c_dbl, c_i64, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_int),
                ctypes.POINTER(c_dbl), P, ctypes.POINTER(c_i64), P),
    "pslr_workspace_create": (c_int, ctypes.POINTER(P), c_int),
    "pslr_csr_spmv": (c_int, c_i64, c_i64, P, P, P, P, P, P),
    "pslr_arnoldi_op": (c_int, P, c_i64, VEC_FN, P, c_i64, P, P, P, ctypes.POINTER(c_i64), P),
    "pslr_gmres_op": (c_int, P, c_i64, c_i64, VEC_FN, P, VEC_FN, P, c_int, P, P, c_dbl, c_i64, c_i64, c_int,
                      ctypes.POINTER(c_i64), ctypes.POINTER(c_int), ctypes.POINTER(c_dbl), P,
                      ctypes.POINTER(c_i64), P),
    "pslr_cg_op": (c_int, P, c_i64, c_i64, VEC_FN, P, VEC_FN, P, c_int, P, P, c_dbl, c_i64,
                   ctypes.POINTER(c_i64), ctypes.POINTER(c_int), ctypes.POINTER(c_dbl), P,
                   ctypes.POINTER(c_i64), P),
}

fns = {name: _sig(name, sig[0], *sig[1:]) for name, sig in EXPORTS.items()}


class CorrectionSingularError(RuntimeError):
    """I - H is numerically singular (lowrank.py:22-23)."""


class NotSpdError(RuntimeError):
    """CG hit a non-positive curvature direction: matrix not SPD (krylov.py:18-19)."""


def check(rc: int):
    """Map a C-ABI status to the reference's exception types (include/pslr.h)."""
    if rc == PSLR_OK:
        return
    msg = fns["pslr_last_error"]().decode(errors="replace")
    if rc in (PSLR_EDIM, PSLR_EINVAL):
        raise ValueError(msg)
    if rc == PSLR_ENONFINITE:
        raise ArithmeticError(msg)
    if rc == PSLR_ESINGULAR:
        raise CorrectionSingularError(msg)
    if rc == PSLR_ENOTSPD:
        raise NotSpdError(msg)
    raise RuntimeError(f"libpslr error {rc}: {msg}")


def ptr(a) -> int | None:
    """Address of a contiguous numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def csr_struct(M, keep: list) -> Csr:
    """pslr_csr view of a scipy CSR matrix; arrays appended to `keep` stay alive."""
    ip = np.ascontiguousarray(M.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(M.indices, dtype=np.int32)
    dv = np.ascontiguousarray(M.data, dtype=np.float64)
    keep += [ip, ix, dv]
    return Csr(M.shape[0], M.shape[1], int(dv.size), ip.ctypes.data, ix.ctypes.data, dv.ctypes.data)
