"""Device context: owns one `pslr_ctx` (libpslr.so) per preconditioner.

PyTorch is plumbing here: device selection, streams and device buffers for
numpy<->device transfers.  All arithmetic runs in libpslr.so's sm_100a
kernels.  There is no CPU fallback: without a CUDA device every operator
raises RuntimeError.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_torch = None
# numpy vectors at least this large travel through pinned host memory (vec_op)
_PIN_BYTES = 1 << 20
_PIN_CHUNK = 1 << 20  # doubles per pipelined host-copy / DMA chunk (8 MB; tools/single_call.py)


def torch_mod():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


def require_cuda():
    t = torch_mod()
    if not t.cuda.is_available():
        raise RuntimeError("no CUDA device: the PSLR hot path runs only on the B200 "
                           "(libpslr.so, sm_100a); there is no CPU fallback")
    return t


class DeviceContext:
    """A `pslr_ctx` built from the host system + factors (pslr_ctx_create)."""

    def __init__(self, ps, b_ilu, c0_ilu, C0, Cg, device=None, packed=None, want_packed=False):
        """packed: a packed-format blob from an earlier context of the same system (the
        setup cache's pack_*.bin) — pslr_ctx_create_packed skips the level analysis and
        chunk packing when it fits; want_packed: keep the blob in use as self.packed."""
        t = require_cuda()
        if device is None:
            device = t.cuda.current_device()
        self.device = int(device)
        self.dev = t.device("cuda", self.device)
        keep = []
        empty = lambda r, c: _empty_csr(r, c)  # noqa: E731
        sysd = _lib.System()
        sysd.n, sysd.p, sysd.q, sysd.s = ps.n, ps.p, ps.q, ps.num_parts
        io = np.concatenate([[0], np.cumsum(ps.interior_sizes)]).astype(np.int64)
        fo = np.concatenate([[0], np.cumsum(ps.interface_sizes)]).astype(np.int64)
        keep += [io, fo]
        sysd.interior_offsets = io.ctypes.data
        sysd.interface_offsets = fo.ctypes.data
        sysd.LB = _lib.csr_struct(b_ilu.L, keep)
        sysd.UB = _lib.csr_struct(b_ilu.U, keep)
        sysd.LC = _lib.csr_struct(c0_ilu.L if ps.q else empty(0, 0), keep)
        sysd.UC = _lib.csr_struct(c0_ilu.U if ps.q else empty(0, 0), keep)
        sysd.E = _lib.csr_struct(ps.E, keep)
        sysd.F = _lib.csr_struct(ps.F, keep)
        sysd.C = _lib.csr_struct(ps.C, keep)
        sysd.C0 = _lib.csr_struct(C0 if ps.q else empty(0, 0), keep)
        sysd.Cg = _lib.csr_struct(Cg if ps.q else empty(0, 0), keep)
        sysd.A = _lib.csr_struct(ps.matrix, keep)
        h = ctypes.c_void_p()
        blob_out, blob_len, reused = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int()
        pin = packed if packed is not None else b""
        with t.cuda.device(self.device):
            _lib.check(_lib.fns["pslr_ctx_create_packed"](
                ctypes.byref(h), self.device, ctypes.byref(sysd), pin if pin else None, len(pin),
                ctypes.byref(blob_out) if want_packed else None, ctypes.byref(blob_len) if want_packed else None,
                ctypes.byref(reused)))
        self.handle = h
        self.packed_reused = bool(reused.value)
        self.packed = None
        if want_packed and blob_out.value:
            self.packed = ctypes.string_at(blob_out.value, blob_len.value)
            _lib.fns["pslr_blob_free"](blob_out)
        self.n, self.p, self.q, self.s = ps.n, ps.p, ps.q, ps.num_parts

    # ------------------------------------------------------------------ plumbing
    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.fns["pslr_ctx_destroy"](h)
            except Exception:  # interpreter shutdown
                pass
            self.handle = None

    def clone(self) -> "DeviceContext":
        """A context sharing this one's factors, matrices and correction, with its own
        scratch (pslr_ctx_clone): independent applies on another stream.  Keeps a
        reference to this context, which must outlive it."""
        h = ctypes.c_void_p()
        with torch_mod().cuda.device(self.device):
            _lib.check(_lib.fns["pslr_ctx_clone"](self.handle, ctypes.byref(h)))
        c = object.__new__(DeviceContext)
        c.device, c.dev, c.handle = self.device, self.dev, h
        c.n, c.p, c.q, c.s = self.n, self.p, self.q, self.s
        c._parent = self
        c._bound = getattr(self, "_bound", None)
        return c

    def info(self) -> dict:
        inf = _lib.CtxInfo()
        _lib.check(_lib.fns["pslr_ctx_info"](self.handle, ctypes.byref(inf)))
        return {k: int(getattr(inf, k)) for k, _ in _lib.CtxInfo._fields_}

    def stream(self) -> int:
        return torch_mod().cuda.current_stream(self.dev).cuda_stream

    def ensure_correction(self, corr):
        """Make `corr` (a LowRankCorrection) the correction state the device applies."""
        if getattr(self, "_bound", None) is not corr:
            self.set_correction(corr.V if corr.rank else None, corr.G if corr.rank else None)
            self._bound = corr

    def set_correction(self, V, G):
        """Upload a LowRankCorrection (V host numpy or device tensor, G host)."""
        t = torch_mod()
        r = 0 if V is None else int(V.shape[1])
        G = np.ascontiguousarray(G if G is not None else np.zeros((0, 0)), dtype=np.float64)
        if isinstance(V, t.Tensor):
            V = V.contiguous()
            _lib.check(_lib.fns["pslr_ctx_set_correction_device"](self.handle, r, V.data_ptr(),
                                                                  G.ctypes.data))
            self._bound = None
        else:
            Vh = np.ascontiguousarray(V if V is not None else np.zeros((self.q, 0)), dtype=np.float64)
            _lib.check(_lib.fns["pslr_ctx_set_correction"](self.handle, r, Vh.ctypes.data,
                                                           G.ctypes.data))
        self._bound = None  # the state no longer belongs to a LowRankCorrection object

    def vec_op(self, name, x, n_in, n_out, *scalars):
        """Run a vector->vector C-ABI operator on numpy (copied) or CUDA-tensor (zero-copy) input."""
        t = torch_mod()
        if isinstance(x, t.Tensor):
            if x.device != self.dev or x.dtype != t.float64:
                raise ValueError("device vectors must be float64 CUDA tensors on the context's device")
            if x.dim() != 1 or x.shape[0] != n_in:
                raise ValueError(f"vector has length {x.shape[0]}, operator expects {n_in}")
            xt = x.contiguous()
            out = t.empty(n_out, dtype=t.float64, device=self.dev)
            _lib.check(_lib.fns[name](self.handle, *scalars, xt.data_ptr(), out.data_ptr(), self.stream()))
            return out
        xa = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        if xa.ndim != 1 or xa.shape[0] != n_in:
            raise ValueError(f"vector has length {xa.shape[0]}, operator expects {n_in}")
        if xa.nbytes < _PIN_BYTES:
            xt = t.from_numpy(xa).to(self.dev)
            out = t.empty(n_out, dtype=t.float64, device=self.dev)
            _lib.check(_lib.fns[name](self.handle, *scalars, xt.data_ptr(), out.data_ptr(), self.stream()))
            return out.cpu().numpy()
        # large vectors: the input goes through torch's pinned host cache (its copy into
        # pinned memory runs on the intra-op threads), both DMA copies are asynchronous on
        # the operator's stream, and the result lands in a pinned host array returned as is
        # (a fresh array, as the reference returns): no pageable, driver-staged transfer
        # the host copy into pinned memory and the DMA overlap chunk by chunk
        src = t.from_numpy(xa)
        xp = t.empty(n_in, dtype=t.float64, pin_memory=True)
        xt = t.empty(n_in, dtype=t.float64, device=self.dev)
        step = _PIN_CHUNK
        for i in range(0, n_in, step):
            xp[i:i + step].copy_(src[i:i + step])
            xt[i:i + step].copy_(xp[i:i + step], non_blocking=True)
        out = t.empty(n_out, dtype=t.float64, device=self.dev)
        _lib.check(_lib.fns[name](self.handle, *scalars, xt.data_ptr(), out.data_ptr(), self.stream()))
        res = t.empty(n_out, dtype=t.float64, pin_memory=True)
        res.copy_(out, non_blocking=True)
        t.cuda.current_stream(self.dev).synchronize()
        return res.numpy()

    def spmv(self, which: int, x, n_in, n_out):
        return self.vec_op("pslr_spmv", x, n_in, n_out, int(which))


def _empty_csr(r, c):
    import scipy.sparse as sp
    return sp.csr_matrix((r, c))
