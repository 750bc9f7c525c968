"""On-disk setup cache for build() (SURVEY §7 "setup cache", §8f rank 2).

Setup is host work outside the hot path (partition + reorder, ILUT, the device Arnoldi
that builds the correction), but it dominates repeated benchmark and sweep runs on big
grids (cfg5 at 8 GPUs partitions a 16.8M-vertex graph on every rank).  The cache stores,
per matrix + configuration, everything build() derives before the device context exists:

  setup  (key: matrix bytes, s, droptol, fill_cap, seed):
      the reordering (perm.forward, interior/interface sizes) and both assembled block
      factors (L, U, offsets, per-block nnz and pivot repairs);
  correction  (key: setup key + series degree m + rank):
      V, H, G and the achieved rank;
  packed  (key: setup key; pack_<key>.bin):
      the device context's packed format — per-block level schedules and the TMA-streamed
      factor chunks (csrc/pack.cpp), the host work of pslr_ctx_create.  The blob carries
      its own build / shared-memory-plan header; a stale one is re-packed, never used.

A hit rebuilds the PartitionedSystem by one symmetric permutation (no adjacency, no
BFS), skips ILUT and Arnoldi, and yields the same factors and correction bit for bit
(tests/test_setup_cache.py).  Files are plain .npz, written atomically (temp + rename),
so concurrent ranks sharing a directory are safe.  Enabled by build(..., cache_dir=...)
or PSLR_SETUP_CACHE=<dir>.
"""

from __future__ import annotations

import hashlib
import os
import tempfile

import numpy as np
import scipy.sparse as sp

from .ilu import BlockILU
from .partition import PartitionedSystem
from .sparse import Permutation, canonical, permute_symmetric

FORMAT = 1


def cache_dir(explicit=None):
    d = explicit if explicit is not None else os.environ.get("PSLR_SETUP_CACHE")
    return d or None


def matrix_digest(A) -> str:
    A = canonical(A)
    h = hashlib.sha256()
    h.update(np.asarray(A.shape, dtype=np.int64).tobytes())
    for arr, dt in ((A.indptr, np.int64), (A.indices, np.int32), (A.data, np.float64)):
        h.update(np.ascontiguousarray(arr, dtype=dt).tobytes())
    return h.hexdigest()


def setup_key(digest: str, cfg) -> str:
    return hashlib.sha256(f"v{FORMAT}|{digest}|s={cfg.num_subdomains}|dt={cfg.droptol!r}|"
                          f"fc={cfg.fill_cap}|seed={cfg.seed}".encode()).hexdigest()[:32]


def correction_key(skey: str, cfg) -> str:
    return hashlib.sha256(f"{skey}|m={cfg.series_degree}|r={cfg.rank}".encode()).hexdigest()[:32]


def _save(path, **arrays):
    d = os.path.dirname(path)
    os.makedirs(d, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=d, suffix=".tmp.npz")
    os.close(fd)
    np.savez(tmp, **arrays)
    os.replace(tmp, path)


def _csr_arrays(prefix, M):
    return {prefix + "_indptr": np.asarray(M.indptr, dtype=np.int64),
            prefix + "_indices": np.asarray(M.indices, dtype=np.int32),
            prefix + "_data": np.asarray(M.data, dtype=np.float64),
            prefix + "_shape": np.asarray(M.shape, dtype=np.int64)}


def _csr_load(d, prefix):
    return sp.csr_matrix((d[prefix + "_data"], d[prefix + "_indices"], d[prefix + "_indptr"]),
                         shape=tuple(int(x) for x in d[prefix + "_shape"]))


def _ilu_arrays(prefix, f: BlockILU):
    out = {prefix + "_offsets": np.asarray(f.offsets, dtype=np.int64)}
    out.update(_csr_arrays(prefix + "_L", f.L))
    out.update(_csr_arrays(prefix + "_U", f.U))
    if f.block_nnz is not None:
        out[prefix + "_block_nnz"] = np.asarray(f.block_nnz, dtype=np.int64)
    if f.block_repairs is not None:
        out[prefix + "_block_repairs"] = np.asarray(f.block_repairs, dtype=np.int64)
    return out


def _ilu_load(d, prefix) -> BlockILU:
    return BlockILU(offsets=d[prefix + "_offsets"], L=_csr_load(d, prefix + "_L"),
                    U=_csr_load(d, prefix + "_U"),
                    block_nnz=d[prefix + "_block_nnz"] if prefix + "_block_nnz" in d else None,
                    block_repairs=d[prefix + "_block_repairs"] if prefix + "_block_repairs" in d else None)


def save_setup(path, system: PartitionedSystem, b_ilu: BlockILU | None = None,
               c0_ilu: BlockILU | None = None) -> None:
    """The reordering, plus the block factors when given (the sharded path caches only the
    global reordering: each rank factors its own blocks)."""
    arrays = {"format": np.asarray([FORMAT]), "forward": system.perm.forward,
              "num_parts": np.asarray([system.num_parts]),
              "interior_sizes": system.interior_sizes, "interface_sizes": system.interface_sizes}
    if b_ilu is not None and c0_ilu is not None:
        arrays.update(_ilu_arrays("B", b_ilu))
        arrays.update(_ilu_arrays("C0", c0_ilu))
    _save(path, **arrays)


def load_setup(path, A, need_factors: bool = True):
    """(PartitionedSystem, b_ilu, c0_ilu) from a setup file, or None if absent/stale (or if
    need_factors and the file holds only the reordering; factors are None otherwise)."""
    if not path or not os.path.exists(path):
        return None
    with np.load(path) as d:
        if int(d["format"][0]) != FORMAT:
            return None
        has = "B_offsets" in d
        if need_factors and not has:
            return None
        perm = Permutation.from_forward(d["forward"])
        s = int(d["num_parts"][0])
        isz, fsz = d["interior_sizes"].astype(np.int64), d["interface_sizes"].astype(np.int64)
        b_ilu, c0_ilu = (_ilu_load(d, "B"), _ilu_load(d, "C0")) if has else (None, None)
    A = canonical(A)
    reordered = permute_symmetric(A, perm)
    p = int(isz.sum())
    q = A.shape[0] - p
    system = PartitionedSystem(
        matrix=reordered, perm=perm, num_parts=s, p=p, q=q, interior_sizes=isz, interface_sizes=fsz,
        B=canonical(reordered[:p, :p]) if p else sp.csr_matrix((0, 0)),
        E=canonical(reordered[:p, p:]) if p and q else sp.csr_matrix((p, q)),
        F=canonical(reordered[p:, :p]) if p and q else sp.csr_matrix((q, p)),
        C=canonical(reordered[p:, p:]) if q else sp.csr_matrix((0, 0)))
    return system, b_ilu, c0_ilu


def save_correction(path, V, H, G, r) -> None:
    _save(path, format=np.asarray([FORMAT]), V=np.ascontiguousarray(V, dtype=np.float64),
          H=np.asarray(H, dtype=np.float64), G=np.asarray(G, dtype=np.float64), rank=np.asarray([r]))


def load_correction(path):
    if not path or not os.path.exists(path):
        return None
    with np.load(path) as d:
        if int(d["format"][0]) != FORMAT:
            return None
        return d["V"], d["H"], d["G"], int(d["rank"][0])


def save_packed(path, blob: bytes) -> None:
    """The packed device format (pslr_ctx_create_packed's blob), written atomically."""
    if not path or not blob:
        return
    d = os.path.dirname(path)
    os.makedirs(d, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=d, suffix=".tmp.bin")
    with os.fdopen(fd, "wb") as fh:
        fh.write(blob)
    os.replace(tmp, path)


def load_packed(path):
    if not path or not os.path.exists(path):
        return None
    with open(path, "rb") as fh:
        return fh.read()
