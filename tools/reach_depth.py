"""Dependency depth of the cfg5 B blocks: L and U levels, the joint L+U DAG, and the depths
restricted to the Horner B solve (rhs E y non-zero only at E rows, output read by F only at
F columns): L reach and U closure.  CPU only (native setup).  usage: python tools/reach_depth.py"""
import sys, numpy as np, scipy.sparse as sp
sys.path.insert(0, '/root/repo')
from paper_2002_00917_b200 import workloads
from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph
from paper_2002_00917_b200.ilu import factor_blocks
A = workloads.laplacian3d(128,128,128, 0.5)
spec = partition_graph(A, 32, seed=0)
ps = classify_and_reorder(A, spec)
bi = factor_blocks(ps.B, ps.interior_sizes, droptol=1e-2)
def depths(L, U):
    n = L.shape[0]
    Lc = L.tocsr(); Uc = U.tocsr()
    lvL = np.zeros(n, np.int64)
    ip, ix = Lc.indptr, Lc.indices
    for i in range(n):
        m = 0
        for j in ix[ip[i]:ip[i+1]]:
            if j < i and lvL[j] + 1 > m: m = lvL[j] + 1
        lvL[i] = m
    lvU = np.zeros(n, np.int64); lvC = np.zeros(n, np.int64)
    ip, ix = Uc.indptr, Uc.indices
    for i in range(n-1, -1, -1):
        m = 0; mc = lvL[i] + 1
        for j in ix[ip[i]:ip[i+1]]:
            if j > i:
                if lvU[j] + 1 > m: m = lvU[j] + 1
                if lvC[j] + 1 > mc: mc = lvC[j] + 1
        lvU[i] = m; lvC[i] = mc
    return lvL.max()+1, lvU.max()+1, lvC.max()+1
blocks = bi.blocks() if hasattr(bi,'blocks') else None
off = bi.offsets
res=[]
for b in range(len(off)-1):
    lo, hi = int(off[b]), int(off[b+1])
    dL, dU, dC = depths(bi.L[lo:hi, lo:hi], bi.U[lo:hi, lo:hi])
    res.append((dL+dU, dL, dU, dC, b))
res.sort(reverse=True)
for r in res[:8]: print("block %d: L %d U %d sum %d combined %d" % (r[4], r[1], r[2], r[0], r[3]))

print("---- restricted (Horner: rhs = E y, output read by F)")
E = ps.E.tocsr(); F = ps.F.tocsc()
erow = np.diff(E.indptr) > 0
fcol = np.diff(F.indptr) > 0
def restricted(L, U, src, dst):
    n = L.shape[0]
    Lc = L.tocsr(); Uc = U.tocsr()
    inR = src.copy(); lv = np.full(n, -1, np.int64)
    ip, ix = Lc.indptr, Lc.indices
    for i in range(n):
        m = 0 if src[i] else -1
        for j in ix[ip[i]:ip[i+1]]:
            if j < i and lv[j] >= 0 and lv[j] + 1 > m: m = lv[j] + 1
        lv[i] = m
    reach = lv >= 0
    # U closure backward from dst
    need = dst.copy()
    ip, ix = Uc.indptr, Uc.indices
    for i in range(n):  # closure: i needed -> all its deps j>i needed; process ascending
        if need[i]:
            for j in ix[ip[i]:ip[i+1]]:
                if j > i: need[j] = True
    lu = np.full(n, -1, np.int64)
    for i in range(n-1, -1, -1):
        if not need[i]: continue
        m = 0
        for j in ix[ip[i]:ip[i+1]]:
            if j > i and lu[j] + 1 > m: m = lu[j] + 1
        lu[i] = m
    return reach.sum(), lv.max()+1, need.sum(), lu.max()+1, n
for r in res[:6]:
    b = r[4]; lo, hi = int(off[b]), int(off[b+1])
    rs, dl, ns, du, n = restricted(bi.L[lo:hi, lo:hi], bi.U[lo:hi, lo:hi], erow[lo:hi], fcol[lo:hi])
    print("block %d n %d: E-rows %d, L reach %d depth %d (full %d); F-cols %d, U closure %d depth %d (full %d)" % (b, n, erow[lo:hi].sum(), rs, dl, r[1], fcol[lo:hi].sum(), ns, du, r[2]))
