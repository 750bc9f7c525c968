import os, sys, time, json
sys.path.insert(0, os.getcwd())
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29544", RANK="0", WORLD_SIZE="1")
import numpy as np, torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_2002_00917_b200 import shard, workloads
from paper_2002_00917_b200.partition import classify_and_reorder, partition_graph
import paper_2002_00917_b200 as pg
base = workloads.CONFIGS["cfg5"]
A = workloads.laplacian3d(*base.grid, base.shift)
ps = classify_and_reorder(A, partition_graph(A, base.s, seed=0))
P = shard.build_sharded(ps, pg.PslrConfig(num_subdomains=base.s, series_degree=base.m, rank=base.rank))
n = P.ops.n
b = torch.randn(n, dtype=torch.float64, device="cuda")
bh = b.cpu().pin_memory(); zh = torch.empty(n, dtype=torch.float64).pin_memory()
def t(fn, k=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/k
print("apply", t(lambda: P.apply(b)))
print("h2d", t(lambda: bh.to("cuda", non_blocking=True)))
print("d2h", t(lambda: zh.copy_(b, non_blocking=True)))
print("all", t(lambda: zh.copy_(P.apply(bh.to("cuda", non_blocking=True)), non_blocking=True)))
print("pinned?", bh.is_pinned(), zh.is_pinned())
dist.destroy_process_group()
