"""Dev aid: host cost of the batched execute call itself, fresh vs after the permute sweep."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import contraction, dense

dist = bench.Dist()
flush = bench.L2Flush()
pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]


def probe(tag):
    outs = tnb.contract_batched(pairs)  # warm, plan cached
    plan = next(iter(contraction._BS_PLANS.values()))[0]
    aps = [dense.block_ptrs(a._blocks) for a, _ in pairs]
    bps = [dense.block_ptrs(b._blocks) for _, b in pairs]
    ops = [[x._p0 for x in o._blocks] for o in outs]
    torch.cuda.synchronize()
    ts, tf = [], []
    for i in range(6):
        t0 = time.perf_counter()
        flush()
        t1 = time.perf_counter()
        plan.execute_batched(aps, bps, ops, dense.stream_handle())
        t2 = time.perf_counter()
        tf.append((t1 - t0) * 1e3)
        ts.append((t2 - t1) * 1e3)
    torch.cuda.synchronize()
    print(tag, "flush enqueue ms", [round(t, 3) for t in tf], "execute_batched host ms", [round(t, 3) for t in ts])


probe("fresh")
bench.gpu_permute(tnb, 4, 3, flush, dist)
probe("after permute")
