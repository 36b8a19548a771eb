"""Dev aid: per-step device times of the batched C4 leg (time_steps without the sum)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch

import bench
import paper_2401_01921_b200 as tnb

dist = bench.Dist()
flush = bench.L2Flush()
pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]


def steps(tag):
    for _ in range(3):
        tnb.contract_batched(pairs)
    torch.cuda.synchronize()
    ev = []
    for _ in range(6):
        flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        tnb.contract_batched(pairs)
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    print(tag, [round(a.elapsed_time(b), 3) for a, b in ev], "reserved GB", round(torch.cuda.memory_reserved() / 1e9, 2))


steps("fresh")
bench.gpu_permute(tnb, 4, 3, flush, dist)
steps("after permute (old pairs)")
pairs[:] = [bench.c4_tensors(tnb, seed=5777 + 2 * i) for i in range(64)]
steps("after permute (new pairs)")
import time
t0 = time.perf_counter()
for _ in range(5):
    tnb.contract_batched(pairs)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host ms per batched call (new pairs)", (t1 - t0) / 5 * 1e3)
