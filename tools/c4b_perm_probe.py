"""Dev aid: C4 batch leg after the permute sweep (allocator state), with/without empty_cache."""
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
bench.gpu_permute(tnb, 4, 3, flush, dist)
r = bench.gpu_c4_batch(tnb, 64, 5, 3, flush, dist)
print("after permute", round(r["ms_per_step"], 3), round(r["ms_per_step_pairwise"], 3))
print(torch.cuda.memory_stats()["num_alloc_retries"], torch.cuda.memory_reserved() / 1e9, "GB reserved")
torch.cuda.empty_cache()
r = bench.gpu_c4_batch(tnb, 64, 5, 3, flush, dist)
print("after empty_cache", round(r["ms_per_step"], 3), round(r["ms_per_step_pairwise"], 3))

# bad state again (permute sweep), then profile one batched step
bench.gpu_permute(tnb, 4, 3, flush, dist)
import cProfile, pstats, time
pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
tnb.contract_batched(pairs)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    tnb.contract_batched(pairs)
torch.cuda.synchronize()
print("bad state wall ms per batch", (time.perf_counter() - t0) / 5 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    tnb.contract_batched(pairs)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
