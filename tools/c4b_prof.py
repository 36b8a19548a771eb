"""Dev aid: cProfile of contract_batched over 64 C4 pairs."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
import paper_2401_01921_b200 as tnb

pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
for _ in range(3):
    tnb.contract_batched(pairs)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    tnb.contract_batched(pairs)
torch.cuda.synchronize()
print("ms per batch", (time.perf_counter() - t0) / 10 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    tnb.contract_batched(pairs)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
