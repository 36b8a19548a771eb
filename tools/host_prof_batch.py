"""cProfile of the host side of contract_batched (64 x C4) and of one contract (dev aid)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch

import bench
import paper_2401_01921_b200 as tnb

torch.cuda.set_device(0)
pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
for _ in range(3):
    tnb.contract_batched(pairs)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    tnb.contract_batched(pairs)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per contract_batched call: {(t1 - t0) / 10 * 1e3:.3f} ms")
A, E = pairs[0]
t0 = time.perf_counter()
for _ in range(100):
    tnb.contract(A, E)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per contract call: {(t1 - t0) / 100 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    tnb.contract_batched(pairs)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
