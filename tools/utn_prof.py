"""Dev aid: cProfile of load_unitensor (C4 A tensor)."""
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

A, _ = bench.c4_tensors(tnb)
path = "/tmp/utn_prof.utn"
tnb.save_unitensor(A, path)
for _ in range(5):
    tnb.load_unitensor(path)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    tnb.load_unitensor(path)
torch.cuda.synchronize()
print("ms per load", (time.perf_counter() - t0) / 50 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    tnb.load_unitensor(path)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
