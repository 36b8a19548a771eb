"""Host-side cost of an eager C1 Network.launch (dev aid)."""
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
from paper_2401_01921_b200 import workloads as WL

torch.cuda.set_device(0)
net, _ = bench.make_network(tnb, WL.LAWR_NET, WL.lawr_inputs(128))
for _ in range(20):
    net.launch()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    net.launch()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per eager launch: {(t1 - t0) / 200 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    net.launch()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
