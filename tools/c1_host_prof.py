"""cProfile of the host side of an eager C1 Network.launch (dev aid)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import workloads as WL

inp = WL.lawr_inputs(128, dtype=np.float64, seed=1)
net, _ = bench.lawr_network(tnb, inp)
for _ in range(20):
    net.launch()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    net.launch()
torch.cuda.synchronize()
print("wall per launch us", (time.perf_counter() - t0) / 200 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    net.launch()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
