"""C3 c128 step gap (dev aid): device time per Network.launch vs its GEMM + narrow kernel time,
host time per call, and the caching allocator's cudaMalloc / free counters around the loop."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import workloads as WL

torch.cuda.set_device(0)
dt = np.complex128 if (len(sys.argv) < 2 or sys.argv[1] == "c128") else np.float64
net, _ = bench.make_network(tnb, WL.LAWR_NET, WL.lawr_inputs(1024, dtype=dt))
flush = bench.L2Flush()
for _ in range(3):
    net.launch()
torch.cuda.synchronize()
s0 = torch.cuda.memory_stats()
for trial in range(3):
    evs = []
    hts = []
    for _ in range(8):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        net.launch()
        hts.append(time.perf_counter() - t0)
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    print(f"trial {trial}: device ms/step {np.round(ms, 3).tolist()} host us/call {np.round(np.array(hts) * 1e6, 0).tolist()}")
s1 = torch.cuda.memory_stats()
for k in ("num_alloc_retries", "num_device_alloc", "num_device_free", "num_sync_all_streams"):
    print(k, s1.get(k, 0) - s0.get(k, 0))
