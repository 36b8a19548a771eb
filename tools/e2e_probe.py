"""Dev aid: host<->HBM bandwidth and the L.A.W.R e2e step timeline (uploads overlap)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb

torch.cuda.set_device(0)
x = torch.empty(100 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(100 << 20, dtype=torch.uint8, device="cuda")
for d in ("h2d", "d2h"):
    for _ in range(3):
        y.copy_(x, non_blocking=True) if d == "h2d" else x.copy_(y, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y.copy_(x, non_blocking=True) if d == "h2d" else x.copy_(y, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(d, "GB/s", 10 * x.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9)


class D:
    world = 1
    rank = 0

    def barrier(self):
        pass

    def max(self, v):
        return v

    def sum(self, v):
        return v


r = bench.gpu_lawr(tnb, 1024, np.float64, 10, 3, bench.L2Flush(), D(), e2e=True, roof=False)
print("device ms", r["ms_per_step"], "e2e", r["e2e"])
