"""Run only the chi=1024 float64 L.A.W.R Network launch n times (dev probe for ncu captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import workloads as WL

torch.cuda.set_device(0)
chi = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
net, _ = bench.make_network(tnb, WL.LAWR_NET, WL.lawr_inputs(chi, dtype=np.float64))
for _ in range(n):
    net.launch()
torch.cuda.synchronize()
print("ok", chi)
