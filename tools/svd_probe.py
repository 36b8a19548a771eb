"""Block SVD of the f3 workload (C4-bond two-site wavefunction): kernel time, sector shapes and
sweeps used (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import linalg

torch.cuda.set_device(0)
psi = bench.c4_two_site(tnb)
orig = tnb._lib.svd_jacobi_batched
seen = {}


def spy(jobs, stream, dtype):
    seen["jobs"] = jobs.copy()
    return orig(jobs, stream, dtype=dtype)


tnb._lib.svd_jacobi_batched = spy
linalg.svd_truncate(psi, keepdim=1024)
torch.cuda.synchronize()
tnb._lib.svd_jacobi_batched = orig
jobs = seen["jobs"]
shapes = sorted(((int(j["m"]), int(j["n"])) for j in jobs), reverse=True)
print("sectors", len(shapes), "largest", shapes[:6])
for _ in range(2):
    linalg.svd_truncate(psi, keepdim=1024)
torch.cuda.synchronize()
tnb._lib.ktimer_reset()
tnb._lib.ktimer_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    linalg.svd_truncate(psi, keepdim=1024)
e1.record()
torch.cuda.synchronize()
tnb._lib.ktimer_enable(False)
k, ms, _ = tnb._lib.ktimer_read(tnb._lib.KF_OTHER)
print(f"svd_truncate {e0.elapsed_time(e1) / 5:.2f} ms/call; jacobi kernel {ms / max(k, 1):.2f} ms/launch ({k} launches)")
