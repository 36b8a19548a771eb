"""Lanczos step kernels: per-iteration vector-work time at chi=1024 (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib, dense, eig

torch.cuda.set_device(0)
n, m = 2 * 1024 * 1024, 31
ds = eig._DeviceSteps(n, m, "float64", "cuda")
ds.Qt.normal_()
w = torch.randn(n, dtype=torch.float64, device="cuda")
for r in (1, 10, 30):
    for _ in range(2):
        ds.step(r, w.clone(), r, slot=0)
    torch.cuda.synchronize()
    _lib.ktimer_reset()
    _lib.ktimer_enable(True)
    for _ in range(10):
        ds.step(r, w.clone(), r, slot=0)
    torch.cuda.synchronize()
    _lib.ktimer_enable(False)
    k, ms, work = _lib.ktimer_read(_lib.KF_OTHER)
    print(f"r={r}: {ms / 10 * 1e3:.1f} us per step, {work / (ms / 1e3) / 1e9:.0f} GB/s")
