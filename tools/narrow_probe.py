"""Dev aid: kernel time of the T1.W (narrow) step at chi=1024."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib

torch.cuda.set_device(0)
chi = 1024
rng = np.random.default_rng(0)
T1 = tnb.UniTensor(tnb.storage.from_numpy(rng.standard_normal((2, chi, chi, 5))), labels=["p", "vr", "b", "w"])
W = tnb.UniTensor(tnb.storage.from_numpy(rng.standard_normal((5, 5, 2, 2))), labels=["w", "w2", "q", "p"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    tnb.contract(T1, W)
torch.cuda.synchronize()
_lib.ktimer_reset()
_lib.ktimer_enable(True)
for _ in range(20):
    flush.zero_()
    tnb.contract(T1, W)
torch.cuda.synchronize()
_lib.ktimer_enable(False)
n, ms, _ = _lib.ktimer_read(_lib.KF_GEMM_SKINNY)
us = ms / n * 1e3
print(f"T1.W narrow: {us:.1f} us per launch, {2 * 84e6 / (us * 1e-6) / 1e9:.0f} GB/s (168 MB algorithmic)")
