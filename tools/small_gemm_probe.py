"""Dev aid: kernel time of the C1 (chi=128) contraction steps (ktimer), for dispatch sweeps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib

torch.cuda.set_device(0)
chi = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rng = np.random.default_rng(0)


def ut(shape, labels):
    return tnb.UniTensor(tnb.storage.from_numpy(rng.standard_normal(shape)), labels=labels)


def kern_us(fn, fam, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    _lib.ktimer_reset()
    _lib.ktimer_enable(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    _lib.ktimer_enable(False)
    n, ms, _ = _lib.ktimer_read(fam)
    return ms / max(n, 1) * 1e3


A = ut((chi, 2, chi), ["vl", "p", "vr"])
L = ut((chi, 5, chi), ["b", "w", "vl"])
T2 = ut((chi, chi, 5, 2), ["vr", "b", "w2", "q"])
R = ut((chi, 5, chi), ["b2", "w2", "vr"])
print(f"A.L us {kern_us(lambda: tnb.contract(A, L), _lib.KF_GEMM):.2f}  "
      f"T2.R us {kern_us(lambda: tnb.contract(T2, R), _lib.KF_GEMM):.2f}")
