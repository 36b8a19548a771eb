"""Dev aid: GEMM time of L.A.W.R column panels (chunked e2e path) vs the full steps."""
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


def ut(shape, labels):
    return tnb.UniTensor(tnb.storage.from_numpy(rng.standard_normal(shape)), labels=labels)


def gemm_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    _lib.ktimer_reset()
    _lib.ktimer_enable(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    _lib.ktimer_enable(False)
    n, ms, fl = _lib.ktimer_read(_lib.KF_GEMM)
    return ms / reps, fl / (ms / 1e3) / 1e12 if ms else 0


A = ut((chi, 2, chi), ["vl", "p", "vr"])
for nb in (chi, chi // 2, chi // 4, chi // 8):
    L = ut((nb, 5, chi), ["b", "w", "vl"])
    print("A.L  b=%4d  ms %.4f  TF %.2f" % ((nb,) + gemm_ms(lambda: tnb.contract(A, L))))
T2 = ut((chi, chi, 5, 2), ["vr", "b", "w2", "q"])
for nb in (chi, chi // 2, chi // 4, chi // 8):
    R = ut((nb, 5, chi), ["b2", "w2", "vr"])
    print("T2.R b2=%4d ms %.4f  TF %.2f" % ((nb,) + gemm_ms(lambda: tnb.contract(T2, R))))
