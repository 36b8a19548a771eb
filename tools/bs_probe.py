"""Dev aid: block-sparse plan creation cost (pairing kernel) vs cached calls."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib

torch.cuda.set_device(0)
A, E = bench.c4_tensors(tnb)
tnb.contract(A, E)  # warm CUDA context, kernels
torch.cuda.synchronize()
for trial in range(3):
    # a new structure each trial: drop one sector's degeneracy by one
    import numpy as np
    sec = bench.WL.c4_sectors()
    sec = [(q, d + (1 if q == trial else 0)) for q, d in sec]
    u1 = tnb.Symmetry.u1()
    V = tnb.Bond(btype=tnb.IN, sectors=sec, syms=[u1])
    P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    A2 = tnb.UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
    E2 = tnb.UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
    torch.cuda.synchronize()
    _lib.ktimer_reset()
    _lib.ktimer_enable(True)
    t0 = time.perf_counter()
    tnb.contract(A2, E2)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tnb.contract(A2, E2)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    _lib.ktimer_enable(False)
    print("first call wall ms %.3f, cached call wall ms %.3f" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3),
          "pair kernel", _lib.ktimer_read(_lib.KF_BS_PAIR), "gemm", _lib.ktimer_read(_lib.KF_BS_GEMM))
