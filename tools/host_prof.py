"""cProfile of the host side of a block-sparse contract (dev aid)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import workloads as WL

u1 = tnb.Symmetry.u1()
V = tnb.Bond(btype=tnb.IN, sectors=WL.c4_sectors(), syms=[u1])
P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
A = tnb.UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
E = tnb.UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
tnb.random.normal_(A, seed=1)
tnb.random.normal_(E, seed=2)
for _ in range(10):
    tnb.contract(A, E)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    tnb.contract(A, E)
torch.cuda.synchronize()
print("wall per call us", (time.perf_counter() - t0) * 1e4)
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    tnb.contract(A, E)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
