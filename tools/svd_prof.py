"""Dev aid: host/device split of svd_truncate on the C4 two-site tensor."""
import cProfile, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib, linalg, workloads as WL
torch.cuda.set_device(0)
u1 = tnb.Symmetry.u1()
V = tnb.Bond(btype=tnb.IN, sectors=WL.c4_sectors(), syms=[u1])
P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
psi = tnb.UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], name="psi", rowrank=2)
tnb.random.normal_(psi, seed=5)
linalg.svd_truncate(psi, keepdim=1024)
torch.cuda.synchronize()
_lib.ktimer_reset(); _lib.ktimer_enable(True)
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
linalg.svd_truncate(psi, keepdim=1024)
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) * 1e3)
pr.disable(); _lib.ktimer_enable(False)
print("jacobi", _lib.ktimer_read(_lib.KF_OTHER))
pstats.Stats(pr).sort_stats("cumtime").print_stats(18)
