"""Dev aid: f64 and c128 C4 two-site svd_truncate, engine vs oracle CPU."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import linalg, workloads as WL
import tnkit_np as oracle
torch.cuda.set_device(0)
u1 = tnb.Symmetry.u1()
V = tnb.Bond(btype=tnb.IN, sectors=WL.c4_sectors(), syms=[u1])
P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
for dt in (np.float64, np.complex128):
    psi = tnb.UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], name="psi", rowrank=2, dtype=dt)
    tnb.random.normal_(psi, seed=5)
    for _ in range(2):
        linalg.svd_truncate(psi, keepdim=1024)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    linalg.svd_truncate(psi, keepdim=1024)
    torch.cuda.synchronize()
    g = (time.perf_counter() - t0) * 1e3
    mz = linalg._Matricized(psi)
    mats = [v[k].cpu().numpy() for m, n, mem, off, v in mz.groups for k in range(len(mem))]
    t0 = time.perf_counter()
    oracle.svd_truncate_values(mats, 1024)
    c = (time.perf_counter() - t0) * 1e3
    print(np.dtype(dt).name, "gpu ms %.1f" % g, "cpu ms %.1f" % c)
