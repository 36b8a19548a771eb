"""Dev aid: block-sparse truncated SVD of a C4-scale two-site wavefunction (GPU vs oracle CPU)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import linalg, workloads as WL

torch.cuda.set_device(0)
u1 = tnb.Symmetry.u1()
V = tnb.Bond(btype=tnb.IN, sectors=WL.c4_sectors(), syms=[u1])
P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
psi = tnb.UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], name="psi", rowrank=2)
tnb.random.normal_(psi, seed=5)
print("blocks", psi.nblocks, "elements", sum(b.size for b in psi.get_blocks_()))
for driver in (None,):
    for _ in range(2):
        linalg.svd_truncate(psi, keepdim=1024)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        linalg.svd_truncate(psi, keepdim=1024)
    torch.cuda.synchronize()
    print("gpu svd_truncate ms", (time.perf_counter() - t0) / 3 * 1e3)
mz = linalg._Matricized(psi)
print("sectors", [(s.m, s.n) for s in mz.sectors])
torch.cuda.synchronize()
for m, n, members, off, view in mz.groups:
    t0 = time.perf_counter()
    torch.linalg.svd(view, full_matrices=False)
    torch.cuda.synchronize()
    print("group", m, n, len(members), "ms %.2f" % ((time.perf_counter() - t0) * 1e3))
mats = [view[k].cpu().numpy() for m, n, members, off, view in mz.groups for k in range(len(members))]
import tnkit_np as oracle
t0 = time.perf_counter()
oracle.svd_truncate_values(mats, 1024)
print("cpu oracle ms", (time.perf_counter() - t0) * 1e3)
