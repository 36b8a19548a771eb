"""Dev aid: Jacobi SVD kernel statuses / sweeps / kernel time on the C4 two-site sectors."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib, linalg, workloads as WL

torch.cuda.set_device(0)
u1 = tnb.Symmetry.u1()
V = tnb.Bond(btype=tnb.IN, sectors=WL.c4_sectors(), syms=[u1])
P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
psi = tnb.UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], name="psi", rowrank=2)
tnb.random.normal_(psi, seed=5)
orig = linalg._library_svd
calls = []
linalg._library_svd = lambda v: (calls.append(tuple(v.shape)), orig(v))[1]
mz = linalg._Matricized(psi)
torch.cuda.synchronize()
_lib.ktimer_reset()
_lib.ktimer_enable(True)
t0 = time.perf_counter()
facs = linalg._factorise(mz)
torch.cuda.synchronize()
print("factorise ms", (time.perf_counter() - t0) * 1e3, "jacobi kernel", _lib.ktimer_read(_lib.KF_OTHER))
_lib.ktimer_enable(False)
print("library fallbacks", calls)
for tol in (2.0, 8.0, 32.0):
    for sweeps in (30,):
        jobs = []
        a = torch.randn(516, 516, dtype=torch.float64, device="cuda")
        q = torch.empty_like(a); u = torch.empty_like(a); vh = torch.empty_like(a); w = torch.empty_like(a)
        s = torch.empty(516, dtype=torch.float64, device="cuda"); st = torch.zeros(1, dtype=torch.int32, device="cuda")
        jobs.append((a.data_ptr(), w.data_ptr(), q.data_ptr(), u.data_ptr(), s.data_ptr(), vh.data_ptr(), st.data_ptr(), 516, 516))
        ref = torch.linalg.svdvals(a.clone())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.svd_jacobi_batched(np.array(jobs, dtype=_lib.SVD_SECTOR_DTYPE), torch.cuda.current_stream().cuda_stream,
                                max_sweeps=sweeps, tol=tol)
        torch.cuda.synchronize()
        print("516 alone tol", tol, "ms %.2f" % ((time.perf_counter() - t0) * 1e3), "status", int(st.item()),
              "max rel err sv", float((s - ref).abs().max() / ref.max()))
