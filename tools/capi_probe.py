"""Dev aid: host cost of one tnb_contract_dense call (C1 step shapes), buffers preallocated."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2401_01921_b200 import _lib, dense

torch.cuda.set_device(0)
chi = 128
cases = {
    "A.L": ((chi, 2, chi), (chi, 5, chi), [0], [2]),
    "T1.W": ((2, chi, chi, 5), (5, 5, 2, 2), [0, 3], [3, 0]),
    "T2.R": ((chi, chi, 5, 2), (chi, 5, chi), [0, 2], [2, 1]),
}
L = _lib.lib()
st = dense.stream_handle()
for nm, (sa, sb, xa, xb) in cases.items():
    a = torch.randn(sa, dtype=torch.float64, device="cuda")
    b = torch.randn(sb, dtype=torch.float64, device="cuda")
    nout = a.numel() * b.numel()
    for x in xa:
        nout //= sa[x]
    for x in xb:
        nout //= sb[x]
    o = torch.empty(nout, dtype=torch.float64, device="cuda")
    arrs, (psa, ppa, psb, ppb, pxa, pxb) = _lib.dense_args(sa, list(range(len(sa))), sb, list(range(len(sb))), xa, xb)

    def call():
        return L.tnb_contract_dense(a.data_ptr(), _lib.TNB_F64, len(sa), psa, ppa, b.data_ptr(), _lib.TNB_F64, len(sb),
                                    psb, ppb, len(xa), pxa, pxb, o.data_ptr(), _lib.CPLX_4M, st)
    for _ in range(50):
        call()
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        call()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{nm}: host us per call {(t1 - t0) / n * 1e6:.2f}  (with drain {(t2 - t0) / n * 1e6:.2f})")
