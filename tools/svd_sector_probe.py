"""One-sector Jacobi timing: kernel ms and sweeps for an m x n float64 N(0,1) matrix (dev aid).
Usage: svd_sector_probe.py m n [count]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np
import torch

from paper_2401_01921_b200 import _lib

torch.cuda.set_device(0)
m, n = int(sys.argv[1]), int(sys.argv[2])
cnt = int(sys.argv[3]) if len(sys.argv) > 3 else 1
dev = "cuda"
g = torch.Generator(device="cpu").manual_seed(1)
bufs = []
jobs = []
for k in range(cnt):
    a = torch.randn(m, n, generator=g, dtype=torch.float64).to(dev)
    lw, lq = n + (n & 1), m + (m & 1)
    b = torch.empty(m, lw, dtype=torch.float64, device=dev)
    q = torch.empty(m, lq, dtype=torch.float64, device=dev)
    u = torch.empty(m, m, dtype=torch.float64, device=dev)
    s = torch.empty(m, dtype=torch.float64, device=dev)
    vh = torch.empty(m, n, dtype=torch.float64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    bufs.append((a, b, q, u, s, vh, st))
    jobs.append((a.data_ptr(), b.data_ptr(), q.data_ptr(), u.data_ptr(), s.data_ptr(), vh.data_ptr(), st.data_ptr(), m, n))
jobs = np.array(jobs, dtype=_lib.SVD_SECTOR_DTYPE)
stream = torch.cuda.current_stream().cuda_stream
_lib.svd_jacobi_batched(jobs, stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_lib.svd_jacobi_batched(jobs, stream)
e1.record()
torch.cuda.synchronize()
a, b, q, u, s, vh, st = bufs[0]
sw = int(st.item())
ref = torch.linalg.svdvals(a)
err = (s - ref).abs().max().item() / ref.max().item()
rounds = sw * (m + (m & 1) - 1)
print(f"m={m} n={n} x{cnt}: {e0.elapsed_time(e1):.2f} ms, sweeps {sw}, {e0.elapsed_time(e1) * 1e3 / max(rounds, 1):.2f} us/round, "
      f"sigma rel err {err:.1e}")
