"""Dev aid: per-round cost of the Jacobi SVD kernel (orthogonal input = no rotations)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2401_01921_b200 import _lib
torch.cuda.set_device(0)
for name, mk in [("identity", lambda n: torch.eye(n, dtype=torch.float64, device="cuda")),
                 ("random", lambda n: torch.randn(n, n, dtype=torch.float64, device="cuda"))]:
    for n in (64, 256, 516):
        a = mk(n)
        bufs = [torch.empty_like(a) for _ in range(4)]
        s = torch.empty(n, dtype=torch.float64, device="cuda"); st = torch.zeros(1, dtype=torch.int32, device="cuda")
        job = (a.data_ptr(), bufs[0].data_ptr(), bufs[1].data_ptr(), bufs[2].data_ptr(), s.data_ptr(), bufs[3].data_ptr(),
               st.data_ptr(), n, n)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.svd_jacobi_batched(np.array([job], dtype=_lib.SVD_SECTOR_DTYPE), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        sw = int(st.item())
        print(name, n, "ms %.2f" % (dt * 1e3), "sweeps", sw, "us/round %.2f" % (dt * 1e6 / max(1, abs(sw)) / (n - 1 + (n & 1))))
