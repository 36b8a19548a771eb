"""Dev aid: cuSOLVER SVD drivers and multi-stream concurrency on the C4 two-site sectors."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

torch.cuda.set_device(0)
sizes = [9, 1, 21, 3, 45, 86, 149, 233, 330, 423, 490, 516, 490, 423, 330, 233, 149, 86, 45, 21, 9, 3, 1]
g = torch.Generator(device="cuda").manual_seed(0)
mats = [torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) for n in sizes]
for driver in ("gesvd", "gesvdj", None):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for m in mats:
            torch.linalg.svd(m, full_matrices=False, driver=driver)
        torch.cuda.synchronize()
    print("sequential", driver, "ms %.1f" % ((time.perf_counter() - t0) * 1e3))
    streams = [torch.cuda.Stream() for _ in range(8)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        order = sorted(range(len(mats)), key=lambda i: -sizes[i])
        for k, i in enumerate(order):
            s = streams[k % len(streams)]
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                torch.linalg.svd(mats[i], full_matrices=False, driver=driver)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
    print("8 streams", driver, "ms %.1f" % ((time.perf_counter() - t0) * 1e3))
# eigh route timing for reference
torch.cuda.synchronize()
t0 = time.perf_counter()
for m in mats:
    torch.linalg.eigh(m.T @ m)
torch.cuda.synchronize()
print("eigh(A^T A) sequential ms %.1f" % ((time.perf_counter() - t0) * 1e3))
