"""Dev aid: headline L.A.W.R chi=1024 f64 per-launch and GEMM-only timing."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import bench, paper_2401_01921_b200 as tnb
class D:
    world = 1; rank = 0
    def barrier(s): pass
    def max(s, x): return x
    def sum(s, x): return x
f = bench.L2Flush()
for _ in range(2):
    r = bench.gpu_lawr(tnb, 1024, np.float64, 10, 3, f, D(), e2e=False)
    print(os.environ.get("TNB_SK_BK", "16"), "launch TF %.2f" % (r["gflops"] / 1e3), "gemm TF", r["roofline"]["achieved"])
