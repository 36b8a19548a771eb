"""Dev aid: complex128 L.A.W.R chi=1024 in 4M vs 3M (algorithmic 8 flop per complex MAC)."""
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
for mode in ("4M", "3M"):
    tnb.set_complex_mode(mode)
    r = bench.gpu_lawr(tnb, 1024, np.complex128, 6, 3, f, D(), e2e=False)
    print(mode, "launch TF %.2f" % (r["gflops"] / 1e3), "gemm TF", r["roofline"]["achieved"], r["steps_ms"])
