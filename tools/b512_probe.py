import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import bench, paper_2401_01921_b200 as tnb, numpy as np, torch
class D:
    world=1; rank=0
    def barrier(s): pass
    def max(s,x): return x
    def sum(s,x): return x
f=bench.L2Flush()
for _ in range(3):
    print(bench.gpu_lawr_batch(tnb, 64, 512, np.complex128, 3, 1, f, D()))
r = bench.gpu_lawr(tnb, 512, np.complex128, 10, 3, f, D(), e2e=False)
print(r["gflops"], r["steps_ms"], r["roofline"]["achieved"])
