"""Dev aid: C4 block-sparse kernel time (ktimer) + the bench's C4 leg."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench
import paper_2401_01921_b200 as tnb


flush = bench.L2Flush()
for _ in range(2):
    r = bench.gpu_c4(tnb, 20, 3, flush, bench.Dist())
    print({k: v for k, v in r.items() if k != "cpu_baseline"})
