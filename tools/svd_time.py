"""Dev aid: the bench's SVD leg (ms per svd_truncate on the C4 two-site tensor)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench
import paper_2401_01921_b200 as tnb

r = bench.gpu_svd(tnb, 3, 1, bench.L2Flush(), bench.Dist())
print("svd ms", round(r["ms_per_call"], 3))
