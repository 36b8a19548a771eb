"""Dev aid: the C4 batch-64 leg of bench.py (batched vs pairwise)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench
import paper_2401_01921_b200 as tnb

r = bench.gpu_c4_batch(tnb, 64, 5, 3, bench.L2Flush(), bench.Dist())
print(r)
