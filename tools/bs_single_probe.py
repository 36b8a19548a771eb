"""Single C4 contraction kernel time from a flushed L2 (as the bench times it) (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch

import bench
import paper_2401_01921_b200 as tnb

torch.cuda.set_device(0)
A, E = bench.c4_tensors(tnb)
flush, dist = bench.L2Flush(), bench.Dist()
for _ in range(3):
    tnb.contract(A, E)
(n, ms, _), = bench.ktimer(tnb, lambda: bench.time_steps(lambda: tnb.contract(A, E), 20, flush, dist), tnb._lib.KF_BS_GEMM)
g = tnb.graphs.capture(lambda: tnb.contract(A, E))
gms = bench.time_steps(g.replay, 20, flush, dist) / 20
tag = os.environ.get("TNB_BS_EXP", "0")
print(f"[exp={tag}] single C4 kernel {ms / n * 1e3:.1f} us (flushed L2), graph replay {gms * 1e3:.1f} us")
