"""Graph replay time of one C4 contract (fast host path vs full path at capture) (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import contraction as C


def replay_ms(g, n=20):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


torch.cuda.set_device(0)
A, E = bench.c4_tensors(tnb)
for _ in range(3):
    tnb.contract(A, E)
g_fast = tnb.graphs.capture(lambda: tnb.contract(A, E))
print("graph (fast path captured) ms", replay_ms(g_fast))
orig = C._contract_blocks_fast
C._contract_blocks_fast = lambda a, b: None
g_full = tnb.graphs.capture(lambda: tnb.contract(A, E))
print("graph (full path captured) ms", replay_ms(g_full))
C._contract_blocks_fast = orig
print("graph (fast path captured) again ms", replay_ms(g_fast))

flush = bench.L2Flush()
dist = bench.Dist()
print("with flush: fast-captured", bench.time_steps(g_fast.replay, 10, flush, dist) / 10,
      "full-captured", bench.time_steps(g_full.replay, 10, flush, dist) / 10,
      "eager", bench.time_steps(lambda: tnb.contract(A, E), 10, flush, dist) / 10)
r = bench.gpu_c4(tnb, 10, 3, flush, dist)
print("gpu_c4:", {k: v for k, v in r.items() if k not in ("out_blocks", "roofline", "e2e")})
