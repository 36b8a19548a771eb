"""Dev aid: bench.gpu_c4_batch after the permute sweep, with per-step event times."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch

import bench
import paper_2401_01921_b200 as tnb

dist = bench.Dist()
flush = bench.L2Flush()
orig = bench.time_steps


def ts(fn, steps, fl, d):
    pairs = []
    torch.cuda.synchronize()
    for _ in range(steps):
        fl()
        e0, e1 = bench._events()
        e0.record()
        fn()
        e1.record()
        pairs.append((e0, e1))
    torch.cuda.synchronize()
    t = [round(a.elapsed_time(b), 3) for a, b in pairs]
    print("  steps", getattr(fn, "__name__", "?"), t)
    return sum(t)


bench.time_steps = ts
bench.gpu_permute(tnb, 4, 3, flush, dist)
print({k: v for k, v in bench.gpu_c4_batch(tnb, 64, 5, 3, flush, dist).items() if "ms" in k})
