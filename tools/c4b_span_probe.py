"""Dev aid: where the device span of a batched C4 step goes (fresh vs after the permute sweep)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib

dist = bench.Dist()
flush = bench.L2Flush()
pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
orig = _lib.BsPlan.execute_batched
marks = []


def wrapped(self, *a, **k):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    t = time.perf_counter()
    r = orig(self, *a, **k)
    e2 = torch.cuda.Event(enable_timing=True)
    e2.record()
    marks.append((e, e2, time.perf_counter() - t))
    return r


_lib.BsPlan.execute_batched = wrapped


def probe(tag):
    for _ in range(3):
        tnb.contract_batched(pairs)
    torch.cuda.synchronize()
    rows = []
    for i in range(5):
        marks.clear()
        flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        tnb.contract_batched(pairs)
        h1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        a, b, hx = marks[0]
        rows.append((round(e0.elapsed_time(e1), 3), round(e0.elapsed_time(a), 3), round(a.elapsed_time(b), 3),
                     round((h1 - h0) * 1e3, 3)))
    print(tag, "(span, e0->exec, exec, host ms)", rows)


probe("fresh")
bench.gpu_permute(tnb, 4, 3, flush, dist)
probe("after permute")
