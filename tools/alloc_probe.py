"""Dev aid: torch allocator cost for a 180 MB block after many graph captures (permute sweep)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch

import bench
import paper_2401_01921_b200 as tnb

dist = bench.Dist()
flush = bench.L2Flush()


def probe(tag):
    n = 180 << 20
    ts = []
    for i in range(8):
        flush()
        t0 = time.perf_counter()
        x = torch.empty(n, dtype=torch.uint8, device="cuda")
        t1 = time.perf_counter()
        del x
        ts.append((t1 - t0) * 1e3)
    torch.cuda.synchronize()
    print(tag, "alloc ms", [round(t, 3) for t in ts])


probe("fresh")
bench.gpu_permute(tnb, 4, 3, flush, dist)
probe("after permute")
st = torch.cuda.memory_stats()
print({k: v for k, v in st.items() if "segment" in k and "all" in k and "current" in k})
