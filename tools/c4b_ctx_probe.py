"""Dev aid: the C4 batch leg after the bench's earlier workloads (allocator / heap state)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb

dist = bench.Dist()
flush = bench.L2Flush()
print("fresh", {k: round(v, 3) for k, v in bench.gpu_c4_batch(tnb, 64, 5, 3, flush, dist).items() if isinstance(v, float)})
if "head" in sys.argv:
    bench.gpu_lawr(tnb, 1024, np.float64, 10, 3, flush, dist)
    print("after headline", {k: round(v, 3) for k, v in bench.gpu_c4_batch(tnb, 64, 5, 3, flush, dist).items()
                             if isinstance(v, float)})
if "ctx" in sys.argv:
    bench.gpu_lawr(tnb, 1024, np.complex128, 3, 3, flush, dist, e2e=False)
    bench.gpu_lawr(tnb, 128, np.float64, 10, 3, flush, dist, e2e=False, roof=False, graph=True)
    bench.gpu_permute(tnb, 4, 3, flush, dist)
    bench.gpu_c4(tnb, 10, 3, flush, dist)
    print("after ctx", {k: round(v, 3) for k, v in bench.gpu_c4_batch(tnb, 64, 5, 3, flush, dist).items() if isinstance(v, float)})
    import cProfile, pstats
    pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
    tnb.contract_batched(pairs)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        flush()
        tnb.contract_batched(pairs)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
