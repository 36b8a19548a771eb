"""Per-permutation back-to-back permute rates (dev aid): K graph replays after one flush."""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb

torch.cuda.set_device(0)
flush, dist = bench.L2Flush(), bench.Dist()
hbm = bench.peaks()[0]
shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "64x64x64x64").split("x"))
dt = np.complex128 if (len(sys.argv) > 2 and sys.argv[2] == "c128") else np.float64
src = tnb.storage.uniform(list(shape), dtype=dt, seed=11)
if len(shape) == 4:
    perms = [p for p in itertools.permutations(range(4)) if p != (0, 1, 2, 3)]
else:
    g = np.random.default_rng(606)
    perms = []
    while len(perms) < 32:
        p = tuple(int(x) for x in g.permutation(len(shape)))
        if p != tuple(range(len(shape))):
            perms.append(p)
nbytes = 2 * src.size * src.itemsize
rates = []
for p in perms:
    g = tnb.graphs.capture(lambda: src.permute(*p).contiguous(), warmup=1)
    ms = bench.time_steps(lambda: [g.replay() for _ in range(8)], 1, flush, dist)
    rates.append(nbytes * 8 / ms / 1e6 / hbm)
    del g
tag = os.environ.get("TNB_T2D_T", "16")
print(f"T={tag} {shape} {np.dtype(dt).name}: median {np.median(rates):.3f} min {min(rates):.3f} max {max(rates):.3f}")
print("  " + " ".join(f"{''.join(map(str, p))}:{r:.2f}" for p, r in zip(perms, rates)))

# steady-state copy ceiling in the same harness: torch device-to-device copy of the same bytes
buf = src.storage()
dst = torch.empty_like(buf)
ms = bench.time_steps(lambda: [dst.copy_(buf) for _ in range(8)], 1, flush, dist)
print(f"  torch copy_ back-to-back: {nbytes * 8 / ms / 1e6 / hbm:.3f} of HBM peak")

# 1-byte elements (bool) take the generic tiled path
if os.environ.get("BOOL"):
    b = tnb.storage.DenseTensor(np.random.default_rng(1).integers(0, 2, size=shape).astype(np.bool_))
    rates = []
    for p in perms:
        g = tnb.graphs.capture(lambda: b.permute(*p).contiguous(), warmup=1)
        ms = bench.time_steps(lambda: [g.replay() for _ in range(8)], 1, flush, dist)
        rates.append(2 * b.size * 8 / ms / 1e6 / hbm)  # 8 replays x 2 x bytes
        del g
    print(f"  bool: median {np.median(rates):.3f} min {min(rates):.3f} of HBM")
