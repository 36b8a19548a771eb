"""Per-permutation device timing (graph replay, L2 flushed) for the C2 sweep (dev aid)."""
import itertools, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2401_01921_b200 as tnb
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd_buf = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
for shape, dt in [((64,) * 4, np.float64), ((64,) * 4, np.complex128), ((16,) * 6, np.float64), ((16,) * 6, np.complex128)]:
    src = tnb.storage.uniform(list(shape), dtype=dt, seed=1)
    nbytes = 2 * src.size * src.itemsize
    perms = [p for p in itertools.permutations(range(len(shape)))][1:] if len(shape) == 4 else \
        [tuple(int(x) for x in np.random.default_rng(i).permutation(6)) for i in range(10)]
    res = []
    for p in perms:
        g = tnb.graphs.capture(lambda: src.permute(*p).contiguous(), warmup=1)
        ts = []
        for _ in range(5):
            flush_buf.zero_(); rd_buf.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res.append((p, nbytes / np.median(ts) / 1e6))
    print(shape, np.dtype(dt).name, "median", round(float(np.median([r for _, r in res]))), "min", round(min(r for _, r in res)))
    print("   ", " ".join(f"{''.join(map(str,p))}:{r:.0f}" for p, r in res))
