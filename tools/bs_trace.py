"""Dev aid: per-CTA timeline of the grouped stream-K block-sparse GEMM (TNB_BS_TRACE)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = os.path.join(ROOT, "gpurun_out", "bs_trace.bin")
if len(sys.argv) > 1 and sys.argv[1] == "run":
    if os.path.exists(path):
        os.remove(path)
    os.environ["TNB_BS_TRACE"] = path
    import torch
    import bench
    import paper_2401_01921_b200 as tnb
    A, E = bench.c4_tensors(tnb)
    flush = bench.L2Flush() if "flush" in sys.argv else None
    from paper_2401_01921_b200 import _lib
    for i in range(5):
        if flush:
            flush()
        if i == 4:
            torch.cuda.synchronize()
            _lib.ktimer_reset()
            _lib.ktimer_enable(True)
        tnb.contract(A, E)
    torch.cuda.synchronize()
    _lib.ktimer_enable(False)
    print("event-timed bs kernel (count, ms, work)", _lib.ktimer_read(_lib.KF_BS_GEMM))
else:
    W = 64
    d = np.fromfile(path, dtype=np.int64).reshape(-1, 148, W)[-1]
    t0 = d[:, W - 1].min()
    print("kernel span us (first CTA entry -> last CTA end)", (d[:, 1].max() - t0) / 1e3,
          "entry spread us", (d[:, W - 1].max() - t0) / 1e3, "setup us (max over CTAs)", ((d[:, 0] - d[:, W - 1]).max()) / 1e3)
    order = np.argsort(d[:, 1])
    for c in list(order[:3]) + list(order[-8:]):
        r = d[c]
        segs = [(int(r[6 + 4 * k]), int(r[7 + 4 * k]), round((r[4 + 4 * k] - t0) / 1e3, 1), round((r[5 + 4 * k] - t0) / 1e3, 1))
                for k in range(min(int(r[2]), 14))]
        print(f"cta {c}: start {(r[0]-t0)/1e3:.1f} end {(r[1]-t0)/1e3:.1f} iters {r[3]} segs(tile,n,consumed,done) {segs}")
    if "stages" in sys.argv:
        for c in list(order[-3:]):
            r = d[c]
            st = [(r[30 + g] - t0) / 1e3 for g in range(24) if r[30 + g] > 0]
            print(f"cta {c} producer stage issue times (us):", " ".join(f"{x:.2f}" for x in st))
