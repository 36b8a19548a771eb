"""Block-sparse kernel timing under TNB_BS_EXP modes (dev aid): single C4 and 64 x C4,
kernel time from the library's kernel timer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch

import bench
import paper_2401_01921_b200 as tnb


def ktime(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tnb._lib.ktimer_reset()
    tnb._lib.ktimer_enable(True)
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    tnb._lib.ktimer_enable(False)
    k, ms, _ = tnb._lib.ktimer_read(tnb._lib.KF_BS_GEMM)
    return ms / max(k, 1)


torch.cuda.set_device(0)
A, E = bench.c4_tensors(tnb)
pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
t1 = ktime(lambda: tnb.contract(A, E))
tb = ktime(lambda: tnb.contract_batched(pairs), 5)
f = 2 * bench.C4_MACS
print(f"EXP={os.environ.get('TNB_BS_EXP', '0')} single {t1 * 1e3:.1f} us ({f / t1 / 1e9:.2f} TF)  "
      f"batch64 {tb:.3f} ms ({64 * f / tb / 1e9:.2f} TF)")
