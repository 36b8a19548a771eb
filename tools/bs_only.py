"""Run only one block-sparse workload (dev probe for ncu captures): `single` (one C4 contract,
repeated) or `batch` (64 x C4 contract_batched, repeated)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch

import bench
import paper_2401_01921_b200 as tnb

torch.cuda.set_device(0)
what = sys.argv[1] if len(sys.argv) > 1 else "batch"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if what == "single":
    A, E = bench.c4_tensors(tnb)
    fn = lambda: tnb.contract(A, E)  # noqa: E731
else:
    pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
    fn = lambda: tnb.contract_batched(pairs)  # noqa: E731
for _ in range(n):
    fn()
torch.cuda.synchronize()
print("ok", what)
