"""Dev aid: per-step kernel timing of one C5 PEPS site launch (kernel timer families)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib, workloads as WL

torch.cuda.set_device(0)
shapes = WL.peps_shapes(256, 8, 2)
net = tnb.Network(WL.PEPS_NET)
for k, (nm, shp) in enumerate(shapes.items()):
    t = tnb.UniTensor(tnb.storage.from_numpy(tnb.storage.host_normal(shp, seed=9000 + k)),
                      labels=[f"x{j}" for j in range(len(shp))])
    net.put_tensor(nm, t)
net.set_order(optimal=True)
net.launch()
torch.cuda.synchronize()
# time each pairwise step: monkeypatch contract_pair to record events
from paper_2401_01921_b200 import blueprint, contraction
orig = contraction.contract_pair
rec = []


def timed(a, b, out_order=None):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = orig(a, b, out_order=out_order)
    e1.record()
    rec.append((a.labels, b.labels, a.shape, b.shape, out.shape, e0, e1))
    if len(a.shape) == 7:
        print("SLOW STEP a", a.labels, a._blocks[0].storage_shape, a._blocks[0].perm)
        print("          b", b.labels, b._blocks[0].storage_shape, b._blocks[0].perm, "out", out.labels)
    return out


blueprint.contract_pair = timed
net._dense_signature = lambda: None  # no launch replay: time the pairwise path
_lib.ktimer_reset()
_lib.ktimer_enable(True)
net.launch()
_lib.ktimer_enable(False)
torch.cuda.synchronize()
tot = 0
for al, bl, ash, bsh, osh, e0, e1 in rec:
    ms = e0.elapsed_time(e1)
    sa, sb = set(al), set(bl)
    macs = 1
    dims = {}
    for l, d in zip(al, ash):
        dims[l] = d
    for l, d in zip(bl, bsh):
        dims[l] = d
    for l in sa | sb:
        macs *= dims[l]
    tot += ms
    print(f"{ms:8.3f} ms  {2*macs/ms/1e9:8.2f} TFLOP/s  A{ash} x B{bsh} -> {osh}")
print("total", tot)
for fam, nm in [(0, "gemm"), (1, "skinny"), (2, "permute"), (5, "other")]:
    print(nm, _lib.ktimer_read(fam))
