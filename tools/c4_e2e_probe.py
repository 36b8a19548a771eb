"""Breakdown of the C4 host-buffer step (dev aid)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import io as tio

torch.cuda.set_device(0)
A, E = bench.c4_tensors(tnb)
hA = torch.empty(tio.payload_nbytes(A), dtype=torch.uint8, pin_memory=True)
hE = torch.empty(tio.payload_nbytes(E), dtype=torch.uint8, pin_memory=True)
tio.download_payload(A, hA)
tio.download_payload(E, hE)
out = tnb.contract(A, E)
hO = torch.empty(tio.payload_nbytes(out), dtype=torch.uint8, pin_memory=True)
A2, E2 = bench.c4_tensors(tnb, seed=1)


def step():
    A2.upload_payload_(hA)
    E2.upload_payload_(hE)
    tnb.contract(A2, E2).download_payload(hO)


for _ in range(5):
    step()
torch.cuda.synchronize()
for name, fn in [("upload A", lambda: A2.upload_payload_(hA)), ("contract", lambda: tnb.contract(A2, E2)),
                 ("download", lambda: out.download_payload(hO)), ("step", step)]:
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: host {(t1 - t0) / 20 * 1e6:.1f} us, device {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
