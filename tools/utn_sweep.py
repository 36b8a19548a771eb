"""Sweep the native .utn reader's threads / piece size on the C4 A tensor (dev aid)."""
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
A, _ = bench.c4_tensors(tnb)
path = "/tmp/tnb_sweep_A.utn"
tnb.save_unitensor(A, path)
nbytes = sum(b.size * b.itemsize for b in A.get_blocks_())
for readers in (1, 2, 4, 8, 12):
    for chunk in (256 << 10, 512 << 10, 1 << 20, 2 << 20):
        tio._READERS, tio._CHUNK = readers, chunk
        for _ in range(5):
            tnb.load_unitensor(path)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(40):
            tnb.load_unitensor(path)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / 40 * 1e3
        print(f"readers {readers:2d} chunk {chunk >> 10:5d} KB: {ms:.3f} ms ({nbytes / ms / 1e6:.1f} GB/s)")
