"""Break down load_unitensor of the C4 A tensor (dev aid): header + UniTensor build, page-cache
reads, host->device copies, scatter."""
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import io as tio

torch.cuda.set_device(0)
A, _ = bench.c4_tensors(tnb)
path = os.path.join(tempfile.gettempdir(), "tnb_probe_A.utn")
tnb.save_unitensor(A, path)
nbytes = sum(b.size * b.itemsize for b in A.get_blocks_())
for _ in range(3):
    tnb.load_unitensor(path)
torch.cuda.synchronize()


def tm(fn, n=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print(f"payload {nbytes / 1e6:.2f} MB")
print(f"load_unitensor {tm(lambda: tnb.load_unitensor(path)):.3f} ms")
buf = bytearray(nbytes + 4096)
def rd():
    with open(path, "rb") as f:
        f.readinto(buf)
print(f"plain file read into bytearray {tm(rd):.3f} ms")
pin = torch.empty(nbytes + 4096, dtype=torch.uint8, pin_memory=True)
def rdp():
    with open(path, "rb") as f:
        f.readinto(memoryview(pin.numpy()))
print(f"file read into pinned {tm(rdp):.3f} ms")
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
print(f"H2D copy {tm(lambda: dev.copy_(pin[:nbytes], non_blocking=True)):.3f} ms")
import concurrent.futures as cf
ex = cf.ThreadPoolExecutor(8)
fd = os.open(path, os.O_RDONLY)
mv = memoryview(pin.numpy())
def prd(k):
    sz = (nbytes + 7) // 8
    o = k * sz
    n = min(sz, nbytes - o)
    return os.preadv(fd, [mv[o:o + n]], o)
print(f"8-thread preadv into pinned {tm(lambda: list(ex.map(prd, range(8)))):.3f} ms")
print(f"oracle load {tm(lambda: bench.ORACLE.load_utn(path)):.3f} ms")
import json, struct
from paper_2401_01921_b200 import UniTensor
with open(path, "rb") as f:
    f.read(5); f.read(4)
    (hlen,) = struct.unpack("<I", f.read(4))
    hb = f.read(hlen)
header = json.loads(hb.decode())
print(f"json parse {tm(lambda: json.loads(hb.decode())):.3f} ms")
bonds = [tio._bond_from_json(d) for d in header["bonds"]]
print(f"bonds {tm(lambda: [tio._bond_from_json(d) for d in header['bonds']]):.3f} ms")
dt = tio._DTYPES[header["dtype"]]
print(f"UniTensor() {tm(lambda: UniTensor(bonds, labels=header['labels'], name=header['name'], dtype=dt, rowrank=header['rowrank'])):.3f} ms")
ut = UniTensor(bonds, labels=header['labels'], name=header['name'], dtype=dt, rowrank=header['rowrank'])
print(f"get_blocks_ + checks {tm(lambda: [ (tuple(i['qn']) == ut.block_qn_indices(k), tuple(i['shape'])==b.shape) for k,(b,i) in enumerate(zip(ut.get_blocks_(), header['blocks']))]):.3f} ms")
blocks = ut.get_blocks_()
print(f"_segments {tm(lambda: tio._segments(blocks, dt.itemsize, packed_to_slab=True)):.3f} ms")
