"""The ``.utn`` tensor container, read straight into / written straight from HBM.

Format (pkg/src/tnkit/io.py:1-19, byte-identical): ``b"TNXU\\x00"``, uint32 version (1),
uint32 header length, a UTF-8 JSON header (``name``, ``labels``, ``rowrank``, ``dtype``,
``bonds``, ``blocks``), then every block's C-order little-endian element bytes,
concatenated in block-enumeration order.

B200 path: the payload is read with ONE ``readinto`` into a pinned host
buffer and crosses PCIe in ONE copy; a single ``tnb_copy2d_batched`` launch scatters the
packed blocks to their 64-byte-aligned places in the tensor's HBM slab. Saving runs the
same in reverse: lazily
permuted blocks are materialised by ``tnb_permute``, one gather launch packs the blocks,
one device->host copy, one write. Files interchange with the reference's
``save_unitensor`` / ``load_unitensor`` (io.py:56-107) in both directions.
"""
import json
import struct
import sys

import numpy as np
import torch

from . import _lib, dense
from .charges import Bond, BondType, symmetry_from_str
from .dense import DenseTensor
from .labeled import UniTensor

MAGIC = b"TNXU\x00"
VERSION = 1

_DTYPES = {"float64": np.dtype(np.float64), "complex128": np.dtype(np.complex128),
           "int64": np.dtype(np.int64), "bool": np.dtype(np.bool_)}
_NAMES = {v: k for k, v in _DTYPES.items()}

if sys.byteorder != "little":  # the payload is little-endian and moves as raw bytes
    raise ImportError("the .utn device loader needs a little-endian host")


def _bond_to_json(b):
    return {"btype": b.btype.name, "dim": b.dim, "syms": [str(s) for s in b.syms],
            "sectors": [[list(q), d] for q, d in b.sectors]}


def _bond_from_json(d):
    btype = BondType[d["btype"]]
    if d["sectors"]:
        return Bond(btype=btype, sectors=[(tuple(q), deg) for q, deg in d["sectors"]],
                    syms=[symmetry_from_str(t) for t in d["syms"]])
    return Bond(d["dim"], btype)


def _segments(blocks, itemsize, packed_to_slab):
    """One TnbCopy2D row per block between the packed payload and the block buffers.
    Returns (segments, slab-side base pointer)."""
    ptrs = [b.data_ptr for b in blocks]
    base = min(ptrs) if ptrs else 0
    segs = np.zeros(len(blocks), dtype=_lib.COPY2D_DTYPE)
    off = 0
    for k, (b, p) in enumerate(zip(blocks, ptrs)):
        n = b.size * itemsize
        packed_off, slab_off = off, p - base
        segs[k] = (packed_off, slab_off, 1, n, n, n) if packed_to_slab else (slab_off, packed_off, 1, n, n, n)
        off += n
    return segs, base, off


def save_unitensor(ut, path):
    """Write ``ut`` in the reference's container format (io.py:56-80)."""
    blocks = [b.contiguous() for b in ut.get_blocks_()]  # tnb_permute for lazily permuted blocks
    dt = ut.dtype
    header = {
        "name": ut.name,
        "labels": ut.labels,
        "rowrank": ut.rowrank,
        "dtype": _NAMES[dt],
        "bonds": [_bond_to_json(b) for b in ut.bonds],
        "blocks": [{"qn": list(ut.block_qn_indices(i)) if ut.is_sym else None, "shape": list(blk.shape)}
                   for i, blk in enumerate(blocks)],
    }
    raw = json.dumps(header).encode()
    segs, base, nbytes = _segments(blocks, dt.itemsize, packed_to_slab=False)
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    if nbytes:
        packed = torch.empty(nbytes, dtype=torch.uint8, device=dense.device())
        _lib.copy2d_batched(base, packed.data_ptr(), segs, dense.stream_handle())
        host.copy_(packed)  # synchronous: the payload is on the host when this returns
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", VERSION))
        f.write(struct.pack("<I", len(raw)))
        f.write(raw)
        f.write(memoryview(host.numpy()))


def load_unitensor(path):
    """Read a container written by this module or by the reference (io.py:83-107)."""
    with open(path, "rb") as f:
        magic = f.read(5)
        if magic != MAGIC:
            raise ValueError(f"{path}: not a tensor container (bad magic {magic!r})")
        (version,) = struct.unpack("<I", f.read(4))
        if version != VERSION:
            raise ValueError(f"{path}: unsupported format version {version}")
        (hlen,) = struct.unpack("<I", f.read(4))
        header = json.loads(f.read(hlen).decode())
        dt = _DTYPES[header["dtype"]]
        bonds = [_bond_from_json(d) for d in header["bonds"]]
        ut = UniTensor(bonds, labels=header["labels"], name=header["name"], dtype=dt,
                       rowrank=header["rowrank"])
        blocks = ut.get_blocks_()
        binfo = header["blocks"]
        if len(binfo) != len(blocks):
            raise ValueError(f"{path}: {len(binfo)} blocks in the file, the bonds give {len(blocks)}")
        for i, (b, info) in enumerate(zip(blocks, binfo)):
            if ut.is_sym and tuple(info["qn"]) != ut.block_qn_indices(i):
                raise ValueError(f"{path}: block {i} has Qn indices {tuple(info['qn'])}, "
                                 f"expected {ut.block_qn_indices(i)}")
            if tuple(info["shape"]) != b.shape:
                raise ValueError(f"{path}: block {i} has shape {tuple(info['shape'])}, expected {b.shape}")
        segs, base, nbytes = _segments(blocks, dt.itemsize, packed_to_slab=True)
        host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        got = f.readinto(memoryview(host.numpy())) if nbytes else 0
        if got != nbytes:
            raise ValueError(f"{path}: truncated payload ({got} of {nbytes} bytes)")
    if nbytes:
        # one PCIe copy of the packed payload (pinned source: torch's host allocator keeps
        # it alive until the copy has run), then one scatter launch into the block slab
        staging = host.to(dense.device(), non_blocking=True)
        _lib.copy2d_batched(staging.data_ptr(), base, segs, dense.stream_handle())
    return ut


def _save_method(self, path):
    save_unitensor(self, path)


def _load_method(cls, path):
    return load_unitensor(path)


UniTensor.save = _save_method
UniTensor.Save = _save_method
UniTensor.load = classmethod(_load_method)
UniTensor.Load = classmethod(_load_method)
