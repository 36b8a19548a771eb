"""The ``.utn`` tensor container, read straight into / written straight from HBM.

Format (pkg/src/tnkit/io.py:1-19, byte-identical): ``b"TNXU\\x00"``, uint32 version (1),
uint32 header length, a UTF-8 JSON header (``name``, ``labels``, ``rowrank``, ``dtype``,
``bonds``, ``blocks``), then every block's C-order little-endian element bytes,
concatenated in block-enumeration order.

B200 path: the payload is read in 4 MB chunks into two pinned host
buffers while the previous chunk crosses PCIe (file read and transfer overlap); a single
``tnb_copy2d_batched`` launch scatters the
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


_SECTORS = {}  # (syms, raw sectors) -> validated (sectors, syms, dim); tuples only (immutable)


def _bond_from_json(d):
    btype = BondType[d["btype"]]
    if not d["sectors"]:
        return Bond(d["dim"], btype)
    key = (tuple(d["syms"]), tuple((tuple(q), deg) for q, deg in d["sectors"]))
    hit = _SECTORS.get(key)
    if hit is None:
        ref = Bond(btype=btype, sectors=list(key[1]), syms=[symmetry_from_str(t) for t in d["syms"]])
        hit = (ref.sectors, ref.syms, ref.dim)
        if len(_SECTORS) >= 1024:
            _SECTORS.clear()
        _SECTORS[key] = hit
    # a fresh Bond per load (bonds have in-place mutators); the validated fields are shared
    b = Bond.__new__(Bond)
    b.btype, (b.sectors, b.syms, b.dim), b._offsets = btype, hit, None
    return b


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
        if nbytes:
            staging = torch.empty(nbytes, dtype=torch.uint8, device=dense.device())
            _read_to_device(f, staging, nbytes, path)
            # one scatter launch: packed payload -> 64-byte-aligned blocks of the slab
            _lib.copy2d_batched(staging.data_ptr(), base, segs, dense.stream_handle())
    return ut


_CHUNK = 2 << 20   # read / copy piece
# threads reading pieces from the page cache (tnb_file_to_device): 2 for a few-MB payload
# (C4 A tensor, 6.1 MB: 1 / 2 / 4 / 8 readers 0.70 / 0.57 / 0.65 / 0.67 ms -- thread wake-ups
# cost more than they save beyond that), one more per 8 MB above, at most 8
_READERS = 0       # (0 = by size as above)
_PINNED = []       # [pinned payload buffer, event: its last host->device copy done]


def _read_to_device(f, staging, nbytes, path):
    """Pipelined file -> HBM through the native reader (tnb_file_to_device, csrc/fileio.cpp):
    pooled pread()s of _CHUNK pieces into one pinned buffer, each piece copied to HBM as soon
    as it and every earlier piece have landed -- the page-cache copy, the cost here, runs on
    _READERS threads and the PCIe transfer behind it."""
    if not _PINNED or _PINNED[0].numel() < nbytes:
        if _PINNED:
            _PINNED[1].synchronize()
        _PINNED[:] = [torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True), torch.cuda.Event()]
    buf, done = _PINNED
    done.synchronize()  # the previous load's copies out of the buffer have finished
    start = f.tell()
    try:
        readers = _READERS or max(2, min(8, 1 + nbytes // (8 << 20)))
        _lib.file_to_device(f.fileno(), start, nbytes, buf.data_ptr(), staging.data_ptr(), _CHUNK, readers,
                            dense.stream_handle())
    except _lib.EngineError as e:
        raise ValueError(f"{path}: truncated payload ({e})") from None
    done.record(torch.cuda.current_stream())
    f.seek(start + nbytes)


_PAYLOAD_SEGS = {}  # (structure id, direction) -> (segments, packed bytes, slab byte offset of block 0)


def _cached_segments(ut, packed_to_slab):
    """Payload <-> slab segments of a block-sparse tensor held in one slab (contraction._bs_info):
    computed once per block structure; returns (segments, slab base pointer, bytes) or None."""
    from .contraction import _bs_info
    info = _bs_info(ut) if ut.is_sym else None
    if info is None:
        return None
    sid, slab, offs, dt = info
    key = (sid, bool(packed_to_slab))
    hit = _PAYLOAD_SEGS.get(key)
    if hit is None:
        isz = dt.itemsize
        sizes = np.array([int(np.prod(b, dtype=np.int64)) for b in _shapes_of(ut)], dtype=np.int64) * isz
        packed = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        slab_off = (offs - offs[0]) * isz
        segs = np.zeros(len(sizes), dtype=_lib.COPY2D_DTYPE)
        src, dst = (packed, slab_off) if packed_to_slab else (slab_off, packed)
        segs["src_off"], segs["dst_off"], segs["rows"] = src, dst, 1
        segs["row_bytes"], segs["src_pitch"], segs["dst_pitch"] = sizes, sizes, sizes
        if len(_PAYLOAD_SEGS) >= 256:
            _PAYLOAD_SEGS.clear()
        hit = _PAYLOAD_SEGS[key] = (segs, int(sizes.sum()), int(offs[0]) * isz)
    segs, nbytes, off0 = hit
    return segs, slab.data_ptr() + off0, nbytes, slab


def _shapes_of(ut):
    if ut._blk is None:
        return ut._lazy[3]
    return [b.storage_shape for b in ut._blk]


def payload_nbytes(ut):
    """Bytes of the packed payload of ``ut``: every block's C-order elements concatenated in
    block order (the ``.utn`` payload layout, io.py:56-80)."""
    return sum(b.size for b in ut.get_blocks_()) * ut.dtype.itemsize


def upload_payload_(ut, host, after=None):
    """Fill every block of ``ut`` from a host payload (pinned CPU tensor or numpy array in
    the packed ``.utn`` layout, same dtype): one host->device copy into a staging buffer and
    one ``tnb_copy2d_batched`` scatter to the blocks' places in the slab, both queued on the
    engine's upload stream (asynchronous for pinned input); the next engine call reading the
    tensor waits for them on its own stream (as ``DenseTensor.upload_``). ``after`` (a CUDA
    event): order the upload after this event only instead of after everything queued on the
    current stream (serving loops: the event that follows the last read of the old
    contents). Blocks must be stored contiguously (a freshly built or loaded tensor)."""
    h = torch.as_tensor(host) if not isinstance(host, torch.Tensor) else host
    fast = _cached_segments(ut, True)
    if fast is not None and ut._blk is not None and ut._blk and ut._blk[0]._perm != tuple(range(ut.rank)):
        fast = None  # lazily permuted blocks: the payload is in logical order
    if fast is not None:
        segs, base, nbytes, slab = fast
        owners = [slab]
    else:
        blocks = ut.get_blocks_()
        if any(not b.is_contiguous for b in blocks):
            raise ValueError("upload_payload_: blocks must be contiguous (materialise with contiguous_() first)")
        nbytes = payload_nbytes(ut)
    if h.numel() * h.element_size() != nbytes:
        raise ValueError(f"upload_payload_: host payload has {h.numel() * h.element_size()} bytes, expected {nbytes}")
    if not nbytes:
        return ut
    if fast is None:
        segs, base, _ = _segments(blocks, ut.dtype.itemsize, packed_to_slab=True)
    if fast is None:
        owners = list({id(o): o for o in (dense._owner(b) for b in blocks)}.values())
    up = dense.upload_stream()
    if after is None:
        up.wait_stream(torch.cuda.current_stream())  # WAR: earlier readers of the blocks
    else:
        up.wait_event(after)
    for o in owners:
        o.record_stream(up)
    with torch.cuda.stream(up):
        staging = torch.empty(nbytes, dtype=torch.uint8, device=dense.device())
        staging.copy_(h.reshape(-1).view(torch.uint8), non_blocking=True)
        _lib.copy2d_batched(staging.data_ptr(), base, segs, up.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(up)
    for o in owners:  # a still-pending earlier upload into o precedes ev on the same stream
        o._tnb_ready = ev
    return ut


def download_payload(ut, host, done=None):
    """Copy every block of ``ut`` into a host payload (pinned CPU tensor in the packed
    ``.utn`` layout): one gather launch and one device->host copy queued on the current
    stream; synchronise (or wait on an event) before reading ``host``. With ``done`` (a CUDA
    event) both run on the engine's download stream instead, after everything queued on the
    current stream, and ``done`` is recorded once ``host`` holds the payload -- the current
    stream moves on to the next step's work meanwhile."""
    fast = _cached_segments(ut, False)
    if fast is not None and ut._blk is not None and ut._blk and ut._blk[0]._perm != tuple(range(ut.rank)):
        fast = None
    if fast is not None:
        segs, base, nbytes, slab = fast
        dense._await(slab)
    else:
        blocks = [b.contiguous() for b in ut.get_blocks_()]
        nbytes = payload_nbytes(ut)
    if host.numel() * host.element_size() != nbytes:
        raise ValueError(f"download_payload: host buffer has {host.numel() * host.element_size()} bytes, "
                         f"expected {nbytes}")
    if not nbytes:
        return host
    if fast is None:
        segs, base, _ = _segments(blocks, ut.dtype.itemsize, packed_to_slab=False)
    if done is None:
        packed = torch.empty(nbytes, dtype=torch.uint8, device=dense.device())
        _lib.copy2d_batched(base, packed.data_ptr(), segs, dense.stream_handle())
        host.reshape(-1).view(torch.uint8).copy_(packed, non_blocking=True)
        return host
    d2h = dense.download_stream()
    d2h.wait_stream(torch.cuda.current_stream())
    for o in ([slab] if fast is not None else {id(dense._owner(b)): dense._owner(b) for b in blocks}.values()):
        o.record_stream(d2h)  # the blocks may be freed (to the current stream's pool) before d2h reads them
    with torch.cuda.stream(d2h):
        packed = torch.empty(nbytes, dtype=torch.uint8, device=dense.device())
        _lib.copy2d_batched(base, packed.data_ptr(), segs, d2h.cuda_stream)
        host.reshape(-1).view(torch.uint8).copy_(packed, non_blocking=True)
        done.record(d2h)
    return host


def _save_method(self, path):
    save_unitensor(self, path)


def _load_method(cls, path):
    return load_unitensor(path)


UniTensor.upload_payload_ = upload_payload_
UniTensor.download_payload = download_payload
UniTensor.save = _save_method
UniTensor.Save = _save_method
UniTensor.load = classmethod(_load_method)
UniTensor.Load = classmethod(_load_method)
