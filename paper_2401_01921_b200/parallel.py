"""Multi-GPU execution of the hot path: one process per GPU.

* independent units (the C3b batch of matvecs, C5 PEPS sites) are sharded by index
  (``shard``) -- no data-path collective;
* a block-sparse contraction (C4) is partitioned by OUTPUT ROW PANELS
  (``TNB_BS_PANEL_ROWS`` rows of one output block) with an LPT schedule on their DMMA
  cost; every rank computes its panels with the whole K reduction locally (no
  cross-GPU reduction) and one all-gather (NCCL over NVLink on GPUs, gloo on CPU in
  the tests) assembles the output slab on every rank.

The partition and gather logic is backend-agnostic torch code so it is tested with
``gloo`` on CPU (tests/test_parallel_gloo.py).
"""
import numpy as np
import torch

from . import _lib

PANEL_ROWS = _lib.BS_PANEL_ROWS


def shard(n, world, rank):
    """Indices of `n` independent units owned by `rank` (round robin)."""
    return list(range(rank, n, world))


def lpt_partition(costs, nparts):
    """Longest-processing-time-first assignment: heaviest unit to the least-loaded part.

    Deterministic: ties in cost keep index order, ties in load pick the lowest part."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * nparts
    owner = [0] * len(costs)
    for i in order:
        p = min(range(nparts), key=lambda q: (load[q], q))
        owner[i] = p
        load[p] += costs[i]
    return owner


def panels_of(out_shapes, n_row_axes):
    """Panels in the C ABI's order: (block, row0, row1, rows, cols) per output block,
    TNB_BS_PANEL_ROWS rows each; rows = product of the first n_row_axes dims."""
    panels = []
    for o, shp in enumerate(out_shapes):
        rows = int(np.prod(shp[:n_row_axes], dtype=np.int64)) if n_row_axes else 1
        cols = int(np.prod(shp[n_row_axes:], dtype=np.int64)) if len(shp) > n_row_axes else 1
        for r0 in range(0, rows, PANEL_ROWS):
            panels.append((o, r0, min(rows, r0 + PANEL_ROWS), rows, cols))
    return panels


def block_pair_k(a_qns, a_shapes, a_pos, b_qns, b_pos, a_free, b_free, out_qns):
    """Total contracted extent per output block (host bookkeeping for the cost model)."""
    lookup = {tuple(q): k for k, q in enumerate(out_qns)}
    by_key = {}
    for j, q in enumerate(b_qns):
        by_key.setdefault(tuple(q[p] for p in b_pos), []).append(j)
    ktot = [0] * len(out_qns)
    for i, q in enumerate(a_qns):
        kdim = int(np.prod([a_shapes[i][p] for p in a_pos], dtype=np.int64)) if a_pos else 1
        for j in by_key.get(tuple(q[p] for p in a_pos), ()):
            o = lookup[tuple([q[p] for p in a_free] + [b_qns[j][p] for p in b_free])]
            ktot[o] += kdim
    return ktot


def panel_plan(out_shapes, n_row_axes, ktot, world):
    """(panels, owner per panel) with LPT on cost = rows * cols * sum_K."""
    panels = panels_of(out_shapes, n_row_axes)
    costs = [(r1 - r0) * cols * max(ktot[o], 1) for (o, r0, r1, _, cols) in panels]
    return panels, lpt_partition(costs, world)


def panel_spans(panels, block_offsets):
    """Element spans (start, length) of each panel inside the output slab."""
    return [(block_offsets[o] + r0 * cols, (r1 - r0) * cols) for (o, r0, r1, _, cols) in panels]


def gather_layout(spans, owner, rank, world, itemsize):
    """Host bookkeeping of the panel all-gather: (maxlen, pack segments, unpack segments).

    Each rank packs the spans it owns, in span order, into a send buffer of `maxlen`
    elements (the largest per-rank payload, known on every rank without communication);
    the all-gather concatenates the ranks' buffers, and every span owned by another rank
    is copied from its place in that concatenation back into the slab. Segments are
    TnbCopy2D records (one row each, byte offsets) for tnb_copy2d_batched."""
    sizes = [0] * world
    for (_, n), o in zip(spans, owner):
        sizes[o] += n
    maxlen = max(sizes) if sizes else 0
    pack, unpack = [], []
    pos = [0] * world
    for (s, n), o in zip(spans, owner):
        if n > 0:
            if o == rank:
                pack.append((s * itemsize, pos[o] * itemsize, 1, n * itemsize, 0, 0))
            else:
                unpack.append(((o * maxlen + pos[o]) * itemsize, s * itemsize, 1, n * itemsize, 0, 0))
        pos[o] += n
    return (maxlen, np.array(pack, dtype=_lib.COPY2D_DTYPE).reshape(-1),
            np.array(unpack, dtype=_lib.COPY2D_DTYPE).reshape(-1))


def _apply_segments(src, dst, segs):
    """Execute TnbCopy2D segments between two 1-D tensors: ONE tnb_copy2d_batched launch on
    the GPU; on CPU tensors (gloo tests, host-staged buffers) plain slice copies."""
    if len(segs) == 0:
        return
    if dst.is_cuda:
        from . import dense
        _lib.copy2d_batched(src.data_ptr(), dst.data_ptr(), segs, dense.stream_handle())
        return
    isz = src.element_size()
    for g in segs:
        s0, d0, n = int(g["src_off"]) // isz, int(g["dst_off"]) // isz, int(g["row_bytes"]) // isz
        dst[d0:d0 + n] = src[s0:s0 + n]


def gather_panels(slab, spans, owner, rank, world, group=None):
    """All-gather the panels each rank computed so every rank holds the full slab.

    `slab` is a 1-D tensor; `spans` are element spans, `owner` the rank of each span.
    One pack launch, ONE all-gather (``all_gather_into_tensor``: NCCL over NVLink for
    CUDA slabs), one unpack launch. With a CPU backend (gloo) and a CUDA slab the packed
    buffers are staged through host memory."""
    import torch.distributed as dist
    maxlen, pack, unpack = gather_layout(spans, owner, rank, world, slab.element_size())
    if maxlen == 0:
        return slab
    send = torch.empty(maxlen, dtype=slab.dtype, device=slab.device)
    _apply_segments(slab, send, pack)
    host_staged = slab.is_cuda and dist.get_backend(group) == "gloo"
    if host_staged:
        send = send.cpu()
    recv = torch.empty(world * maxlen, dtype=slab.dtype, device=send.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    if host_staged:
        recv = recv.to(slab.device, non_blocking=False)
    _apply_segments(recv, slab, unpack)
    return slab


_SHARD_PLANS = {}


def _shard_plan(a, b, a_pos, b_pos, a_free, b_free, out_bonds, qns, world, rank, itemsize):
    """Per-structure host bookkeeping of a sharded contraction, cached: the LPT panel
    owners, this rank's panel mask and the all-gather's pack/unpack segments."""
    a_shapes = tuple(tuple(blk.shape) for blk in a._blocks)
    key = (tuple(a._qns), a_shapes, tuple(b._qns), tuple(a_pos), tuple(b_pos), tuple(out_bonds), world, rank,
           itemsize)
    hit = _SHARD_PLANS.get(key)
    if hit is not None:
        return hit
    from .labeled import _slab_layout
    shapes = [tuple(x.sectors[k][1] for x, k in zip(out_bonds, qn)) for qn in qns]
    ktot = block_pair_k(a._qns, a_shapes, a_pos, b._qns, b_pos, a_free, b_free, qns)
    panels, owner = panel_plan(shapes, len(a_free), ktot, world)
    mask = np.array([1 if o == rank else 0 for o in owner], dtype=np.uint8)
    offsets, _ = _slab_layout(shapes, np.dtype(np.complex128 if itemsize == 16 else np.float64))
    spans = panel_spans(panels, list(offsets))
    if len(_SHARD_PLANS) >= 256:
        _SHARD_PLANS.clear()
    _SHARD_PLANS[key] = hit = (mask, spans, owner, list(offsets))
    return hit


def contract_sharded(a, b, group=None):
    """Block-sparse ``contract_pair`` partitioned over the ranks of `group`: each rank
    computes its LPT share of output panels (one grouped launch with a panel mask, the
    whole K reduction local), then one all-gather assembles the slab on every rank."""
    import torch.distributed as dist
    from . import contraction as C
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1 or not a.is_sym:
        return C.contract_pair(a, b)
    a_pos, b_pos, a_free, b_free, out_labels, out_bonds = C._pair_layout(a, b)
    from .labeled import zero_flux_combos
    qns = zero_flux_combos(out_bonds)
    dt = C._result_dtype(a.dtype, b.dtype)
    mask, spans, owner, offsets = _shard_plan(a, b, a_pos, b_pos, a_free, b_free, out_bonds, qns, world, rank,
                                     np.dtype(dt).itemsize)
    out = C._contract_blocks(a, b, a_pos, b_pos, a_free, b_free, out_labels, out_bonds, panel_mask=mask)
    slab = out._blocks[0]._slab
    if [blk._off for blk in out._blocks] != offsets:
        raise _lib.EngineError("contract_sharded: output slab layout differs from the panel plan")
    gather_panels(slab, spans, owner, rank, world, group)
    return out
