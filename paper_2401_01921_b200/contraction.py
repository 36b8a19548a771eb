"""Label-driven contraction: the hot path's host layer.

Public functions and their reference counterparts (pkg/src/tnkit/contract.py):

* ``contract_pair``       -> contract_pair :100-134 (dense) / _contract_pair_blocks :137-167
* ``contract``            -> contract :172-219, ``execute_tree`` :222-226
* ``find_optimal_order``  -> find_optimal_order :271-343 (native DP, same tie-break)
* ``contraction_cost``, ``brute_force_order``, ``parse_order``, ``render_order``,
  ``tree_leaves``          -> :19-79, :253-268, :351-372

Validation (labels, directions, sectors, duplicate free labels) happens here,
before any device work, with the reference's exception types. The arithmetic
is libtnb: ``tnb_contract_dense`` (DMMA GEMM reading lazily permuted operands in
place) and ``tnb_bs_plan``/``tnb_bs_execute`` (device pairing once per block
structure + grouped stream-K GEMM per call). There is no CPU
fallback: int64/bool contractions raise TypeError.
"""
import itertools
import os
import re

import numpy as np
import torch

from . import _lib, dense
from .charges import REGULAR
from .dense import Complex128, DenseTensor, Float64
from .labeled import UniTensor

_NAME_RE = re.compile(r"[A-Za-z0-9_*'+\-]+")

_CPLX_MODE = _lib.CPLX_3M if os.environ.get("TNB_CPLX", "4M").upper() == "3M" else _lib.CPLX_4M


def set_complex_mode(mode):
    """'4M' (four real DMMA products per complex MAC) or '3M' (Gauss, 3 products)."""
    global _CPLX_MODE
    mode = str(mode).upper()
    if mode not in ("4M", "3M"):
        raise ValueError("complex mode must be '4M' or '3M'")
    _CPLX_MODE = _lib.CPLX_3M if mode == "3M" else _lib.CPLX_4M


def get_complex_mode():
    return "3M" if _CPLX_MODE == _lib.CPLX_3M else "4M"


# -- order trees: leaf = name (str), node = (left, right) ------------------------------
def render_order(tree):
    return tree if isinstance(tree, str) else "(" + render_order(tree[0]) + "," + render_order(tree[1]) + ")"


def parse_order(text):
    """Grammar ``name | "(" order "," order ")"`` (whitespace allowed between tokens)."""
    n = len(text)

    def bad(pos, msg):
        raise ValueError(f"malformed order string {text!r} at {pos}: {msg}")

    def ws(pos):
        while pos < n and text[pos].isspace():
            pos += 1
        return pos

    def node(pos):
        pos = ws(pos)
        if pos >= n:
            bad(pos, "unexpected end")
        if text[pos] == "(":
            left, pos = node(pos + 1)
            pos = ws(pos)
            if pos >= n or text[pos] != ",":
                bad(pos, "expected ','")
            right, pos = node(pos + 1)
            pos = ws(pos)
            if pos >= n or text[pos] != ")":
                bad(pos, "expected ')'")
            return (left, right), pos + 1
        m = _NAME_RE.match(text, pos)
        if not m:
            bad(pos, "expected a tensor name")
        return m.group(), m.end()

    tree, pos = node(0)
    pos = ws(pos)
    if pos != n:
        bad(pos, "trailing characters")
    return tree


def tree_leaves(tree):
    if isinstance(tree, str):
        return [tree]
    return tree_leaves(tree[0]) + tree_leaves(tree[1])


# -- pairwise ---------------------------------------------------------------------------------
def _check_pair_bond(label, ba, bb):
    if ba.dim != bb.dim:
        raise ValueError(f"label {label!r}: dimension mismatch ({ba.dim} vs {bb.dim})")
    if (ba.btype == REGULAR) != (bb.btype == REGULAR):
        raise ValueError(f"label {label!r}: cannot contract a REGULAR bond with a directed bond")
    if ba.btype != REGULAR and ba.btype == bb.btype:
        raise ValueError(f"label {label!r}: only bonds with opposite directions can be contracted "
                         f"(both {ba.btype})")
    if (ba.has_qnums or bb.has_qnums) and (ba.syms != bb.syms or ba.sectors != bb.sectors):
        raise ValueError(f"label {label!r}: quantum-number sectors do not match")


def _pair_layout(a, b):
    """Shared labels (a's order), contracted/free positions, output labels/bonds."""
    al, bl = a._labels, b._labels
    bset = set(bl)
    shared = [l for l in al if l in bset]
    a_pos = [al.index(l) for l in shared]
    b_pos = [bl.index(l) for l in shared]
    for l, pa, pb in zip(shared, a_pos, b_pos):
        _check_pair_bond(l, a._bonds[pa], b._bonds[pb])
    sset = set(shared)
    a_free = [i for i, l in enumerate(al) if l not in sset]
    b_free = [i for i, l in enumerate(bl) if l not in sset]
    out_labels = [al[i] for i in a_free] + [bl[i] for i in b_free]
    if len(set(out_labels)) != len(out_labels):
        raise ValueError(f"duplicate free labels in contraction result: {out_labels}")
    out_bonds = [a._bonds[i] for i in a_free] + [b._bonds[i] for i in b_free]
    return a_pos, b_pos, a_free, b_free, out_labels, out_bonds


def _result_dtype(da, db):
    dt = np.result_type(da, db)
    if dt not in (Float64, Complex128):
        raise TypeError(f"contraction of {da} x {db} is not supported on the GPU engine "
                        "(float64 / complex128 only; there is no CPU fallback)")
    return dt


def contract_pair(a, b, out_order=None):
    """Contract two UniTensors over all shared labels; output = a_free then b_free labels.
    out_order (dense operands only): the PHYSICAL order of the output's axes (a tuple of
    logical axis indices) -- the result is the same tensor, stored in that order and read
    back as a lazy permute (Network launches lay intermediates out for their consumer)."""
    if not isinstance(a, UniTensor) or not isinstance(b, UniTensor):
        raise TypeError("contract expects UniTensors")
    if a.is_sym != b.is_sym:
        raise ValueError("cannot contract a block-sparse tensor with a dense one; use convert_from first")
    if a.is_sym:
        out = _contract_blocks_fast(a, b)  # a structure pair seen (and checked) before
        if out is not None:
            return out
    a_pos, b_pos, a_free, b_free, out_labels, out_bonds = _pair_layout(a, b)
    if not a.is_sym:
        return _contract_dense(a, b, a_pos, b_pos, a_free, b_free, out_labels, out_bonds, out_order)
    return _contract_blocks(a, b, a_pos, b_pos, a_free, b_free, out_labels, out_bonds)


def _contract_dense(a, b, a_pos, b_pos, a_free, b_free, out_labels, out_bonds, out_order=None):
    A, B = a._blocks[0], b._blocks[0]
    dt = _result_dtype(A.dtype, B.dtype)
    out_shape = [A.shape[i] for i in a_free] + [B.shape[j] for j in b_free]
    chunks = dense.pending_chunks(B)
    k0 = B.perm.index(0) if B.rank else -1  # logical axis stored outermost
    if out_order is not None and (chunks or tuple(out_order) == tuple(range(len(out_shape)))):
        out_order = None
    if out_order is not None:
        out_order = tuple(int(x) for x in out_order)
        inv = [0] * len(out_order)
        for p, x in enumerate(out_order):
            inv[x] = p
        out = DenseTensor.empty([out_shape[x] for x in out_order], dt).permute(*inv)
    else:
        out = DenseTensor.empty(out_shape, dt)
    if chunks and b_free and b_free[0] == k0 and A.dtype == B.dtype:
        _contract_dense_panels(A, B, a_pos, b_pos, b_free, out, chunks)
    else:
        _lib.contract_dense(A.data_ptr, dense.dtype_code(A.dtype), A.storage_shape, A.perm,
                            B.data_ptr, dense.dtype_code(B.dtype), B.storage_shape, B.perm,
                            a_pos, b_pos, out.data_ptr, _CPLX_MODE, dense.stream_handle(), out_order=out_order)
        if _RECORD is not None:
            _RECORD.append((A, B, tuple(a_pos), tuple(b_pos), tuple(out_shape), dt, out,
                            out_bonds, out_labels, len(a_free)))
    if not out_shape:
        return UniTensor.scalar(out)
    return UniTensor._assemble(out_bonds, out_labels, len(a_free), "", [out], None)


# set (to a list) by Network.launch while it records a dense launch program
_RECORD = None


def _contract_dense_panels(A, B, a_pos, b_pos, b_free, out, chunks):
    """B is being uploaded in chunks along its outermost storage axis, which is its first
    free axis: each chunk is a column panel [s0*inner, s1*inner) of the (row-major) output.
    Launch one panel contraction per chunk, each waiting only for its own chunk's event."""
    cur = torch.cuda.current_stream()
    ncols = 1
    for j in b_free:
        ncols *= B.shape[j]
    inner = ncols // B.storage_shape[0]
    bstride = B.size // B.storage_shape[0]
    es, oes = B.itemsize, out.itemsize
    a_ptr, b_base, o_base = A.data_ptr, dense.raw_ptr(B), out.data_ptr
    sink = _PANEL_SINK
    if sink is not None and not (sink.tensor.numel() == out.size and
                                 dense._NP_OF_TORCH.get(sink.tensor.dtype) == out.dtype):
        sink = None
    d2h = dense.download_stream() if sink is not None else None
    rows = out.size // ncols
    for (s0, s1), ev in chunks:
        cur.wait_event(ev)
        shp = (s1 - s0,) + tuple(B.storage_shape[1:])
        _lib.contract_dense(a_ptr, dense.dtype_code(A.dtype), A.storage_shape, A.perm,
                            b_base + s0 * bstride * es, dense.dtype_code(B.dtype), shp, B.perm,
                            a_pos, b_pos, o_base + s0 * inner * oes, _CPLX_MODE, dense.stream_handle(),
                            out_ld=ncols)
        if d2h is not None:  # stream this panel to the host while the next one computes
            done = torch.cuda.Event()
            done.record(cur)
            d2h.wait_event(done)
            _lib.memcpy2d_async(sink.tensor.data_ptr() + s0 * inner * oes, ncols * oes,
                                o_base + s0 * inner * oes, ncols * oes, (s1 - s0) * inner * oes, rows, 2,
                                d2h.cuda_stream)
    if d2h is not None:
        cur.wait_stream(d2h)  # the caller's stream sees the whole host result
        sink.used = True
    dense._owner(B)._tnb_ready = None  # every chunk is now ordered before this stream's work


class _Sink:
    __slots__ = ("tensor", "used")

    def __init__(self, tensor):
        self.tensor, self.used = tensor, False


# set by Network.launch(host_out=...) around the root contraction only
_PANEL_SINK = None


def _common_perm(t):
    blks = t._blocks
    p0 = blks[0]._perm if blks else ()
    if all(blk._perm == p0 for blk in blks):
        return blks, p0
    # blocks were permuted individually (put_block_/contiguous_ on one block): materialise
    return [blk.contiguous() for blk in t._blocks], tuple(range(t.rank))


def _widen(blocks, dt):
    if blocks:
        o = blocks[0]._slab
        if o is not None and dense._NP_OF_TORCH[o.dtype] == dt and all(b._slab is o for b in blocks):
            return blocks  # one slab of the target dtype: nothing to widen
    return [b if b.dtype == dt else b.astype(dt) for b in blocks]


# -- cached block-sparse structure (host fast path) ---------------------------------------------------
_SIG_IDS = {}          # structure signature -> id (ids are never reused, so stale ids cannot collide)
_SIG_NEXT = [1]


def _bond_key(b):
    return (b.btype, b.dim, tuple(b.sectors), tuple(b.syms))


def _bs_info(t):
    """(structure id, slab, element offsets, dtype) of a block-sparse tensor whose blocks are
    all views of ONE slab with ONE common perm -- every tensor the engine itself builds --
    else None. The structure id stands for (dtype, labels, bonds by
    value, qn tuples, block storage shapes, perm): equal ids mean the reference's pair checks
    and the device plan of pair 0 hold for this tensor too. Cached on the tensor until the next
    in-place metadata mutation anywhere (dense._EPOCH)."""
    ep = dense._EPOCH[0]
    c = getattr(t, "_bsc", None)
    if c is not None and c[0] == ep:
        return c[1]
    info = None
    if t._qns is not None:
        if t._blk is None:  # lazily held output blocks: contiguous views of one slab
            slab, base, offs, shapes, isz = t._lazy
            perm = tuple(range(len(shapes[0]))) if shapes else ()
            offs = np.asarray(offs, dtype=np.int64) + base
            sshapes = tuple(shapes)
        else:
            blks = t._blk
            slab = blks[0]._slab if blks else None
            perm = blks[0]._perm if blks else ()
            ok = slab is not None and all(b._slab is slab and b._perm == perm for b in blks)
            if ok:
                offs = np.fromiter((b._off for b in blks), dtype=np.int64, count=len(blks))
                sshapes = tuple(b._sshape for b in blks)
            else:
                slab = None
        if slab is not None:
            dt = dense._NP_OF_TORCH[slab.dtype]
            sig = (dt.char, tuple(t._labels), tuple(_bond_key(b) for b in t._bonds), tuple(t._qns), sshapes, perm)
            sid = _SIG_IDS.get(sig)
            if sid is None:
                if len(_SIG_IDS) >= 4096:
                    _SIG_IDS.clear()
                sid = _SIG_IDS[sig] = _SIG_NEXT[0]
                _SIG_NEXT[0] += 1
            info = (sid, slab, offs, dt)
    t._bsc = (ep, info)
    return info


def _info_ptrs(info):
    """Device addresses of the blocks of a tensor described by _bs_info (awaits a pending
    upload into its slab, as block_ptrs does)."""
    sid, slab, offs, dt = info
    dense._await(slab)
    return slab.data_ptr() + offs * dt.itemsize


# (structure id of a, structure id of b) -> everything a contraction of that pair of
# structures needs besides data pointers: the reference's pair checks passed for it once.
_FAST = {}


def _fast_entry(ia, ib):
    return _FAST.get((ia[0], ib[0])) if ia is not None and ib is not None else None


def _remember_fast(ia, ib, plan, lay, shapes, qns, dt):
    if ia is None or ib is None or ia[3] != dt or ib[3] != dt:
        return
    offs, total = _slab_layout_of(shapes, dt)
    if len(_FAST) >= 512:
        _FAST.clear()
    _FAST[(ia[0], ib[0])] = (plan, lay, tuple(shapes), list(qns), {q: i for i, q in enumerate(qns)},
                             np.asarray(offs, dtype=np.int64), int(max(total, 1)), dt)


def _slab_layout_of(shapes, dt):
    from .labeled import _slab_layout
    return _slab_layout(tuple(shapes), dt)


def _fast_outputs(entry, pairs):
    """Lazily held results of one structure for every (a, b) in `pairs`, in ONE allocation:
    (results, pointer table [n][nout]). Each result's bonds are its own a's / b's Bond objects
    (a_free then b_free), as the reference builds them (contract.py:124)."""
    plan, lay, shapes, qns, lookup, offs, total, dt = entry
    n = len(pairs)
    slab = dense._alloc(total * n, dt)
    isz = dt.itemsize
    base = slab.data_ptr()
    ptrs = base + (np.arange(n, dtype=np.int64)[:, None] * total + offs[None, :]) * isz
    a_free, b_free, out_labels = lay[2], lay[3], lay[4]
    offl = offs.tolist()
    outs = []
    for i, (a, b) in enumerate(pairs):
        bonds = [a._bonds[x] for x in a_free] + [b._bonds[x] for x in b_free]
        outs.append(UniTensor._assemble_lazy(bonds, out_labels, len(a_free), "", (slab, i * total, offl, shapes, isz),
                                             qns, lookup))
    return outs, ptrs


def _contract_blocks_fast(a, b):
    """contract_pair of two block-sparse tensors whose structure pair was contracted before:
    pointer arrays from the cached slab descriptors, cached plan, lazily held output. Returns
    None when the fast path does not apply (the caller takes the full path)."""
    ia, ib = _bs_info(a), _bs_info(b)
    entry = _fast_entry(ia, ib)
    if entry is None:
        return None
    outs, optrs = _fast_outputs(entry, ((a, b),))
    if not entry[0].execute(_info_ptrs(ia).tolist(), _info_ptrs(ib).tolist(), optrs[0].tolist(),
                            dense.stream_handle()):
        _FAST.clear()
        _BS_PLANS.clear()
        return None
    return outs[0]


def _contract_blocks(a, b, a_pos, b_pos, a_free, b_free, out_labels, out_bonds, panel_mask=None):
    dt = _result_dtype(a.dtype, b.dtype)
    ablk, aperm = _common_perm(a)
    bblk, bperm = _common_perm(b)
    ablk, bblk = _widen(ablk, dt), _widen(bblk, dt)
    if not out_bonds:
        return _contract_blocks_scalar(a, b, ablk, bblk, a_pos, b_pos, dt)
    from .labeled import _slab_blocks, zero_flux_combos
    if not all(x.syms == out_bonds[0].syms for x in out_bonds):
        raise ValueError("all bonds must carry the same symmetries")
    qns = zero_flux_combos(out_bonds)
    if not qns:
        raise ValueError("no valid blocks: no combination of these bonds' sectors has zero flux")
    plan, shapes = _bs_plan(dt, a, ablk, aperm, b, bblk, bperm, a_pos, b_pos, out_bonds, qns, panel_mask)
    # every output block is fully written by the kernel (with a panel mask: the panels
    # of this rank; parallel.gather_panels fills the rest)
    oblk, _ = _slab_blocks(shapes, dt, zero=False)
    aptrs, bptrs, optrs = dense.block_ptrs(ablk), dense.block_ptrs(bblk), [x._p0 for x in oblk]
    if not plan.execute(aptrs, bptrs, optrs, dense.stream_handle()):
        _BS_PLANS.clear()  # the library flushed its plan cache: re-plan this structure
        plan, _ = _bs_plan(dt, a, ablk, aperm, b, bblk, bperm, a_pos, b_pos, out_bonds, qns, panel_mask)
        if not plan.execute(aptrs, bptrs, optrs, dense.stream_handle()):
            raise _lib.EngineError("block-sparse plan went stale twice")
    if panel_mask is None:
        _remember_fast(_bs_info(a), _bs_info(b), plan, (a_pos, b_pos, a_free, b_free, out_labels, out_bonds), shapes,
                       qns, dt)
    return UniTensor._assemble(out_bonds, out_labels, len(a_free), "", oblk, qns)


# Device-resident block-sparse plans (tnb_bs_plan), keyed by the block STRUCTURE of a
# contraction: a repeated call (Lanczos matvec, equal-structure sites) only marshals the
# block pointers and launches the grouped GEMM.
_BS_PLANS = {}


def _bs_plan(dt, a, ablk, aperm, b, bblk, bperm, a_pos, b_pos, out_bonds, qns, panel_mask=None):
    a_sh = tuple(x.storage_shape for x in ablk)
    b_sh = tuple(x.storage_shape for x in bblk)
    key = (dt.char, tuple(a._qns), a_sh, tuple(aperm), tuple(b._qns), b_sh, tuple(bperm), tuple(a_pos),
           tuple(b_pos), tuple(out_bonds), None if panel_mask is None else bytes(np.asarray(panel_mask, np.uint8)))
    hit = _BS_PLANS.get(key)
    if hit is not None:
        return hit
    shapes = tuple(tuple(x.sectors[k][1] for x, k in zip(out_bonds, qn)) for qn in qns)
    plan = _lib.bs_plan(dense.dtype_code(dt), a._qns, list(a_sh), aperm, b._qns, list(b_sh), bperm, a_pos, b_pos,
                        qns, shapes, dense.stream_handle(), panel_mask=panel_mask)
    if len(_BS_PLANS) >= 512:
        _BS_PLANS.clear()
    _BS_PLANS[key] = (plan, shapes)
    return plan, shapes


def contract_batched(pairs):
    """``[contract_pair(a, b) for a, b in pairs]`` for block-sparse pairs that share ONE block
    structure (same labels, qn tuples, block shapes, storage perms, dtypes: e.g. the
    equal-structure sites of a sweep), as ONE grouped stream-K launch over the output tiles
    of all of them (``tnb_bs_execute_batched``); each result equals the single-pair
    contraction (same per-tile pair order). Dense pairs, scalar results and mixed
    structures are contracted pair by pair (mixed structures raise ValueError). The
    reference has no batched call; this is the batched form of contract.py:137-167."""
    pairs = [tuple(p) for p in pairs]
    if not pairs:
        return []
    for p in pairs:
        if len(p) != 2 or not isinstance(p[0], UniTensor) or not isinstance(p[1], UniTensor):
            raise TypeError("contract_batched expects (UniTensor, UniTensor) pairs")
    a0, b0 = pairs[0]
    if not (a0.is_sym and b0.is_sym) or len(pairs) == 1:
        return [contract_pair(a, b) for a, b in pairs]
    # fast path: every pair has the structure ids of a pair of structures contracted (and
    # checked) before -> pointer tables straight from the cached slab descriptors
    ia0, ib0 = _bs_info(a0), _bs_info(b0)
    entry = _fast_entry(ia0, ib0)
    if entry is not None:
        infos = [(_bs_info(a), _bs_info(b)) for a, b in pairs]
        if all(x is not None and y is not None and x[0] == ia0[0] and y[0] == ib0[0] for x, y in infos):
            outs, optrs = _fast_outputs(entry, pairs)
            aps = np.stack([_info_ptrs(x) for x, _ in infos])
            bps = np.stack([_info_ptrs(y) for _, y in infos])
            if entry[0].execute_batched(aps, bps, optrs, dense.stream_handle()):
                return outs
            _FAST.clear()  # the library flushed its plans: re-plan on the full path
            _BS_PLANS.clear()
    a_pos, b_pos, a_free, b_free, out_labels, out_bonds = _pair_layout(a0, b0)
    if not out_bonds:
        return [contract_pair(a, b) for a, b in pairs]
    dt = _result_dtype(a0.dtype, b0.dtype)
    from .labeled import _slab_blocks_batch, zero_flux_combos
    if not all(x.syms == out_bonds[0].syms for x in out_bonds):
        raise ValueError("all bonds must carry the same symmetries")
    qns = zero_flux_combos(out_bonds)
    if not qns:
        raise ValueError("no valid blocks: no combination of these bonds' sectors has zero flux")

    def structure(a, b):
        ablk, aperm = _common_perm(a)
        bblk, bperm = _common_perm(b)
        sig = (a.dtype, b.dtype, a._qns, b._qns, [x._sshape for x in ablk], [x._sshape for x in bblk],
               tuple(aperm), tuple(bperm))
        return sig, _widen(ablk, dt), aperm, _widen(bblk, dt), bperm

    sig0, ablk0, aperm, bblk0, bperm = structure(a0, b0)
    plan, shapes = _bs_plan(dt, a0, ablk0, aperm, b0, bblk0, bperm, a_pos, b_pos, out_bonds, qns)
    # all outputs in one allocation (one allocator call per batch; the results share its lifetime)
    out_blocks = _slab_blocks_batch(shapes, dt, len(pairs))
    aps, bps, ops, outs = [], [], [], []
    # converted (_widen) or materialised (_common_perm) operand blocks must outlive the
    # launch: only their raw pointers travel in the tables, and the caching allocator would
    # otherwise hand their memory to the next pair's conversion before the kernel runs
    keep = []
    for k, (a, b) in enumerate(pairs):
        if k == 0:
            ablk, bblk, lay = ablk0, bblk0, (a_pos, b_pos, a_free, b_free, out_labels, out_bonds)
        else:
            lay = _pair_layout(a, b)  # the reference's checks, per pair, before any arithmetic
            sig, ablk, _, bblk, _ = structure(a, b)
            if (sig != sig0 or lay[0] != a_pos or lay[1] != b_pos or lay[4] != out_labels
                    or lay[5] != out_bonds):
                raise ValueError(f"contract_batched: pair {k} does not share the block structure of pair 0")
        oblk = out_blocks[k]
        keep.append((ablk, bblk))
        aps.append(dense.block_ptrs(ablk))
        bps.append(dense.block_ptrs(bblk))
        ops.append([x._p0 for x in oblk])
        outs.append(UniTensor._assemble(lay[5], lay[4], len(lay[2]), "", oblk, qns))
    if not plan.execute_batched(aps, bps, ops, dense.stream_handle()):
        _BS_PLANS.clear()
        plan, _ = _bs_plan(dt, a0, ablk0, aperm, b0, bblk0, bperm, a_pos, b_pos, out_bonds, qns)
        if not plan.execute_batched(aps, bps, ops, dense.stream_handle()):
            raise _lib.EngineError("block-sparse plan went stale twice")
    del keep  # the launch is queued on the stream: the allocator reuses these only after it
    _remember_fast(ia0, ib0, plan, (a_pos, b_pos, a_free, b_free, out_labels, out_bonds), shapes, qns, dt)
    return outs


def block_pairs(a, b):
    """Device pairing table of a block-sparse contraction as (i, j, out_idx) rows in
    reference accumulation order (contract.py:148-164): builds (or reuses) the
    structure's device plan -- the pairing kernel -- and reads the table back."""
    a_pos, b_pos, a_free, b_free, out_labels, out_bonds = _pair_layout(a, b)
    dt = _result_dtype(a.dtype, b.dtype)
    ablk, aperm = _common_perm(a)
    bblk, bperm = _common_perm(b)
    ablk, bblk = _widen(ablk, dt), _widen(bblk, dt)
    from .labeled import zero_flux_combos
    qns = zero_flux_combos(out_bonds)
    plan, _ = _bs_plan(dt, a, ablk, aperm, b, bblk, bperm, a_pos, b_pos, out_bonds, qns)
    return plan.pairs(dense.stream_handle())


def _contract_blocks_scalar(a, b, ablk, bblk, a_pos, b_pos, dt):
    """Fully contracted block-sparse pair: sum over matching block pairs in reference
    order, each pair a device dot product (rare path; contract.py:159-166)."""
    by_key = {}
    for j, q in enumerate(b._qns):
        by_key.setdefault(tuple(q[p] for p in b_pos), []).append(j)
    parts = []
    for i, q in enumerate(a._qns):
        for j in by_key.get(tuple(q[p] for p in a_pos), ()):
            A, B = ablk[i], bblk[j]
            out = DenseTensor.empty((), dt)
            _lib.contract_dense(A.data_ptr, dense.dtype_code(A.dtype), A.storage_shape, A.perm,
                                B.data_ptr, dense.dtype_code(B.dtype), B.storage_shape, B.perm,
                                a_pos, b_pos, out.data_ptr, _CPLX_MODE, dense.stream_handle())
            parts.append(out.storage())
    total = DenseTensor.empty((), dt)
    total.storage().zero_()
    for p in parts:  # fixed order, deterministic
        total.storage().add_(p)
    return UniTensor.scalar(total)


# -- multi-tensor ------------------------------------------------------------------------------------
def contract(first, *rest, order=None, optimal=True):
    """contract(a, b) or contract([t1, t2, ...], order=None, optimal=True)."""
    if isinstance(first, UniTensor):
        tensors = [first, *rest]
    else:
        tensors = list(first)
        if rest:
            raise TypeError("pass either several tensors or one list")
    if not tensors:
        raise ValueError("nothing to contract")
    if not all(isinstance(t, UniTensor) for t in tensors):
        raise TypeError("contract expects UniTensors")
    if len(tensors) == 1:
        return tensors[0].clone()
    _reject_hyperedges(tensors)
    if len(tensors) == 2:
        return contract_pair(tensors[0], tensors[1])
    if order is None and not optimal:
        acc = tensors[0]
        for t in tensors[1:]:
            acc = contract_pair(acc, t)
        return acc
    names = [t.name for t in tensors]
    if any(not n for n in names):
        raise ValueError("multi-tensor contraction with an order or the optimal search needs every tensor named")
    if len(set(names)) != len(names):
        raise ValueError(f"tensor names must be distinct, got {names}")
    by_name = dict(zip(names, tensors))
    if order is not None:
        tree = parse_order(order) if isinstance(order, str) else order
        if sorted(tree_leaves(tree)) != sorted(names):
            raise ValueError(f"order {render_order(tree)!r} does not cover exactly the tensors {names}")
    else:
        tree = find_optimal_order({n: t.labels for n, t in by_name.items()}, _label_dims(tensors))
    return execute_tree(tree, by_name)


def execute_tree(tree, by_name):
    if isinstance(tree, str):
        return by_name[tree]
    return contract_pair(execute_tree(tree[0], by_name), execute_tree(tree[1], by_name))


def _reject_hyperedges(tensors):
    counts = {}
    for t in tensors:
        for l in t.labels:
            counts[l] = counts.get(l, 0) + 1
    bad = [l for l, c in counts.items() if c > 2]
    if bad:
        raise ValueError(f"labels {bad} appear on more than two tensors; hyper-edge contraction is not supported")


def _label_dims(tensors):
    dims = {}
    for t in tensors:
        for l, b in zip(t.labels, t.bonds):
            if l in dims and dims[l] != b.dim:
                raise ValueError(f"label {l!r} has inconsistent dimensions ({dims[l]} vs {b.dim})")
            dims[l] = b.dim
    return dims


# -- order search ---------------------------------------------------------------------------------------
def contraction_cost(tree, label_sets, dims):
    """Total multiplication count of executing ``tree`` (step = prod of union of free labels)."""

    def walk(node):
        if isinstance(node, str):
            return 0, list(dict.fromkeys(label_sets[node]))
        c1, f1 = walk(node[0])
        c2, f2 = walk(node[1])
        s1, s2 = set(f1), set(f2)
        union = f1 + [l for l in f2 if l not in s1]
        step = 1
        for l in union:
            step *= dims[l]
        return c1 + c2 + step, [l for l in union if (l in s1) != (l in s2)]

    return walk(tree)[0]


def find_optimal_order(label_sets, dims):
    """Minimal-cost binary tree by subset DP; ties -> smallest rendered string, smaller child left.

    Runs natively (tnb_optimal_order) and falls back to the identical Python DP
    only when a cost exceeds 128 bits or the library is not built.
    """
    names = list(label_sets)
    if not names:
        raise ValueError("empty tensor network")
    if len(names) == 1:
        return names[0]
    if len(names) > 16:
        raise ValueError(f"order search over {len(names)} tensors is not supported (limit 16)")
    try:
        res = _lib.optimal_order(names, [list(label_sets[n]) for n in names], dims)
    except _lib.EngineUnavailable:
        res = None
    if res is not None:
        return parse_order(res[0])
    return _find_optimal_order_py(names, label_sets, dims)


def _find_optimal_order_py(names, label_sets, dims):
    n = len(names)
    full = (1 << n) - 1
    lists = [list(label_sets[nm]) for nm in names]
    free = [frozenset()] * (full + 1)
    for mask in range(1, full + 1):
        cnt = {}
        for i in range(n):
            if mask >> i & 1:
                for l in lists[i]:
                    cnt[l] = cnt.get(l, 0) + 1
        free[mask] = frozenset(l for l, c in cnt.items() if c == 1)

    def pcost(m1, m2):
        c = 1
        for l in free[m1] | free[m2]:
            c *= dims[l]
        return c

    cap = max(1, min(pcost(1 << i, 1 << j) for i in range(n) for j in range(i + 1, n)))
    masks = [m for pc in range(2, n + 1) for m in range(1, full + 1) if bin(m).count("1") == pc]
    while True:
        best = {1 << i: (0, names[i], names[i]) for i in range(n)}
        for mask in masks:
            sub = (mask - 1) & mask
            while sub:
                rest = mask ^ sub
                s1, s2 = (sub, rest) if sub < rest else (rest, sub)
                sub = (sub - 1) & mask
                if s1 not in best or s2 not in best:
                    continue
                c1, t1, r1 = best[s1]
                c2, t2, r2 = best[s2]
                cost = c1 + c2 + pcost(s1, s2)
                if cost > cap:
                    continue
                tree, rendered = (((t1, t2), f"({r1},{r2})") if r1 <= r2 else ((t2, t1), f"({r2},{r1})"))
                cur = best.get(mask)
                if cur is None or (cost, rendered) < (cur[0], cur[2]):
                    best[mask] = (cost, tree, rendered)
        if full in best:
            return best[full][1]
        cap *= 2


def brute_force_order(label_sets, dims):
    """Exhaustive minimum over all binary trees (test helper; small n only)."""
    names = list(label_sets)

    def trees(items):
        if len(items) == 1:
            yield items[0]
            return
        head = items[0]
        for k in range(1, len(items)):
            for left in itertools.combinations(items, k):
                if head not in left:
                    continue
                right = [x for x in items if x not in left]
                if not right:
                    continue
                for lt in trees(list(left)):
                    for rt in trees(right):
                        yield (lt, rt)

    best = None
    for t in trees(names):
        c = contraction_cost(t, label_sets, dims)
        if best is None or c < best[0]:
            best = (c, t)
    return best[1]
