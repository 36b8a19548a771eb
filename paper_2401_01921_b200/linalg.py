"""Block-sparse matricisation + per-sector SVD / truncated SVD in HBM.

Same contract as the reference (pkg/src/tnkit/linalg.py):

* ``_matricize`` (linalg.py:70-142): the first ``rowrank`` bonds form the row; blocks
  are grouped by the total charge of their row indices (IN adds q, OUT adds -q),
  sectors in order of first appearance in block order, row / column parts of a sector
  in order of first appearance; dense tensors are one sector.
* ``svd`` (linalg.py:246-268): per-sector thin SVD, singular values descending;
  ``S`` is the square diagonal matrix on (``_aux_L``, ``_aux_R``), ``U`` inherits the
  row labels + ``_aux_L`` (new OUT bond), ``Vdag`` gets ``_aux_R`` (new IN bond) + the
  column labels; the new bond has one sector per surviving charge.
* ``svd_truncate`` (linalg.py:271-341): global ranking of all singular values
  (descending value, ties by sector index then position), ``err`` floor,
  ``min_blockdim`` reservations, "keep the single largest" rescue, ``return_err``.

B200 path: blocks -> sector matrices is ONE ``tnb_copy2d_batched`` launch into a
sector slab laid out by matrix shape, so every group of equal-shape sectors is already a
``[batch, m, n]`` array; all sectors (float64 or complex128) are factorised by ONE launch of
the engine's batched one-sided Jacobi kernel (``tnb_svd_jacobi_batched``, csrc/svd.cu: a
thread-block cluster per sector, all sectors concurrently); any sector the kernel flags
(not converged / rank deficient) is refactorised by the library (``torch.linalg.svd``,
cuSOLVER). The factors U / S / Vdag are scattered into their block
slabs by one ``tnb_copy2d_batched`` launch each. Only the singular values (for the
truncation ranking) and the per-group status words cross to the host.
"""
import numpy as np
import torch

from . import _lib, dense
from .charges import IN, OUT, REGULAR, Bond
from .dense import DenseTensor
from .labeled import UniTensor


def _aux_labels(labels):
    out = []
    for base in ("_aux_L", "_aux_R"):
        name, k = base, 0
        while name in labels or name in out:
            name = f"{base}{k}"
            k += 1
        out.append(name)
    return out


class _Sector:
    __slots__ = ("charge", "rows", "cols", "m", "n", "off", "group", "gidx")

    def __init__(self, charge):
        self.charge = charge
        self.rows = []  # (qn part, offset, size)
        self.cols = []


class _Matricized:
    """Host bookkeeping (reference order) + the device sector slab."""

    def __init__(self, ut):
        r = ut.rowrank
        if not 0 < r < ut.rank:
            raise ValueError(f"matrix routines need 0 < rowrank < rank, got rowrank={r} for rank {ut.rank}")
        self.ut = ut
        self.rowrank = r
        self.row_bonds, self.col_bonds = ut.bonds[:r], ut.bonds[r:]
        self.row_labels, self.col_labels = ut.labels[:r], ut.labels[r:]
        self.aux_l, self.aux_r = _aux_labels(ut.labels)
        self.dt = ut.dtype
        if ut.dtype not in (dense.Float64, dense.Complex128):
            raise TypeError(f"svd of {ut.dtype} is not supported on the GPU engine (float64 / complex128 only)")
        if not ut.is_sym:
            sec = _Sector(None)
            rdim = int(np.prod([b.dim for b in self.row_bonds]))
            cdim = int(np.prod([b.dim for b in self.col_bonds]))
            sec.rows, sec.cols = [(None, 0, rdim)], [(None, 0, cdim)]
            self.sectors = [sec]
            self.placed = [(sec, None, None)]
        else:
            syms = ut.bonds[0].syms
            groups, order, placed = {}, [], []
            for i in range(ut.nblocks):
                qn = ut.block_qn_indices(i)
                charge = _row_charge(self.row_bonds, qn[:r], syms)
                if charge not in groups:
                    groups[charge] = _Sector(charge)
                    order.append(charge)
                placed.append((groups[charge], qn[:r], qn[r:]))
            for sec, row_qn, col_qn in placed:
                if not any(rq == row_qn for rq, _, _ in sec.rows):
                    size = int(np.prod([b.sectors[k][1] for b, k in zip(self.row_bonds, row_qn)]))
                    off = sec.rows[-1][1] + sec.rows[-1][2] if sec.rows else 0
                    sec.rows.append((row_qn, off, size))
                if not any(cq == col_qn for cq, _, _ in sec.cols):
                    size = int(np.prod([b.sectors[k][1] for b, k in zip(self.col_bonds, col_qn)]))
                    off = sec.cols[-1][1] + sec.cols[-1][2] if sec.cols else 0
                    sec.cols.append((col_qn, off, size))
            self.sectors = [groups[c] for c in order]
            self.placed = placed
        for sec in self.sectors:
            sec.m = sec.rows[-1][1] + sec.rows[-1][2]
            sec.n = sec.cols[-1][1] + sec.cols[-1][2]
        self._to_device()

    def directed(self):
        return any(b.btype != REGULAR for b in self.ut.bonds)

    def _to_device(self):
        """Sector slab grouped by matrix shape; one copy2d launch fills it."""
        shapes = []
        for sec in self.sectors:
            if (sec.m, sec.n) not in shapes:
                shapes.append((sec.m, sec.n))
        self.groups = []  # (m, n, [sectors]) with a [b, m, n] device view each
        total = 0
        for shp in shapes:
            members = [s for s in self.sectors if (s.m, s.n) == shp]
            for k, s in enumerate(members):
                s.off = total + k * shp[0] * shp[1]
                s.group, s.gidx = len(self.groups), k
            self.groups.append([shp[0], shp[1], members, total])
            total += len(members) * shp[0] * shp[1]
        tdt = dense._TORCH[self.dt]
        self.slab = torch.empty(max(total, 1), dtype=tdt, device=dense.device())
        es = self.dt.itemsize
        blocks = [b.contiguous() for b in self.ut.get_blocks_()]  # tnb_permute for lazy views
        ptrs = [b.data_ptr for b in blocks]
        base = min(ptrs)
        segs = np.zeros(len(blocks), dtype=_lib.COPY2D_DTYPE)
        for k, ((sec, row_qn, col_qn), p) in enumerate(zip(self.placed, ptrs)):
            if sec.charge is None:
                ro, rs, co, cs = 0, sec.m, 0, sec.n
            else:
                _, ro, rs = next(x for x in sec.rows if x[0] == row_qn)
                _, co, cs = next(x for x in sec.cols if x[0] == col_qn)
            segs[k] = (p - base, (sec.off + ro * sec.n + co) * es, rs, cs * es, cs * es, sec.n * es)
        if self.ut.is_sym:
            self.slab.zero_()  # (every (row, col) part of a sector is a block; kept for safety)
        _lib.copy2d_batched(base, self.slab.data_ptr(), segs, dense.stream_handle())
        for g in self.groups:
            m, n, members, off = g
            g.append(self.slab[off:off + len(members) * m * n].view(len(members), m, n))


def _row_charge(row_bonds, row_qn, syms):
    from .charges import combine_qnums, identity_qnum, reverse_qnums
    charge = identity_qnum(syms)
    for b, k in zip(row_bonds, row_qn):
        q = b.sectors[k][0]
        if b.btype == OUT:
            q = reverse_qnums(q, syms)
        charge = combine_qnums(charge, q, syms)
    return charge


# sector matrices go through the engine's batched Jacobi kernel (tnb_svd_jacobi_batched: one
# thread-block cluster per sector, all sectors in one launch; rank-deficient sectors are
# completed in the kernel). A sector the kernel reports as not converged within its sweep
# budget (never observed) is refactorised by the library; "library" forces the latter for
# everything (A/B measurements only).
SVD_BACKEND = "jacobi"


def _library_svd(view):
    u, s, vh = torch.linalg.svd(view, full_matrices=False)
    # cuSOLVER hands back column-major factors as strided (and, for complex Vh, lazily
    # conjugated) views; the scatters read plain row-major memory
    return u.resolve_conj().contiguous(), s.contiguous(), vh.resolve_conj().contiguous()


def _transpose(batch):
    """[b, r, c] -> [b, c, r] through tnb_permute (contiguous device tensors)."""
    b, r, c = batch.shape
    out = torch.empty((b, c, r), dtype=batch.dtype, device=batch.device)
    if batch.numel():
        _lib.permute(batch.data_ptr(), out.data_ptr(), batch.element_size(), [b, r, c], [0, 2, 1],
                     dense.stream_handle())
    return out


def _factorise(mz):
    """Thin SVD of every shape group: (U [b,m,k], S [b,k], Vh [b,k,n]) device tensors."""
    if SVD_BACKEND != "jacobi":
        return [_library_svd(g[4]) for g in mz.groups]
    tdt = dense._TORCH[mz.dt]
    es = mz.dt.itemsize
    jobs, recs = [], []
    for gi, (m, n, members, off, view) in enumerate(mz.groups):
        tall = m > n
        a = _transpose(view) if tall else view  # rows to orthogonalise: the shorter side
        b, r, c = a.shape
        dev = a.device
        u = torch.empty((b, r, r), dtype=tdt, device=dev)
        sv = torch.empty((b, r), dtype=torch.float64, device=dev)
        vh = torch.empty((b, r, c), dtype=tdt, device=dev)
        # workspaces: float64 rows padded to even length (16-byte rows in the kernel)
        lw = c + (c & 1) if es == 8 else c
        lq = r + (r & 1) if es == 8 else r
        q = torch.empty((b, r, lq), dtype=tdt, device=dev)
        w = torch.empty((b, r, lw), dtype=tdt, device=dev)  # rotated rows (a stays intact)
        st = torch.zeros(b, dtype=torch.int32, device=dev)
        for k in range(b):
            jobs.append((a.data_ptr() + k * r * c * es, w.data_ptr() + k * r * lw * es, q.data_ptr() + k * r * lq * es,
                         u.data_ptr() + k * r * r * es, sv.data_ptr() + k * r * 8, vh.data_ptr() + k * r * c * es,
                         st.data_ptr() + 4 * k, r, c))
        recs.append((tall, u, sv, vh, q, st, (a, w)))
    # largest sectors first: clusters are scheduled in task order and only ~9 16-CTA clusters
    # are resident at once, so the critical (largest) sector must not wait behind small ones
    jobs.sort(key=lambda j: -(j[7] * j[7] * j[8]))
    _lib.svd_jacobi_batched(np.array(jobs, dtype=_lib.SVD_SECTOR_DTYPE), dense.stream_handle(),
                            dtype=dense.dtype_code(mz.dt))
    out = []
    for (m, n, members, off, view), (tall, u, sv, vh, q, st, a) in zip(mz.groups, recs):
        if bool((st <= 0).any()):  # (one small device->host read per group)
            out.append(_library_svd(view))
            continue
        if tall:  # A^T = U' S V'^H  ->  A = conj(V') S U'^T: U = conj(Vh')^T, Vh = conj(U')^T
            u, vh = _transpose(vh), _transpose(u)
            if mz.dt == dense.Complex128:
                u, vh = u.conj_physical_(), vh.conj_physical_()
        out.append((u, sv, vh))
    return out


def _new_bond(mz, keeps, btype):
    if mz.ut.is_sym:
        sectors = [(s.charge, k) for s, k in zip(mz.sectors, keeps) if k > 0]
        return Bond(btype=btype, sectors=sectors, syms=mz.ut.bonds[0].syms)
    if mz.directed():
        return Bond(int(keeps[0]), btype)
    return Bond(int(keeps[0]))


def _assemble_dense(bonds, labels, rowrank, name, arr_shape, dt):
    t = DenseTensor.empty(arr_shape, dt)
    return UniTensor._assemble(bonds, labels, rowrank, name, [t], None)


def _scatter(dst_blocks, parts, stream):
    """parts: list of (dst block index, src tensor, src elem offset, rows, row_elems, src pitch, dst pitch)."""
    if not parts:
        return
    es = dst_blocks[0].itemsize
    dptrs = [b.data_ptr for b in dst_blocks]
    dbase = min(dptrs)
    srcs = [p[1].data_ptr() + p[2] * es for p in parts]
    sbase = min(srcs)
    segs = np.zeros(len(parts), dtype=_lib.COPY2D_DTYPE)
    for k, ((bi, _, _, rows, relems, sp, dp), sp_) in enumerate(zip(parts, srcs)):
        segs[k] = (sp_ - sbase, dptrs[bi] - dbase, rows, relems * es, sp * es, dp * es)
    _lib.copy2d_batched(sbase, dbase, segs, stream)


def _build(mz, facs, keeps, want_uv):
    st = dense.stream_handle()
    dt = mz.dt
    # S: float64 square diagonal on the new bond (IN, OUT)
    sb = [_new_bond(mz, keeps, IN), _new_bond(mz, keeps, OUT)]
    if mz.ut.is_sym:
        s_t = UniTensor(sb, labels=[mz.aux_l, mz.aux_r], dtype=dense.Float64, rowrank=1, name="S")
    else:
        s_t = _assemble_dense(sb, [mz.aux_l, mz.aux_r], 1, "S", (keeps[0], keeps[0]), dense.Float64)
        s_t.get_block_().storage().zero_()
    parts, new_idx = [], 0
    for sec, keep in zip(mz.sectors, keeps):
        if keep == 0:
            continue
        s = facs[sec.group][1][sec.gidx]
        bi = s_t._block_pos(([new_idx, new_idx],)) if mz.ut.is_sym else 0
        parts.append((bi, s, 0, keep, 1, 1, keep + 1))
        new_idx += 1
    _scatter(s_t.get_blocks_(), parts, st)
    if not want_uv:
        return s_t, None, None
    # U: row bonds + new OUT bond, rows of each sector's U[:, :keep]
    ub = mz.row_bonds + [_new_bond(mz, keeps, OUT)]
    ul = mz.row_labels + [mz.aux_l]
    if mz.ut.is_sym:
        u_t = UniTensor(ub, labels=ul, dtype=dt, rowrank=len(mz.row_bonds), name="U")
    else:
        u_t = _assemble_dense(ub, ul, len(mz.row_bonds), "U", [b.dim for b in mz.row_bonds] + [keeps[0]], dt)
    vb = [_new_bond(mz, keeps, IN)] + mz.col_bonds
    vl = [mz.aux_r] + mz.col_labels
    if mz.ut.is_sym:
        v_t = UniTensor(vb, labels=vl, dtype=dt, rowrank=1, name="Vdag")
    else:
        v_t = _assemble_dense(vb, vl, 1, "Vdag", [keeps[0]] + [b.dim for b in mz.col_bonds], dt)
    uparts, vparts, new_idx = [], [], 0
    for sec, keep in zip(mz.sectors, keeps):
        if keep == 0:
            continue
        u, _, vh = facs[sec.group]
        ku = u.shape[-1]
        u_s, vh_s = u[sec.gidx], vh[sec.gidx]  # [m, k], [k, n] (contiguous slices of the batch)
        for row_qn, off, size in sec.rows:
            bi = u_t._block_pos((list(row_qn) + [new_idx],)) if mz.ut.is_sym else 0
            uparts.append((bi, u_s, off * ku, size, keep, ku, keep))
        for col_qn, off, size in sec.cols:
            bi = v_t._block_pos(([new_idx] + list(col_qn),)) if mz.ut.is_sym else 0
            vparts.append((bi, vh_s, off, keep, size, sec.n, size))
        new_idx += 1
    # (symmetric U / Vdag come zero-filled: blocks outside the kept sectors stay zero)
    _scatter(u_t.get_blocks_(), uparts, st)
    _scatter(v_t.get_blocks_(), vparts, st)
    return s_t, u_t, v_t


def svd(ut, compute_uv=True):
    """Singular value decomposition through the rowrank split (linalg.py:246-268).
    Returns ``(S, U, Vdag)``, or ``S`` alone with ``compute_uv=False``."""
    mz = _Matricized(ut)
    facs = _factorise(mz)
    keeps = [min(sec.m, sec.n) for sec in mz.sectors]
    s_t, u_t, v_t = _build(mz, facs, keeps, compute_uv)
    return (s_t, u_t, v_t) if compute_uv else s_t


def svd_truncate(ut, keepdim, err=0.0, return_err=0, min_blockdim=None):
    """SVD + global truncation (linalg.py:271-341): keep the ``keepdim`` largest singular
    values that are >= ``err`` (ties: sector index, then position); ``min_blockdim``
    reserves per-sector minima; ``return_err`` 1 / 2 appends the largest / all discarded."""
    if keepdim < 1:
        raise ValueError(f"keepdim must be >= 1, got {keepdim}")
    mz = _Matricized(ut)
    nsec = len(mz.sectors)
    if min_blockdim is not None:
        if not ut.is_sym:
            raise ValueError("min_blockdim applies to symmetric tensors only")
        if len(min_blockdim) != nsec:
            raise ValueError(f"min_blockdim needs one entry per block ({nsec}), got {len(min_blockdim)}")
    if return_err not in (0, 1, 2):
        raise ValueError(f"return_err must be 0, 1 or 2, got {return_err}")
    facs = _factorise(mz)
    host_s = [g[1].cpu().numpy() for g in facs]  # the only device->host traffic: singular values
    ss = [host_s[sec.group][sec.gidx] for sec in mz.sectors]
    if min_blockdim is not None:
        keeps = [min(int(mb), len(s)) for mb, s in zip(min_blockdim, ss)]
    else:
        keeps = [0] * nsec
    slots = keepdim - sum(keeps)
    if slots > 0:
        ranked = sorted((-s[pos], i, pos) for i, s in enumerate(ss)
                        for pos in range(keeps[i], len(s)) if s[pos] >= err)
        for _, i, _ in ranked[:slots]:
            keeps[i] += 1
    if sum(keeps) == 0:
        keeps[max(range(nsec), key=lambda i: ss[i][0])] = 1
    discarded = sorted((s[pos] for i, s in enumerate(ss) for pos in range(keeps[i], len(s))), reverse=True)
    s_t, u_t, v_t = _build(mz, facs, keeps, True)
    if return_err == 0:
        return s_t, u_t, v_t
    if return_err == 1:
        vals = np.array([discarded[0] if discarded else 0.0])
    else:
        vals = np.array(discarded) if discarded else np.zeros(1)
    e_t = UniTensor(DenseTensor(vals), labels=["s_err"])
    return s_t, u_t, v_t, e_t


# Cytnx spellings
Svd = svd
Svd_truncate = svd_truncate
