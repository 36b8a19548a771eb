"""ctypes binding of libtnb.so (the C ABI declared in include/tnb.h).

This is the only module that talks to native code. Every compute entry point
needs a CUDA device and the in-tree ``libtnb.so``; there is no CPU fallback:
if either is missing the call raises :class:`EngineUnavailable`.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TNB_LIB_PATH") or os.path.join(_HERE, "libtnb.so")  # override: dev A/B builds

TNB_OK, TNB_EINVAL, TNB_ECUDA, TNB_ENODEV, TNB_ENOMEM, TNB_EUNSUP = 0, 1, 2, 3, 4, 5
TNB_F64, TNB_C128, TNB_I64, TNB_BOOL = 0, 1, 2, 3
CPLX_4M, CPLX_3M = 0, 1

# exported symbols, kept in sync with include/tnb.h (tests check both directions)
EXPORTS = (
    "tnb_version", "tnb_launch_count", "tnb_last_error", "tnb_device_count", "tnb_set_device",
    "tnb_synchronize", "tnb_memcpy2d_async", "tnb_permute", "tnb_contract_dense", "tnb_contract_dense_ld",
    "tnb_zero_flux_blocks", "tnb_bs_contract", "tnb_bs_contract_masked", "tnb_optimal_order",
    "tnb_ktimer_enable", "tnb_ktimer_reset", "tnb_ktimer_read",
    "tnb_bs_plan", "tnb_bs_execute", "tnb_bs_execute_batched", "tnb_bs_plan_pairs", "tnb_copy2d_batched", "tnb_svd_jacobi_batched",
    "tnb_lanczos_work_bytes", "tnb_lanczos_step", "tnb_file_to_device", "tnb_contract_dense_out",
)

# kernel families of the kernel timer (TNB_KF_* in include/tnb.h)
KF_GEMM, KF_GEMM_SKINNY, KF_PERMUTE, KF_BS_GEMM, KF_BS_PAIR, KF_OTHER = 0, 1, 2, 3, 4, 5


class EngineError(RuntimeError):
    """A libtnb call failed (CUDA error, resource limit)."""


class EngineUnavailable(EngineError):
    """No GPU or no libtnb.so: the engine has no CPU fallback."""


_lib = None
_load_error = None

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pi64 = ctypes.POINTER(ctypes.c_int64)


def _declare(lib):
    sig = {
        "tnb_version": ([], ctypes.c_int),
        "tnb_launch_count": ([], ctypes.c_int64),
        "tnb_last_error": ([], ctypes.c_char_p),
        "tnb_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "tnb_set_device": ([ctypes.c_int], ctypes.c_int),
        "tnb_synchronize": ([_p], ctypes.c_int),
        "tnb_memcpy2d_async": ([_p, _i64, _p, _i64, _i64, _i64, ctypes.c_int, _p], ctypes.c_int),
        "tnb_ktimer_enable": ([ctypes.c_int], ctypes.c_int),
        "tnb_ktimer_reset": ([], ctypes.c_int),
        "tnb_ktimer_read": ([ctypes.c_int, _pi64, ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "tnb_permute": ([_p, _p, ctypes.c_int, ctypes.c_int, _pi64, _pi32, _p], ctypes.c_int),
        "tnb_contract_dense": ([_p, ctypes.c_int, ctypes.c_int, _pi64, _pi32,
                                _p, ctypes.c_int, ctypes.c_int, _pi64, _pi32,
                                ctypes.c_int, _pi32, _pi32, _p, ctypes.c_int, _p], ctypes.c_int),
        "tnb_contract_dense_out": ([_p, ctypes.c_int, ctypes.c_int, _pi64, _pi32,
                                    _p, ctypes.c_int, ctypes.c_int, _pi64, _pi32,
                                    ctypes.c_int, _pi32, _pi32, _p, _pi32, ctypes.c_int, _p], ctypes.c_int),
        "tnb_contract_dense_ld": ([_p, ctypes.c_int, ctypes.c_int, _pi64, _pi32,
                                   _p, ctypes.c_int, ctypes.c_int, _pi64, _pi32,
                                   ctypes.c_int, _pi32, _pi32, _p, _i64, ctypes.c_int, _p], ctypes.c_int),
        "tnb_zero_flux_blocks": ([ctypes.c_int, ctypes.c_int, _pi32, _pi32, _pi64, _pi32,
                                  _i64, _pi32, _pi64], ctypes.c_int),
        "tnb_bs_contract": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                             ctypes.c_int, ctypes.c_int,
                             _pi32, _pi64, _pi32, _pi32, _pi64, _pi32,
                             ctypes.c_int, _pi32, _pi32, _pi32, _pi64,
                             _p, _p, _p, _i64, _pi32, _pi64, _p], ctypes.c_int),
        "tnb_bs_contract_masked": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int,
                                    _pi32, _pi64, _pi32, _pi32, _pi64, _pi32,
                                    ctypes.c_int, _pi32, _pi32, _pi32, _pi64,
                                    _p, _p, _p, _i64, _p, _i64, _pi32, _pi64, _p], ctypes.c_int),
        "tnb_bs_plan": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                         _pi32, _pi64, _pi32, _pi32, _pi64, _pi32,
                         ctypes.c_int, _pi32, _pi32, _pi32, _pi64, _i64, _p, _pi64, _pi64, _p], ctypes.c_int),
        "tnb_bs_execute": ([_i64, _p, _p, _p, _p], ctypes.c_int),
        "tnb_bs_execute_batched": ([_i64, _i64, _p, _p, _p, _p], ctypes.c_int),
        "tnb_bs_plan_pairs": ([_i64, _i64, _pi32, _pi64, _p], ctypes.c_int),
        "tnb_copy2d_batched": ([_p, _p, _i64, _p, _p], ctypes.c_int),
        "tnb_file_to_device": ([ctypes.c_int, _i64, _i64, _p, _p, _i64, ctypes.c_int, _p], ctypes.c_int),
        "tnb_lanczos_work_bytes": ([ctypes.c_int, _i64], _i64),
        "tnb_lanczos_step": ([ctypes.c_int, _p, _i64, ctypes.c_int, _p, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
        "tnb_svd_jacobi_batched": ([ctypes.c_int, ctypes.c_int, _p, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_double, _p], ctypes.c_int),
        "tnb_optimal_order": ([ctypes.c_int, ctypes.c_char_p, _pi32, _pi32, _pi64,
                               ctypes.c_char_p, _i64, ctypes.c_char_p], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """The loaded library (raises EngineUnavailable if it is not built)."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise EngineUnavailable(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = (f"{LIB_PATH} is not built; run `python -m paper_2401_01921_b200._build` "
                       "(the engine has no CPU fallback)")
        raise EngineUnavailable(_load_error)
    try:
        handle = ctypes.CDLL(LIB_PATH)
        _declare(handle)
    except OSError as e:
        _load_error = f"cannot load {LIB_PATH}: {e}"
        raise EngineUnavailable(_load_error) from e
    _lib = handle
    return _lib


def launch_count():
    """Number of kernels libtnb has launched in this process."""
    return int(lib().tnb_launch_count())


def ktimer_enable(on=True):
    """Record a CUDA event pair around every libtnb kernel launch (outside graph capture)."""
    check(lib().tnb_ktimer_enable(1 if on else 0), "ktimer_enable")


def ktimer_reset():
    check(lib().tnb_ktimer_reset(), "ktimer_reset")


def ktimer_read(family):
    """(launches, device ms, algorithmic work) of one kernel family since the last reset."""
    n, ms, w = ctypes.c_int64(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
    check(lib().tnb_ktimer_read(int(family), ctypes.byref(n), ctypes.byref(ms), ctypes.byref(w)), "ktimer_read")
    return int(n.value), float(ms.value), float(w.value)


def memcpy2d_async(dst, dpitch, src, spitch, width, height, kind, stream):
    check(lib().tnb_memcpy2d_async(dst, int(dpitch), src, int(spitch), int(width), int(height), int(kind), stream),
          "memcpy2d_async")


def last_error():
    return lib().tnb_last_error().decode(errors="replace")


def check(rc, what):
    if rc == TNB_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == TNB_ENODEV:
        raise EngineUnavailable(msg)
    if rc == TNB_EINVAL:
        raise ValueError(msg)
    if rc == TNB_EUNSUP:
        raise TypeError(msg)
    raise EngineError(msg)


def device_count():
    n = ctypes.c_int(0)
    check(lib().tnb_device_count(ctypes.byref(n)), "device_count")
    return n.value


def _arr64(seq):
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.int64))
    return a, a.ctypes.data_as(_pi64)


def _arr32(seq):
    a = np.ascontiguousarray(np.asarray(seq, dtype=np.int32))
    return a, a.ctypes.data_as(_pi32)


def permute(src_ptr, dst_ptr, elem_size, shape, perm, stream):
    """dst = ascontiguousarray(src.reshape(shape).transpose(perm)) on the GPU."""
    s, sp = _arr64(shape)
    p, pp = _arr32(perm)
    check(lib().tnb_permute(src_ptr, dst_ptr, elem_size, len(shape), sp, pp, stream), "permute")


_DENSE_ARGS = {}


def dense_args(a_shape, a_perm, b_shape, b_perm, a_axes, b_axes):
    """Marshalled descriptor arrays of a dense contraction: (keep-alive arrays, pointers)."""
    arrs = [_arr64(a_shape), _arr32(a_perm), _arr64(b_shape), _arr32(b_perm), _arr32(a_axes), _arr32(b_axes)]
    return arrs, [p for _, p in arrs]


_ORDER_ARGS = {}  # marshalled output orders (tuple -> (array, pointer))


def contract_dense(a_ptr, a_dt, a_shape, a_perm, b_ptr, b_dt, b_shape, b_perm,
                   a_axes, b_axes, out_ptr, cplx_mode, stream, out_ld=0, out_order=None):
    # the integer descriptor arrays of a contraction shape are marshalled once and reused
    # (a Network relaunched on same-shape operands re-marshals nothing)
    key = (tuple(a_shape), tuple(a_perm), tuple(b_shape), tuple(b_perm), tuple(a_axes), tuple(b_axes))
    args = _DENSE_ARGS.get(key)
    if args is None:
        args = dense_args(a_shape, a_perm, b_shape, b_perm, a_axes, b_axes)
        if len(_DENSE_ARGS) >= 4096:
            _DENSE_ARGS.clear()
        _DENSE_ARGS[key] = args
    psa, ppa, psb, ppb, pxa, pxb = args[1]
    if out_order is not None:
        oo = _ORDER_ARGS.get(out_order)
        if oo is None:
            if len(_ORDER_ARGS) >= 4096:
                _ORDER_ARGS.clear()
            oo = _ORDER_ARGS[out_order] = _arr32(out_order)
        check(lib().tnb_contract_dense_out(a_ptr, a_dt, len(a_shape), psa, ppa,
                                           b_ptr, b_dt, len(b_shape), psb, ppb,
                                           len(a_axes), pxa, pxb, out_ptr, oo[1], cplx_mode, stream),
              "contract_dense_out")
        return
    if out_ld:
        check(lib().tnb_contract_dense_ld(a_ptr, a_dt, len(a_shape), psa, ppa,
                                          b_ptr, b_dt, len(b_shape), psb, ppb,
                                          len(a_axes), pxa, pxb, out_ptr, int(out_ld), cplx_mode, stream),
              "contract_dense_ld")
        return
    check(lib().tnb_contract_dense(a_ptr, a_dt, len(a_shape), psa, ppa,
                                   b_ptr, b_dt, len(b_shape), psb, ppb,
                                   len(a_axes), pxa, pxb, out_ptr, cplx_mode, stream),
          "contract_dense")


def zero_flux_blocks(nsec, btype, charges, sym_n):
    """Row-major zero-flux sector tuples (host C++; unitensor.py:31-45)."""
    L = lib()
    ns, pns = _arr32(nsec)
    bt, pbt = _arr32(btype)
    ch, pch = _arr64(charges)
    sn, psn = _arr32(sym_n)
    total = 1
    for n in nsec:
        total *= int(n)
    cap = total
    out = np.empty((max(cap, 1), len(nsec)), dtype=np.int32)
    count = ctypes.c_int64(0)
    check(L.tnb_zero_flux_blocks(len(nsec), len(sym_n), pns, pbt, pch, psn, cap,
                                 out.ctypes.data_as(_pi32), ctypes.byref(count)),
          "zero_flux_blocks")
    return out[:count.value]


BS_PANEL_ROWS = 64  # TNB_BS_PANEL_ROWS


def bs_contract(dtype, a_qn, a_shapes, a_perm, b_qn, b_shapes, b_perm, a_axes, b_axes,
                out_qn, out_shapes, a_ptrs, b_ptrs, out_ptrs, stream, want_pairs=False, panel_mask=None):
    na, nb, nout = len(a_ptrs), len(b_ptrs), len(out_ptrs)
    ra, rb = len(a_perm), len(b_perm)
    aq, paq = _arr32(np.asarray(a_qn, dtype=np.int32).reshape(-1))
    ash, pash = _arr64(np.asarray(a_shapes, dtype=np.int64).reshape(-1))
    ap, pap = _arr32(a_perm)
    bq, pbq = _arr32(np.asarray(b_qn, dtype=np.int32).reshape(-1))
    bsh, pbsh = _arr64(np.asarray(b_shapes, dtype=np.int64).reshape(-1))
    bp, pbp = _arr32(b_perm)
    xa, pxa = _arr32(a_axes)
    xb, pxb = _arr32(b_axes)
    oq, poq = _arr32(np.asarray(out_qn, dtype=np.int32).reshape(-1))
    osh, posh = _arr64(np.asarray(out_shapes, dtype=np.int64).reshape(-1))
    aptr = (ctypes.c_void_p * max(na, 1))(*a_ptrs)
    bptr = (ctypes.c_void_p * max(nb, 1))(*b_ptrs)
    optr = (ctypes.c_void_p * max(nout, 1))(*out_ptrs)
    npairs = ctypes.c_int64(0)
    pairs = None
    cap = 0
    if want_pairs:
        cap = max(na * nb, 1)
        pairs = np.zeros((cap, 3), dtype=np.int32)
    mask = None
    if panel_mask is not None:
        mask = np.ascontiguousarray(np.asarray(panel_mask, dtype=np.uint8))
    check(lib().tnb_bs_contract_masked(dtype, na, nb, nout, ra, rb, paq, pash, pap, pbq, pbsh, pbp,
                                       len(a_axes), pxa, pxb, poq, posh,
                                       ctypes.cast(aptr, _p), ctypes.cast(bptr, _p), ctypes.cast(optr, _p),
                                       0 if mask is None else len(mask),
                                       None if mask is None else mask.ctypes.data_as(_p),
                                       cap, pairs.ctypes.data_as(_pi32) if want_pairs else None,
                                       ctypes.byref(npairs) if want_pairs else None, stream),
          "bs_contract")
    if want_pairs:
        return pairs[:npairs.value].copy()
    return None


class BsPlan:
    """Handle of a device-resident block-sparse plan (tnb_bs_plan): structure-only
    metadata was uploaded and paired once; ``execute`` launches one grouped GEMM."""

    __slots__ = ("id", "npairs", "na", "nb", "nout", "_aptr", "_bptr", "_optr")

    def __init__(self, plan_id, npairs, na, nb, nout):
        self.id, self.npairs, self.na, self.nb, self.nout = plan_id, npairs, na, nb, nout
        self._aptr = (ctypes.c_void_p * max(na, 1))()
        self._bptr = (ctypes.c_void_p * max(nb, 1))()
        self._optr = (ctypes.c_void_p * max(nout, 1))()

    def execute(self, a_ptrs, b_ptrs, out_ptrs, stream):
        """Returns False if the plan went stale (cache flushed): the caller re-plans."""
        self._aptr[:len(a_ptrs)] = a_ptrs
        self._bptr[:len(b_ptrs)] = b_ptrs
        self._optr[:len(out_ptrs)] = out_ptrs
        rc = lib().tnb_bs_execute(self.id, self._aptr, self._bptr, self._optr, stream)
        if rc == TNB_EINVAL and "stale" in last_error():
            return False
        check(rc, "bs_execute")
        return True

    def execute_batched(self, a_ptrs, b_ptrs, out_ptrs, stream):
        """nbatch contractions of this structure in one launch; a_ptrs is [nbatch][na] etc.
        (nested sequences of device addresses). Returns False if the plan went stale."""
        nbatch = len(out_ptrs)
        a = np.ascontiguousarray(np.asarray(a_ptrs, dtype=np.uint64).reshape(nbatch, self.na))
        b = np.ascontiguousarray(np.asarray(b_ptrs, dtype=np.uint64).reshape(nbatch, self.nb))
        o = np.ascontiguousarray(np.asarray(out_ptrs, dtype=np.uint64).reshape(nbatch, self.nout))
        vp = ctypes.c_void_p
        rc = lib().tnb_bs_execute_batched(self.id, nbatch, a.ctypes.data_as(vp), b.ctypes.data_as(vp),
                                          o.ctypes.data_as(vp), stream)
        if rc == TNB_EINVAL and "stale" in last_error():
            return False
        check(rc, "bs_execute_batched")
        return True

    def pairs(self, stream):
        cap = max(self.npairs, 1)
        out = np.zeros((cap, 3), dtype=np.int32)
        n = ctypes.c_int64(0)
        check(lib().tnb_bs_plan_pairs(self.id, cap, out.ctypes.data_as(_pi32), ctypes.byref(n), stream),
              "bs_plan_pairs")
        return out[:n.value].copy()


def bs_plan(dtype, a_qn, a_shapes, a_perm, b_qn, b_shapes, b_perm, a_axes, b_axes, out_qn, out_shapes,
            stream, panel_mask=None):
    na, nb, nout = len(a_qn), len(b_qn), len(out_qn)
    ra, rb = len(a_perm), len(b_perm)
    aq, paq = _arr32(np.asarray(a_qn, dtype=np.int32).reshape(-1))
    ash, pash = _arr64(np.asarray(a_shapes, dtype=np.int64).reshape(-1))
    ap, pap = _arr32(a_perm)
    bq, pbq = _arr32(np.asarray(b_qn, dtype=np.int32).reshape(-1))
    bsh, pbsh = _arr64(np.asarray(b_shapes, dtype=np.int64).reshape(-1))
    bp, pbp = _arr32(b_perm)
    xa, pxa = _arr32(a_axes)
    xb, pxb = _arr32(b_axes)
    oq, poq = _arr32(np.asarray(out_qn, dtype=np.int32).reshape(-1))
    osh, posh = _arr64(np.asarray(out_shapes, dtype=np.int64).reshape(-1))
    mask = None
    if panel_mask is not None:
        mask = np.ascontiguousarray(np.asarray(panel_mask, dtype=np.uint8))
    pid, npairs = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib().tnb_bs_plan(dtype, na, nb, nout, ra, rb, paq, pash, pap, pbq, pbsh, pbp,
                            len(a_axes), pxa, pxb, poq, posh,
                            0 if mask is None else len(mask), None if mask is None else mask.ctypes.data_as(_p),
                            ctypes.byref(pid), ctypes.byref(npairs), stream), "bs_plan")
    return BsPlan(pid.value, npairs.value, na, nb, nout)


COPY2D_DTYPE = np.dtype([("src_off", "<i8"), ("dst_off", "<i8"), ("rows", "<i8"), ("row_bytes", "<i8"),
                         ("src_pitch", "<i8"), ("dst_pitch", "<i8")])  # TnbCopy2D


def lanczos_work_bytes(r_max, n):
    return int(lib().tnb_lanczos_work_bytes(int(r_max), int(n)))


def lanczos_step(dtype, q_ptr, ldq, r, w_ptr, n, q_next_ptr, alpha_ptr, beta_ptr, work_ptr, stream):
    """tnb_lanczos_step: reorthogonalise w against r basis rows, alpha / beta to device memory."""
    check(lib().tnb_lanczos_step(dtype, q_ptr, ldq, r, w_ptr, n, q_next_ptr, alpha_ptr, beta_ptr, work_ptr, stream),
          "lanczos_step")


def file_to_device(fd, offset, nbytes, pinned_ptr, dst_ptr, chunk, nthreads, stream):
    """tnb_file_to_device: pooled pread of a file range into pinned memory, each piece copied
    to the device as it lands (returns once every copy is queued on `stream`)."""
    check(lib().tnb_file_to_device(int(fd), int(offset), int(nbytes), pinned_ptr, dst_ptr, int(chunk), int(nthreads),
                                   stream), "file_to_device")


def copy2d_batched(src_ptr, dst_ptr, segs, stream):
    """One launch of tnb_copy2d_batched; `segs` is a COPY2D_DTYPE structured array."""
    segs = np.ascontiguousarray(segs, dtype=COPY2D_DTYPE)
    check(lib().tnb_copy2d_batched(src_ptr, dst_ptr, len(segs), segs.ctypes.data_as(_p) if len(segs) else None,
                                   stream), "copy2d_batched")


SVD_SECTOR_DTYPE = np.dtype([("a", "<u8"), ("b", "<u8"), ("q", "<u8"), ("u", "<u8"), ("s", "<u8"), ("vh", "<u8"),
                             ("status", "<u8"), ("m", "<i8"), ("n", "<i8")])  # TnbSvdSector


def svd_jacobi_batched(sectors, stream, max_sweeps=30, tol=2.0, rank_tol=1e-13, dtype=TNB_F64):
    """One launch of tnb_svd_jacobi_batched over a SVD_SECTOR_DTYPE structured array."""
    secs = np.ascontiguousarray(sectors, dtype=SVD_SECTOR_DTYPE)
    check(lib().tnb_svd_jacobi_batched(int(dtype), len(secs), secs.ctypes.data_as(_p) if len(secs) else None,
                                       int(max_sweeps), float(tol), float(rank_tol), stream),
          "svd_jacobi_batched")


def optimal_order(names, label_lists, dims):
    """Native DP (contract.py:271-343); returns (rendered order, cost) or None on overflow."""
    ids = {}
    flat, nlab = [], []
    for labels in label_lists:
        nlab.append(len(labels))
        for l in labels:
            if l not in ids:
                ids[l] = len(ids)
            flat.append(ids[l])
    dimv = [0] * len(ids)
    for l, i in ids.items():
        dimv[i] = int(dims[l])
    if any(d >= 2 ** 63 for d in dimv):
        return None
    blob = b"".join(n.encode() + b"\0" for n in names)
    nl, pnl = _arr32(nlab)
    fl, pfl = _arr32(flat if flat else [0])
    dv, pdv = _arr64(dimv if dimv else [1])
    cap = 64 + 4 * sum(len(n) + 3 for n in names)
    out = ctypes.create_string_buffer(cap)
    cost = ctypes.create_string_buffer(64)
    rc = lib().tnb_optimal_order(len(names), blob, pnl, pfl, pdv, out, cap, cost)
    if rc == TNB_EUNSUP:
        return None
    check(rc, "optimal_order")
    return out.value.decode(), int(cost.value.decode())
