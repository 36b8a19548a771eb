"""The reference-side binding: run `tnkit` (the reference package) with its hot path on the
B200 engine (libtnb.so through the engine's ctypes layer).

This is the module a tnkit maintainer would add as ``tnkit/_b200.py``. ``install(tnkit)``
patches the seams SURVEY.md section 8(b) names, in every module that binds them by name:

* ``contract_pair`` -- tnkit/contract.py:100-167 (dense ``np.tensordot`` at :127-128 and
  the block loop at :137-167), re-bound in tnkit.contract (also used by ``contract`` /
  ``execute_tree``, contract.py:197-225), tnkit.network (network.py:31, ``_execute``
  network.py:301-304), tnkit.dmrg (dmrg.py:27), tnkit.circuit (circuit.py:25) and the
  package namespace (__init__.py:19);
* ``DenseTensor.contiguous`` / ``contiguous_`` / ``reshape`` -- the permute
  materialisation ``np.ascontiguousarray(self.view())`` at storage.py:122, :126, :143.

Boundary semantics: tnkit tensors are host (numpy) objects, so every patched call uploads
its operands (each block's storage buffer as is, with its lazy permutation kept as the
engine's view -- the permute is fused into the GEMM operand gather on the device),
contracts on the GPU, and returns a fresh tnkit object holding the downloaded result. The
engine performs the reference's pair checks itself before any device work (same
exception types and messages, contract.py:84-123). The output bonds are tnkit's own Bond
objects (a_free then b_free, contract.py:118-124), exactly as the reference builds them.

There is no CPU fallback: int64 / bool contractions raise the engine's TypeError (the
north star covers float64 / complex128); the permute seams move any dtype on the GPU.
"""
import sys

import numpy as np

import paper_2401_01921_b200 as eng
from paper_2401_01921_b200 import _lib
from paper_2401_01921_b200 import dense as edense

_STATE = {}


def _mod(name):
    return sys.modules[name]


# ------------------------------------------------------------------------- conversions
def _sym_to_engine(s):
    return eng.Symmetry.u1() if s.kind == "U1" else eng.Symmetry.zn(s.n)


def _bond_to_engine(b):
    btype = eng.charges.BondType(b.btype.value)
    if b.sectors:
        return eng.Bond(btype=btype, sectors=[(tuple(q), d) for q, d in b.sectors],
                        syms=[_sym_to_engine(s) for s in b.syms])
    return eng.Bond(b.dim, btype)


def _dense_to_engine(dt):
    """tnkit DenseTensor (host storage buffer + lazy perm) -> engine DenseTensor with the
    same storage buffer in HBM and the same lazy perm (no materialisation)."""
    t = edense.DenseTensor(np.ascontiguousarray(dt._storage))
    if dt._perm != tuple(range(dt._storage.ndim)):
        t = t.permute(*dt._perm)
    return t


def _unitensor_to_engine(ut):
    bonds = [_bond_to_engine(b) for b in ut.bonds]
    blocks = [_dense_to_engine(b) for b in ut._blocks]
    qns = None if ut._qns is None else [tuple(q) for q in ut._qns]
    return eng.UniTensor._assemble(bonds, list(ut.labels), ut.rowrank, ut.name, blocks, qns)


# ------------------------------------------------------------------------- patched seams
def contract_pair_b200(a, b):
    """tnkit.contract.contract_pair on the B200 engine (contract.py:100-167 semantics)."""
    tk = _STATE["tnkit"]
    if not isinstance(a, tk.UniTensor) or not isinstance(b, tk.UniTensor):
        raise TypeError("contract expects UniTensors")
    ea, eb = _unitensor_to_engine(a), _unitensor_to_engine(b)
    res = eng.contract_pair(ea, eb)  # engine pair checks (ValueError/TypeError) before any device work
    _STATE["calls"] += 1
    a_labels, b_labels = a.labels, b.labels
    shared = [l for l in a_labels if l in b_labels]
    a_free = [i for i in range(a.rank) if a_labels[i] not in shared]
    b_free = [i for i in range(b.rank) if b_labels[i] not in shared]
    out_labels = [a_labels[i] for i in a_free] + [b_labels[i] for i in b_free]
    out_bonds = [a.bonds[i] for i in a_free] + [b.bonds[i] for i in b_free]
    if res.rank == 0:
        return tk.UniTensor.scalar(res.item())
    if not a.is_sym:
        arr = res.get_block_().numpy()
        return tk.UniTensor._assemble(out_bonds, out_labels, len(a_free), "",
                                      [tk.DenseTensor(np.ascontiguousarray(arr))], None)
    dt = np.result_type(a.dtype, b.dtype)
    out = tk.UniTensor(out_bonds, labels=out_labels, dtype=dt, rowrank=len(a_free))
    if [tuple(q) for q in out._qns] != [tuple(q) for q in res._qns]:
        raise _lib.EngineError("block enumeration differs between tnkit and the engine")
    for i, blk in enumerate(res.get_blocks_()):
        out._blocks[i] = tk.DenseTensor(blk.numpy())
    return out


def _materialise(dt):
    """The permute seam: the lazily permuted buffer in logical row-major order, computed by
    tnb_permute on the GPU (any dtype: the kernel moves elements as bytes)."""
    return _dense_to_engine(dt).contiguous().numpy()


def contiguous_b200(self):
    """storage.py:114-122 with the copy on the GPU."""
    if self.is_contiguous:
        return _STATE["orig"]["contiguous"](self)
    _STATE["permutes"] += 1
    return type(self)(_materialise(self))


def contiguous__b200(self):
    """storage.py:124-128."""
    if not self.is_contiguous:
        _STATE["permutes"] += 1
        self._storage = _materialise(self)
        self._perm = tuple(range(self._storage.ndim))
    return self


def reshape_b200(self, *shape):
    """storage.py:130-144: a non-contiguous tensor is materialised (on the GPU) first."""
    if self.is_contiguous:
        return _STATE["orig"]["reshape"](self, *shape)
    _STATE["permutes"] += 1
    return _STATE["orig"]["reshape"](type(self)(_materialise(self)), *shape)


# ------------------------------------------------------------------------- install
_BOUND = ("tnkit", "tnkit.contract", "tnkit.network", "tnkit.dmrg", "tnkit.circuit")


def install(tnkit=None):
    """Patch an imported tnkit so its hot path runs on the B200 engine. Idempotent;
    returns the counters dict (calls routed through the engine)."""
    if tnkit is None:
        import tnkit
    if _STATE.get("tnkit") is tnkit:
        return _STATE
    import tnkit.circuit  # noqa: F401  (make sure every binding module is loaded)
    import tnkit.dmrg  # noqa: F401
    import tnkit.network  # noqa: F401
    storage = _mod("tnkit.storage")
    _STATE.update(tnkit=tnkit, calls=0, permutes=0,
                  orig={"contract_pair": _mod("tnkit.contract").contract_pair,
                        "contiguous": storage.DenseTensor.contiguous,
                        "contiguous_": storage.DenseTensor.contiguous_,
                        "reshape": storage.DenseTensor.reshape})
    for name in _BOUND:
        setattr(_mod(name), "contract_pair", contract_pair_b200)
    storage.DenseTensor.contiguous = contiguous_b200
    storage.DenseTensor.contiguous_ = contiguous__b200
    storage.DenseTensor.reshape = reshape_b200
    return _STATE


def uninstall():
    if "tnkit" not in _STATE or _STATE["tnkit"] is None:
        return
    orig = _STATE["orig"]
    for name in _BOUND:
        setattr(_mod(name), "contract_pair", orig["contract_pair"])
    storage = _mod("tnkit.storage")
    storage.DenseTensor.contiguous = orig["contiguous"]
    storage.DenseTensor.contiguous_ = orig["contiguous_"]
    storage.DenseTensor.reshape = orig["reshape"]
    _STATE["tnkit"] = None


def counters():
    return {"contract_pair": _STATE.get("calls", 0), "permute": _STATE.get("permutes", 0),
            "libtnb_launches": _lib.launch_count()}
