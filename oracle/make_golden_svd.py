"""Golden SVD / truncated-SVD results from the REFERENCE (tnkit.linalg, build container only).

tests/golden/svd.npz: for each case the input blocks, and the reference's outputs --
singular values per sector (S diagonal blocks), the bond structure of S / U / Vdag
(btype, sectors), labels, block qn tuples and shapes, and for svd_truncate the kept
sizes and the discarded-values tensor. U / Vdag element values are not stored: they
are unique only up to a phase per singular vector; the tests check the invariants
(reconstruction, isometry) instead.  Usage:  python oracle/make_golden_svd.py
"""
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, REF)

from tnkit import IN, OUT as BOUT, Bond, Complex128, Symmetry, UniTensor, linalg, storage  # noqa: E402
from tnkit import random as trandom  # noqa: E402


def bonds_json(t):
    return [{"btype": b.btype.name, "dim": b.dim, "syms": [str(s) for s in b.syms],
             "sectors": [[list(q), d] for q, d in b.sectors]} for b in t.bonds]


def struct_json(t):
    return {"labels": t.labels, "rowrank": t.rowrank, "name": t.name, "bonds": bonds_json(t),
            "qns": [list(t.block_qn_indices(i)) for i in range(t.nblocks)] if t.is_sym else None,
            "shapes": [list(b.shape) for b in t.get_blocks_()]}


def cases():
    u1, z2 = Symmetry.u1(), Symmetry.zn(2)
    m = UniTensor(storage.arange(24).reshape(2, 2, 6), labels=["a", "b", "c"], name="M")
    yield "rank3_matrix", m.permute(["c", "a", "b"]).set_rowrank(1)
    yield "dense_5x7", UniTensor.normal([5, 7], labels=["a", "b"], seed=11).set_rowrank_(1)
    b12 = Bond(btype=IN, sectors=[(1, 2), (-1, 2)], syms=[u1])
    b3 = Bond(btype=BOUT, sectors=[(2, 2), (0, 4), (-2, 2)], syms=[u1])
    t = UniTensor([b12, b12, b3], labels=["a", "b", "c"], name="uTsym")
    trandom.uniform_(t, low=-1.0, high=1.0, seed=4)
    yield "sym_rank3", t
    V = Bond(btype=IN, sectors=[(-3, 2), (-2, 5), (-1, 9), (0, 12), (1, 9), (2, 5), (3, 2)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    psi = UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], name="psi", rowrank=2)
    trandom.normal_(psi, seed=21)
    yield "two_site_u1", psi
    psic = UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], name="psic", rowrank=2,
                     dtype=Complex128)
    trandom.normal_(psic, seed=22)
    yield "two_site_u1_c128", psic
    b = Bond(btype=IN, sectors=[((1, 0), 3), ((-1, 1), 2), ((0, 1), 4)], syms=[u1, z2])
    mz = UniTensor([b, b, b.redirect(), b.redirect()], labels=["a", "b", "c", "d"], name="mz", rowrank=2)
    trandom.normal_(mz, seed=23)
    yield "u1xz2_rank4", mz


def main():
    arrays, meta = {}, {}
    for name, t in cases():
        for i, blk in enumerate(t.get_blocks_()):
            arrays[f"{name}_in{i}"] = np.ascontiguousarray(blk.view())
        s, u, v = linalg.svd(t)
        entry = {"input": struct_json(t), "dtype": str(t.dtype), "S": struct_json(s), "U": struct_json(u),
                 "Vdag": struct_json(v), "trunc": []}
        for i in range(s.nblocks):
            arrays[f"{name}_s{i}"] = np.diag(s.get_block_(i).view()).copy()
        total = sum(s.get_block_(i).shape[0] for i in range(s.nblocks))
        for kd, err, mb in [(max(1, total // 2), 0.0, None), (max(1, total // 3), 1e-1, None),
                            (3, 0.0, [1] * s.nblocks if t.is_sym else None), (10 ** 6, 1e30, None)]:
            st, ut_, vt, et = linalg.svd_truncate(t, keepdim=kd, err=err, return_err=2, min_blockdim=mb)
            k = len(entry["trunc"])
            entry["trunc"].append({"keepdim": kd, "err": err, "min_blockdim": mb, "S": struct_json(st),
                                   "U": struct_json(ut_), "Vdag": struct_json(vt)})
            arrays[f"{name}_t{k}_err"] = np.asarray(et.get_block_().view()).copy()
            for i in range(st.nblocks):
                arrays[f"{name}_t{k}_s{i}"] = np.diag(st.get_block_(i).view()).copy()
        meta[name] = entry
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, "svd.npz"), **arrays)
    print("wrote", len(meta), "svd cases")


if __name__ == "__main__":
    main()
