"""Write .utn container fixtures with the REFERENCE's own save_unitensor (build container only).

tests/golden/utn/<case>.utn   files written by tnkit.io.save_unitensor (pkg/src/tnkit/io.py:56-80)
tests/golden/utn/blocks.npz   each case's blocks as numpy arrays (C order) + a JSON 'meta'
                              (name, labels, rowrank, dtype, block qn tuples)

The cases mirror pkg/tests/test_io.py (dense / complex+directed / U1 / U1xZ2 / int64) plus
a U(1) tensor with odd sector sizes (block starts that are not 64-byte aligned in HBM).
Usage:  python oracle/make_golden_utn.py
"""
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "utn")
sys.path.insert(0, REF)

from tnkit import IN, OUT as BOUT, Bond, Complex128, Int64, Symmetry, UniTensor, save_unitensor, storage  # noqa: E402
from tnkit import random as trandom  # noqa: E402


def cases():
    u1 = Symmetry.u1()
    z2 = Symmetry.zn(2)
    t = UniTensor.normal([3, 4, 2], labels=["a", "b", "c"], name="T", seed=5).set_rowrank_(2)
    yield "dense", t
    c = UniTensor([Bond(2, IN), Bond(2, BOUT)], labels=["x", "y"], dtype=Complex128)
    c.at([0, 1]).value = 1 - 2j
    c.at([1, 0]).value = 0.5 + 0.25j
    yield "complex_directed", c
    b1 = Bond(btype=IN, sectors=[(1, 2), (-1, 1)], syms=[u1])
    b2 = Bond(btype=BOUT, sectors=[(1, 1), (-1, 2)], syms=[u1])
    s = UniTensor([b1, b2], labels=["a", "b"], name="S")
    trandom.uniform_(s, seed=3)
    yield "u1", s
    b = Bond(btype=IN, sectors=[((1, 0), 1), ((-1, 1), 2)], syms=[u1, z2])
    m = UniTensor([b, b.redirect()], labels=["a", "b"])
    trandom.normal_(m, seed=1)
    yield "u1xz2", m
    yield "int64", UniTensor(storage.ones([2, 2], dtype=Int64), labels=["a", "b"])
    V = Bond(btype=IN, sectors=[(-2, 3), (-1, 5), (0, 7), (1, 5), (2, 3)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    a = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"], name="A")
    trandom.normal_(a, seed=11)
    yield "u1_odd_sectors", a
    cz = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"], name="Ac", dtype=Complex128)
    trandom.normal_(cz, seed=12)
    yield "u1_c128", cz


def main():
    os.makedirs(OUT, exist_ok=True)
    arrays, meta = {}, {}
    for name, t in cases():
        save_unitensor(t, os.path.join(OUT, name + ".utn"))
        blocks = t.get_blocks_()
        for i, blk in enumerate(blocks):
            arrays[f"{name}_b{i}"] = np.ascontiguousarray(blk.view())
        meta[name] = {"name": t.name, "labels": t.labels, "rowrank": t.rowrank, "dtype": str(t.dtype),
                      "nblocks": len(blocks),
                      "qns": [list(t.block_qn_indices(i)) for i in range(len(blocks))] if t.is_sym else None}
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, "blocks.npz"), **arrays)
    print("wrote", len(meta), "cases to", OUT)


if __name__ == "__main__":
    main()
