"""Generate tests/golden/*.npz from the REFERENCE itself (build container only).

Imports the reference package `tnkit` from /root/reference/pkg/src (read-only,
never copied) and records inputs + reference outputs for the hot path:

  permute.npz     DenseTensor.permute(...).contiguous()      storage.py:101-126
  dense.npz       contract / contract_pair (dense)           contract.py:100-134
  blocks.npz      zero-flux block structure + block-sparse    unitensor.py:31-45,
                  contraction (U1, Z2, Z3, U1xZ2)             contract.py:137-167
  order.npz       find_optimal_order / contraction_cost      contract.py:253-343
  network.npz     Network.launch (L.A.W.R, CTM, TOUT)         network.py:213-244
  c4.npz          the full-size C4 config: output structure, pairing triples,
                  per-block reference norms and samples

Each file holds arrays plus a JSON 'meta' string. Usage:
    python oracle/make_golden.py            # writes tests/golden/
The fixtures are committed; /root/reference is not needed afterwards.
"""
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, HERE)

import tnkit  # noqa: E402  (the reference)
from tnkit import Bond, IN, OUT as BOUT, Network, Symmetry, UniTensor, contract, storage  # noqa: E402
from tnkit import random as trandom  # noqa: E402

import tnkit_np as oracle  # noqa: E402


def save(name, arrays, meta):
    os.makedirs(OUT, exist_ok=True)
    arrays = dict(arrays)
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print(f"wrote {name}: {len(arrays) - 1} arrays")


def gen_permute():
    rng = np.random.default_rng(7)
    arrays, cases = {}, []
    specs = [((2, 2, 2), (0, 2, 1), "float64"),     # acceptance golden [0,2,1,3,4,6,5,7]
             ((2, 3, 4), (1, 2, 0), "float64"), ((3, 1, 4, 2), (3, 0, 2, 1), "float64"),
             ((5,), (0,), "float64"), ((4, 6), (1, 0), "complex128"), ((1, 1, 3), (2, 1, 0), "int64"),
             ((7, 5, 3, 2), (0, 2, 1, 3), "float64"), ((7, 5, 3, 2), (3, 2, 1, 0), "complex128"),
             ((8, 8, 8, 8), (1, 0, 3, 2), "float64"), ((3, 4, 5, 6, 2), (4, 0, 3, 1, 2), "float64"),
             ((2, 3, 2, 3, 2, 3), (5, 3, 1, 4, 2, 0), "complex128"), ((16, 16, 16), (2, 0, 1), "bool"),
             ((33, 65, 17), (1, 2, 0), "float64"), ((130, 3, 70), (2, 1, 0), "float64"),
             ((2, 2, 2, 2, 2, 2, 2, 2), (7, 0, 6, 1, 5, 2, 4, 3), "float64")]
    for shape in [(4, 4, 4, 4), (6, 5, 4, 3)]:
        for _ in range(3):
            specs.append((shape, tuple(int(x) for x in rng.permutation(4)), "float64"))
    for k, (shape, perm, dt) in enumerate(specs):
        n = int(np.prod(shape))
        if dt == "int64":
            t = storage.arange(n, dtype=storage.Int64).reshape(*shape)
        elif dt == "bool":
            t = storage.from_numpy(rng.random(shape) < 0.5)
        elif k == 0:
            t = storage.arange(n).reshape(*shape)
        else:
            t = storage.uniform(list(shape), dtype=np.dtype(dt), seed=100 + k)
        src = np.array(t.storage())
        p = t.permute(*perm)
        p.contiguous_()
        arrays[f"in{k}"] = src.reshape(shape)
        arrays[f"out{k}"] = np.array(p.storage()).reshape(p.shape)
        cases.append({"shape": list(shape), "perm": list(perm), "dtype": dt})
    save("permute.npz", arrays, {"cases": cases})


def gen_dense():
    rng = np.random.default_rng(20240611)
    arrays, cases = {}, []
    labels_all = [f"l{i}" for i in range(8)]
    for k in range(40):
        ra, rb = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        rng.shuffle(labels_all)
        a_labels = labels_all[:ra]
        ns = int(rng.integers(0, min(ra, rb) + 1))
        b_labels = a_labels[:ns] + labels_all[ra:ra + rb - ns]
        rng.shuffle(b_labels)
        dims = {l: int(rng.integers(1, 6)) for l in set(a_labels) | set(b_labels)}
        dt = np.complex128 if k % 5 == 4 else np.float64
        a_arr = oracle.normal([dims[l] for l in a_labels], dtype=dt, seed=1000 + k)
        b_arr = oracle.normal([dims[l] for l in b_labels], dtype=np.float64 if k % 7 == 6 else dt, seed=2000 + k)
        a = UniTensor(storage.from_numpy(a_arr), labels=list(a_labels), name="A")
        b = UniTensor(storage.from_numpy(b_arr), labels=list(b_labels), name="B")
        # lazily permuted operands in a third of the cases (test_mixed_symmetries.py:140-156)
        a_perm = list(range(ra))
        if k % 3 == 2 and ra > 1:
            a_perm = [int(x) for x in rng.permutation(ra)]
            a = a.permute(a_perm)
        got = contract(a, b)
        arrays[f"a{k}"] = a_arr
        arrays[f"b{k}"] = b_arr
        arrays[f"out{k}"] = np.array(got.get_block_().view()) if got.rank else np.array(got.item())
        cases.append({"a_labels": list(a_labels), "b_labels": list(b_labels), "a_perm": a_perm,
                      "out_labels": got.labels})
    save("dense.npz", arrays, {"cases": cases})


def _bond_meta(b):
    return {"btype": 1 if b.btype == IN else -1, "sectors": [[list(q), d] for q, d in b.sectors],
            "syms": [str(s) for s in b.syms]}


def _rand_sym_pair(rng, syms, k):
    """A rank-3 tensor and a rank-2/3 partner sharing one or two bonds."""
    def rand_bond(btype):
        space = 1
        for s in syms:
            space *= 5 if s.n == 0 else s.n
        nsec = int(rng.integers(1, min(3, space) + 1))
        seen, sec = set(), []
        while len(sec) < nsec:
            q = tuple(int(rng.integers(-2, 3)) if s.n == 0 else int(rng.integers(0, s.n)) for s in syms)
            if q in seen:
                continue
            seen.add(q)
            sec.append((q, int(rng.integers(1, 4))))
        return Bond(btype=btype, sectors=sec, syms=syms)
    for _ in range(200):
        try:
            b0 = rand_bond(IN if rng.random() < 0.5 else BOUT)
            b1 = rand_bond(IN if rng.random() < 0.5 else BOUT)
            b2 = rand_bond(IN if rng.random() < 0.5 else BOUT)
            a = UniTensor([b0, b1, b2], labels=["x", "y", "s"])
            if k % 2 == 0:
                bb = UniTensor([b2.redirect(), rand_bond(IN if rng.random() < 0.5 else BOUT)], labels=["s", "z"])
            else:
                bb = UniTensor([b1.redirect(), b2.redirect(), rand_bond(IN if rng.random() < 0.5 else BOUT)],
                               labels=["y", "s", "z"])
            out = contract(a, bb)  # may raise "no valid blocks"
            return a, bb
        except ValueError:
            continue
    raise RuntimeError("could not draw a valid pair")


def gen_blocks():
    rng = np.random.default_rng(31)
    u1, z2, z3 = Symmetry.u1(), Symmetry.zn(2), Symmetry.zn(3)
    arrays, cases = {}, []
    symsets = [[u1]] * 8 + [[z2]] * 2 + [[z3]] * 2 + [[u1, z2]] * 3
    for k, syms in enumerate(symsets):
        a, b = _rand_sym_pair(rng, syms, k)
        dt = np.complex128 if k % 4 == 3 else np.float64
        a = a.astype(dt)
        trandom.normal_(a, seed=500 + k)
        trandom.normal_(b, seed=600 + k)
        if k % 3 == 1:  # lazily permuted operand
            a = a.permute(["s", "x", "y"])
        out = contract(a, b)
        ca = {"a_bonds": [_bond_meta(x) for x in a.bonds], "a_labels": a.labels,
              "a_qns": [list(a.block_qn_indices(i)) for i in range(a.nblocks)],
              "a_perm": list(a.get_block_(0)._perm),
              "b_bonds": [_bond_meta(x) for x in b.bonds], "b_labels": b.labels,
              "b_qns": [list(b.block_qn_indices(i)) for i in range(b.nblocks)],
              "out_labels": out.labels, "dtype": np.dtype(dt).name}
        if out.rank:
            ca["out_qns"] = [list(out.block_qn_indices(i)) for i in range(out.nblocks)]
            ca["out_bonds"] = [_bond_meta(x) for x in out.bonds]
            for i in range(out.nblocks):
                arrays[f"c{k}_out{i}"] = np.array(out.get_block_(i).view())
            # oracle pairing triples (checked numerically against the reference outputs)
            ab = [np.array(x.view()) for x in a.get_blocks_()]
            bb_ = [np.array(x.view()) for x in b.get_blocks_()]
            res, trip = oracle.contract_blocks(ca["a_qns"], ab, a.labels, ca["b_qns"], bb_, b.labels,
                                               ca["out_qns"])
            res = oracle.finish_blocks(res, [x.shape for x in out.get_blocks_()], out.dtype)
            for i in range(out.nblocks):
                assert np.allclose(res[i], arrays[f"c{k}_out{i}"], rtol=0, atol=1e-13)
            ca["triples"] = [list(t) for t in trip]
        else:
            arrays[f"c{k}_scalar"] = np.array(out.item())
        # storage-order (un-permuted) block buffers as drawn
        for i, blk in enumerate(a.get_blocks_()):
            arrays[f"c{k}_a{i}"] = np.array(blk._storage)
        for j, blk in enumerate(b.get_blocks_()):
            arrays[f"c{k}_b{j}"] = np.array(blk._storage)
        cases.append(ca)
    # zero-flux enumeration goldens (incl. the acceptance rank-3 tensor, unitensor tests)
    enum_cases = []
    b1 = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    b3 = Bond(btype=BOUT, sectors=[(2, 1), (0, 2), (-2, 1)], syms=[u1])
    zb = Bond(btype=IN, sectors=[(0, 1), (1, 2)], syms=[z2])
    z3i = Bond(btype=IN, sectors=[(1, 1), (2, 1)], syms=[z3])
    z3o = Bond(btype=BOUT, sectors=[(0, 1), (1, 1), (2, 1)], syms=[z3])
    p1 = Bond(btype=IN, sectors=[((1, 0), 1), ((-1, 1), 2)], syms=[u1, z2])
    p2 = Bond(btype=IN, sectors=[((1, 1), 2), ((0, 0), 1)], syms=[u1, z2])
    p3 = Bond(btype=BOUT, sectors=[((2, 1), 1), ((0, 0), 2), ((-1, 0), 1)], syms=[u1, z2])
    for bonds in ([b1, b1, b3], [zb, zb, zb.redirect()], [z3i, z3i, z3o], [p1, p2, p3]):
        t = UniTensor(bonds)
        enum_cases.append({"bonds": [_bond_meta(x) for x in bonds],
                           "qns": [list(t.block_qn_indices(i)) for i in range(t.nblocks)],
                           "shapes": [list(x.shape) for x in t.get_blocks_()]})
    save("blocks.npz", arrays, {"cases": cases, "enum": enum_cases})


def gen_order():
    rng = np.random.default_rng(99)
    cases = []
    fixed = [({"M1": ["i", "j"], "M2": ["j", "k"], "M3": ["k", "l"]}, {"i": 2, "j": 20, "k": 20, "l": 2}),
             ({"A": ["i"], "B": ["j"], "C": ["i", "j", "k"]}, {"i": 2, "j": 2, "k": 100}),
             ({"A": ["i", "j"], "B": ["j"]}, {"i": 2, "j": 3})]
    for sets, dims in fixed:
        t = tnkit.find_optimal_order(sets, dims)
        cases.append({"sets": sets, "dims": dims, "order": tnkit.render_order(t),
                      "cost": str(tnkit.contraction_cost(t, sets, dims))})
    for _ in range(60):
        nt = int(rng.integers(2, 9))
        names = [f"T{i}" for i in range(nt)]
        sets = {n: [] for n in names}
        dims, lbl = {}, 0
        for i in range(nt):
            for j in range(i + 1, nt):
                if rng.random() < 0.5:
                    l = f"e{lbl}"
                    lbl += 1
                    sets[names[i]].append(l)
                    sets[names[j]].append(l)
                    dims[l] = int(rng.integers(2, 9))
        for i in range(nt):
            if rng.random() < 0.5 or not sets[names[i]]:
                l = f"f{lbl}"
                lbl += 1
                sets[names[i]].append(l)
                dims[l] = int(rng.integers(2, 9))
        t = tnkit.find_optimal_order(sets, dims)
        cases.append({"sets": sets, "dims": dims, "order": tnkit.render_order(t),
                      "cost": str(tnkit.contraction_cost(t, sets, dims))})
    # the benchmark networks: LAWR (chi 128/1024/512) and PEPS reading A
    lawr = {"L": ["b", "w", "vl"], "A": ["vl", "p", "vr"], "W": ["w", "w2", "q", "p"], "R": ["b2", "w2", "vr"]}
    for chi in (128, 512, 1024):
        dims = {"b": chi, "vl": chi, "vr": chi, "b2": chi, "w": 5, "w2": 5, "p": 2, "q": 2}
        t = tnkit.find_optimal_order(lawr, dims)
        cases.append({"sets": lawr, "dims": dims, "order": tnkit.render_order(t),
                      "cost": str(tnkit.contraction_cost(t, lawr, dims))})
    save("order.npz", {}, {"cases": cases})


LAWR = ["L: b, w, vl", "A: vl, p, vr", "W: w, w2, q, p", "R: b2, w2, vr", "TOUT: b, q, b2"]
CTM = ["c0: t0-c0, t3-c0", "c1: t1-c1, t0-c1", "c2: t2-c2, t1-c2", "c3: t3-c3, t2-c3",
       "t0: t0-c1, w-t0, t0-c0", "t1: t1-c2, w-t1, t1-c1", "t2: t2-c3, w-t2, t2-c2", "t3: t3-c0, w-t3, t3-c3",
       "w: w-t0, w-t1, w-t2, w-t3", "TOUT:", "ORDER: ((((((((c0,t0),c1),t3),w),t1),c3),t2),c2)"]
PEPS_A = ["C0: c0t0, c0t3", "C1: c1t1, c1t0", "C2: c2t2, c2t1", "C3: c3t3, c3t2",
          "T0: c1t0, u, u', c0t0", "T1: c2t1, r, r', c1t1", "T2: c3t2, dn, dn', c2t2", "T3: c0t3, l, l', c3t3",
          "a: u, l, dn, r, s", "a*: u', l', dn', r', s", "TOUT:"]


def gen_network():
    arrays, cases = {}, []
    # L.A.W.R (C1 blueprint) at small chi, f64 and c128, optimal order
    for k, (chi, dt) in enumerate([(6, np.float64), (7, np.complex128), (16, np.float64)]):
        inp = oracle.lawr_inputs(chi, dtype=dt, seed=4242 + k)
        net = Network(LAWR)
        for nm, arr in inp.items():
            labels = [f"{nm}{i}" for i in range(arr.ndim)]
            net.put_tensor(nm, UniTensor(storage.from_numpy(arr), labels=labels), labels)
        net.set_order(optimal=True)
        out = net.launch()
        for nm, arr in inp.items():
            arrays[f"n{k}_{nm}"] = arr
        arrays[f"n{k}_out"] = np.ascontiguousarray(np.array(out.get_block_().view()))
        cases.append({"net": LAWR, "optimal": True, "order": net.get_order(), "labels": out.labels,
                      "rowrank": out.rowrank, "names": list(inp)})
    # CTM all-ones (test_network.py:243-253): 2^12
    net = Network(CTM)
    shapes = {}
    for nm in ("c0", "c1", "c2", "c3"):
        shapes[nm] = [2, 2]
    for nm in ("t0", "t1", "t2", "t3"):
        shapes[nm] = [2, 2, 2]
    shapes["w"] = [2, 2, 2, 2]
    for nm, s in shapes.items():
        net.put_tensor(nm, UniTensor.ones(s, labels=[f"x{i}" for i in range(len(s))]))
    cases.append({"net": CTM, "optimal": False, "scalar": net.launch().item(), "shapes": shapes})
    # PEPS reading A at a small size, optimal order, scalar out
    chi, D, d = 4, 2, 2
    shp = {"C0": [chi, chi], "C1": [chi, chi], "C2": [chi, chi], "C3": [chi, chi],
           "T0": [chi, D, D, chi], "T1": [chi, D, D, chi], "T2": [chi, D, D, chi], "T3": [chi, D, D, chi],
           "a": [D, D, D, D, d], "a*": [D, D, D, D, d]}
    net = Network(PEPS_A)
    k = 3
    for i, (nm, s) in enumerate(shp.items()):
        arr = oracle.normal(s, seed=7000 + i)
        arrays[f"n{k}_{nm}"] = arr
        net.put_tensor(nm, UniTensor(storage.from_numpy(arr), labels=[f"x{j}" for j in range(len(s))]))
    net.set_order(optimal=True)
    val = net.launch().item()
    cases.append({"net": PEPS_A, "optimal": True, "order": net.get_order(), "scalar": val, "names": list(shp)})
    # TOUT verbatim (test_network.py:200-208)
    net = Network(["A: x, y, z", "TOUT: z, x ; y"])
    t = UniTensor(storage.arange(24).reshape(2, 3, 4), labels=["p", "q", "r"])
    net.put_tensor("A", t, ["p", "q", "r"])
    out = net.launch()
    arrays["n5_out"] = np.ascontiguousarray(np.array(out.get_block_().view()))
    cases.append({"net": ["A: x, y, z", "TOUT: z, x ; y"], "labels": out.labels, "rowrank": out.rowrank})
    save("network.npz", arrays, {"cases": cases})


def gen_c4():
    u1 = Symmetry.u1()
    sec = oracle.c4_sectors()
    V = Bond(btype=IN, sectors=sec, syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
    E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
    S = 777
    trandom.normal_(A, seed=S)
    trandom.normal_(E, seed=S + 1)
    out = contract(A, E)
    aq = [list(A.block_qn_indices(i)) for i in range(A.nblocks)]
    eq = [list(E.block_qn_indices(i)) for i in range(E.nblocks)]
    oq = [list(out.block_qn_indices(i)) for i in range(out.nblocks)]
    ab = [np.array(b.view()) for b in A.get_blocks_()]
    eb = [np.array(b.view()) for b in E.get_blocks_()]
    res, trip = oracle.contract_blocks(aq, ab, A.labels, eq, eb, E.labels, oq)
    norms = [float(np.linalg.norm(np.array(b.view()))) for b in out.get_blocks_()]
    arrays = {"norms": np.array(norms), "sample": np.array([np.array(b.view()).reshape(-1)[:4] for b in
                                                            out.get_blocks_() if b.size >= 4])}
    for i in range(out.nblocks):
        assert np.allclose(res[i], np.array(out.get_block_(i).view()), rtol=0, atol=1e-12)
    meta = {"seed": S, "sectors": sec, "a_qns": aq, "e_qns": eq, "out_qns": oq,
            "out_shapes": [list(b.shape) for b in out.get_blocks_()], "triples": [list(t) for t in trip],
            "out_labels": out.labels, "macs": int(sum(ab[i].shape[0] * ab[i].shape[1] * ab[i].shape[2] *
                                                       eb[j].shape[2] for i, j, _ in trip))}
    save("c4.npz", arrays, meta)


if __name__ == "__main__":
    gen_permute()
    gen_dense()
    gen_blocks()
    gen_order()
    gen_network()
    gen_c4()
