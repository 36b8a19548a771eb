"""Pin the CPU oracle (oracle/tnkit_np.py) against the reference's own outputs.

The golden vectors were produced by oracle/make_golden.py from the reference
package itself; every oracle function the GPU parity tests rely on is checked
here, on CPU, before it is trusted.
"""
import numpy as np

import tnkit_np as oracle
from tnb_testutil import load, oracle_bonds


def test_permute_golden_vectors():
    z, meta = load("permute.npz")
    for k, c in enumerate(meta["cases"]):
        got = oracle.permute_contiguous(z[f"in{k}"], c["perm"])
        assert got.dtype == z[f"out{k}"].dtype
        assert np.array_equal(got, z[f"out{k}"]), c
    # acceptance golden (pkg/tests/test_acceptance.py:54-59)
    assert list(z["out0"].reshape(-1)) == [0, 2, 1, 3, 4, 6, 5, 7]


def test_dense_contract_golden_vectors():
    z, meta = load("dense.npz")
    for k, c in enumerate(meta["cases"]):
        a = z[f"a{k}"]
        a_labels = list(c["a_labels"])
        perm = c["a_perm"]
        av = a.transpose(perm)
        al = [a_labels[p] for p in perm]
        got, labels = oracle.contract_dense(av, al, z[f"b{k}"], c["b_labels"])
        assert labels == c["out_labels"]
        # same numpy primitives -> identical bits on the same machine; allow ulps elsewhere
        assert np.max(np.abs(got - z[f"out{k}"])) <= 1e-13


def test_zero_flux_enumeration_golden():
    _, meta = load("blocks.npz")
    for c in meta["enum"]:
        assert [list(x) for x in oracle.zero_flux_combos(oracle_bonds(c["bonds"]))] == c["qns"]
    # acceptance 1b: 4 blocks (0,0,0),(0,1,1),(1,0,1),(1,1,2)
    assert meta["enum"][0]["qns"] == [[0, 0, 0], [0, 1, 1], [1, 0, 1], [1, 1, 2]]


def test_block_sparse_golden_vectors():
    z, meta = load("blocks.npz")
    for k, c in enumerate(meta["cases"]):
        a_qns = [tuple(q) for q in c["a_qns"]]
        b_qns = [tuple(q) for q in c["b_qns"]]
        perm = c["a_perm"]
        ab = [z[f"c{k}_a{i}"].transpose(perm) for i in range(len(a_qns))]
        bb = [z[f"c{k}_b{j}"] for j in range(len(b_qns))]
        if "out_qns" not in c:
            total, _ = oracle.contract_blocks(a_qns, ab, c["a_labels"], b_qns, bb, c["b_labels"], None)
            assert abs(total - z[f"c{k}_scalar"]) <= 1e-12
            continue
        out_qns = [tuple(q) for q in c["out_qns"]]
        assert [list(q) for q in oracle.zero_flux_combos(oracle_bonds(c["out_bonds"]))] == c["out_qns"]
        res, trip = oracle.contract_blocks(a_qns, ab, c["a_labels"], b_qns, bb, c["b_labels"], out_qns)
        assert [list(t) for t in trip] == c["triples"]
        shapes = [z[f"c{k}_out{i}"].shape for i in range(len(out_qns))]
        res = oracle.finish_blocks(res, shapes, np.result_type(ab[0].dtype, bb[0].dtype))
        for i in range(len(out_qns)):
            assert np.max(np.abs(res[i] - z[f"c{k}_out{i}"])) <= 1e-13


def test_order_dp_golden():
    _, meta = load("order.npz")
    for c in meta["cases"]:
        t = oracle.find_optimal_order(c["sets"], c["dims"])
        assert oracle.render_order(t) == c["order"]
        assert str(oracle.contraction_cost(t, c["sets"], c["dims"])) == c["cost"]
    # pinned known answers (pkg/tests/test_contract.py:211-229)
    assert meta["cases"][0]["order"] == "((M1,M2),M3)" and meta["cases"][0]["cost"] == "880"
    assert meta["cases"][1]["cost"] == "404"


def test_network_golden():
    z, meta = load("network.npz")
    for k in range(3):
        c = meta["cases"][k]
        slots = []
        for line in c["net"][:-1]:
            n, rhs = line.split(":")
            slots.append((n.strip(), [t.strip() for t in rhs.split(",")]))
        arrays = {n: z[f"n{k}_{n}"] for n in c["names"]}
        got, tree = oracle.launch(slots, c["net"][-1].split(":", 1)[1], arrays)
        assert oracle.render_order(tree) == c["order"]
        assert np.max(np.abs(got - z[f"n{k}_out"])) <= 1e-12
    # CTM all-ones with its explicit ORDER: 2^12 (pkg/tests/test_network.py:243-253)
    c = meta["cases"][3]
    slots = []
    for line in c["net"][:-2]:
        n, rhs = line.split(":")
        slots.append((n.strip(), [t.strip() for t in rhs.split(",")]))
    arrays = {n: np.ones(c["shapes"][n]) for n, _ in slots}
    got, _ = oracle.launch(slots, "", arrays, order=c["net"][-1].split(":", 1)[1].strip())
    assert np.asarray(got).item() == c["scalar"] == 4096.0
    c = meta["cases"][4]
    slots = []
    for line in c["net"][:-1]:
        n, rhs = line.split(":")
        slots.append((n.strip(), [t.strip() for t in rhs.split(",")]))
    arrays = {n: z[f"n3_{n}"] for n in c["names"]}
    got, tree = oracle.launch(slots, "", arrays)
    assert oracle.render_order(tree) == c["order"]
    assert abs(np.asarray(got).item() - c["scalar"]) <= 1e-10 * max(1.0, abs(c["scalar"]))


def test_c4_structure_golden():
    z, meta = load("c4.npz")
    assert meta["sectors"] == [list(x) for x in oracle.c4_sectors()]
    assert len(meta["triples"]) == 40 and meta["macs"] == 169073208
    # the oracle's block enumeration and pairing reproduce the reference's structure
    sec = oracle.c4_sectors()
    qv = [(q,) for q, _ in sec]
    V = (1, qv, [0])
    Vr = (-1, qv, [0])
    P = (1, [(1,), (-1,)], [0])
    Pr = (-1, [(1,), (-1,)], [0])
    a_qns = oracle.zero_flux_combos([V, P, Vr])
    e_qns = oracle.zero_flux_combos([V, Pr, Vr])
    out_qns = oracle.zero_flux_combos([V, Vr])
    assert [list(q) for q in a_qns] == meta["a_qns"]
    assert [list(q) for q in e_qns] == meta["e_qns"]
    assert [list(q) for q in out_qns] == meta["out_qns"]
    deg = [d for _, d in sec]
    a_shapes = [(deg[q[0]], 1, deg[q[2]]) for q in a_qns]
    e_shapes = [(deg[q[0]], 1, deg[q[2]]) for q in e_qns]
    ab = oracle.fill_blocks_normal(a_shapes, seed=meta["seed"])
    eb = oracle.fill_blocks_normal(e_shapes, seed=meta["seed"] + 1)
    res, trip = oracle.contract_blocks(a_qns, ab, ["vl", "p", "vr"], e_qns, eb, ["vr", "p", "x"], out_qns)
    assert [list(t) for t in trip] == meta["triples"]
    norms = [np.linalg.norm(r) for r in res]
    assert np.allclose(norms, z["norms"], rtol=1e-12, atol=0)


def test_oracle_utn_loader_matches_reference_files():
    """The oracle's .utn reader reproduces the reference-written fixtures' blocks."""
    import json
    import os
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "utn")
    z = np.load(os.path.join(gold, "blocks.npz"))
    meta = json.loads(str(z["meta"]))
    for case, m in meta.items():
        header, blocks = oracle.load_utn(os.path.join(gold, case + ".utn"))
        assert header["name"] == m["name"] and header["labels"] == m["labels"] and len(blocks) == m["nblocks"]
        for i, b in enumerate(blocks):
            assert np.array_equal(b, z[f"{case}_b{i}"])


def test_oracle_svd_truncate_matches_reference_goldens():
    """Sector matricisation + truncation ranking of the oracle vs the reference's outputs."""
    import json
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "svd.npz"))
    meta = json.loads(str(z["meta"]))
    for name, m in meta.items():
        st = m["input"]
        if st["qns"] is None:
            mats = [z[f"{name}_in0"].reshape(int(np.prod(z[f"{name}_in0"].shape[:st["rowrank"]])), -1)]
        else:
            bonds = st["bonds"]
            r = st["rowrank"]
            nsym = len(bonds[0]["syms"])
            mods = [0 if s == "U1" else int(s[1:]) for s in bonds[0]["syms"]]

            def charge(rq):
                c = [0] * nsym
                for b, k in zip(bonds[:r], rq):
                    q = bonds and b["sectors"][k][0]
                    sgn = -1 if b["btype"] == "OUT" else 1
                    c = [(x + sgn * y) % n if n else x + sgn * y for x, y, n in zip(c, q, mods)]
                return tuple(c)
            blocks = [z[f"{name}_in{i}"] for i in range(len(st["qns"]))]
            mats = [mm for _, mm in oracle.sector_matrices(
                blocks, [tuple(q) for q in st["qns"]],
                lambda rq: int(np.prod([bonds[a]["sectors"][k][1] for a, k in enumerate(rq)])),
                lambda cq: int(np.prod([bonds[r + a]["sectors"][k][1] for a, k in enumerate(cq)])),
                charge, r)]
        smax = max(float(np.max(np.linalg.svd(mm, compute_uv=False))) for mm in mats)
        keeps, ss, _, _, _ = oracle.svd_truncate_values(mats, 10 ** 9)
        for i, s in enumerate(ss):
            assert np.max(np.abs(s - z[f"{name}_s{i}"])) <= 1e-12 * smax
        for k, tr in enumerate(m["trunc"]):
            keeps, ss, _, _, disc = oracle.svd_truncate_values(mats, tr["keepdim"], tr["err"], tr["min_blockdim"])
            assert [x for x in keeps if x > 0] == [shp[0] for shp in tr["S"]["shapes"]]
            want = z[f"{name}_t{k}_err"]
            got = np.array(disc) if disc else np.zeros(1)
            assert np.allclose(got, want, rtol=0, atol=1e-12 * max(1.0, smax))


def test_oracle_lanczos_matches_reference():
    """The oracle's Lanczos restatement reproduces the reference's Ritz values on the
    Hermitian L.A.W.R operator (tests/golden/lanczos.npz, oracle/make_golden_lanczos.py)."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lanczos.npz"))
    inp = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    shape = inp["A"].shape

    def mv(v):
        arrs = dict(inp)
        arrs["A"] = v.reshape(shape)
        out, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", arrs)
        return np.ascontiguousarray(out).reshape(-1)
    for seed in (3, 11):
        theta, _, _ = oracle.lanczos(mv, int(np.prod(shape)), k=2, tol=1e-12, seed=seed)
        assert np.allclose(theta, z[f"theta_seed{seed}"], rtol=0, atol=1e-12)
