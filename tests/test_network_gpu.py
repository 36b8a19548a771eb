"""a16/a17: Network.launch on device tensors vs reference golden launches and the
oracle; reuse, rebinding, TOUT verbatim, order policy, validation."""
import numpy as np
import pytest

import tnkit_np as oracle
from tnb_testutil import load, rel_fro

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import IN, Bond, Network, Symmetry, UniTensor, contract_pair, parse_order, storage, tree_leaves

pytestmark = pytest.mark.gpu

MATMUL = ["M1:  i, j", "M2:  j, k", "TOUT: i, k"]
THREE = ["M1: i, j", "M2: j, k", "M3: k, l", "TOUT: i, l", "ORDER: ((M1,M2),M3)"]


def test_golden_network_launches(cuda):
    z, meta = load("network.npz")
    for k in range(3):
        c = meta["cases"][k]
        net = Network(c["net"])
        for nm in c["names"]:
            arr = z[f"n{k}_{nm}"]
            labels = [f"{nm}{i}" for i in range(arr.ndim)]
            net.put_tensor(nm, UniTensor(storage.from_numpy(arr), labels=labels), labels)
        net.set_order(optimal=True)
        out = net.launch()
        assert net.get_order() == c["order"] and out.labels == c["labels"] and out.rowrank == c["rowrank"]
        assert np.max(np.abs(out.numpy() - z[f"n{k}_out"])) <= 1e-12
    c = meta["cases"][3]
    net = Network(c["net"])
    for nm, s in c["shapes"].items():
        net.put_tensor(nm, UniTensor.ones(s, labels=[f"x{i}" for i in range(len(s))]))
    out = net.launch()
    assert out.rank == 0 and out.item() == 4096.0
    c = meta["cases"][4]
    net = Network(c["net"])
    for nm in c["names"]:
        arr = z[f"n3_{nm}"]
        net.put_tensor(nm, UniTensor(storage.from_numpy(arr), labels=[f"x{j}" for j in range(arr.ndim)]))
    net.set_order(optimal=True)
    val = net.launch().item()
    assert net.get_order() == c["order"]
    assert abs(val - c["scalar"]) <= 1e-10 * max(1.0, abs(c["scalar"]))
    c = meta["cases"][5]
    net = Network(c["net"])
    net.put_tensor("A", UniTensor(storage.arange(24).reshape(2, 3, 4), labels=["p", "q", "r"]), ["p", "q", "r"])
    out = net.launch()
    assert out.labels == c["labels"] == ["z", "x", "y"] and out.shape == (4, 2, 3) and out.rowrank == 2
    assert np.array_equal(out.numpy(), z["n5_out"])


def test_matmul_reuse_and_rebinding(cuda):
    net = Network(MATMUL)
    a = UniTensor.ones([2, 2], labels=["a", "b"], name="A")
    b = UniTensor(storage.arange(4).reshape(2, 2), labels=["a", "b"], name="B")
    net.put_tensor("M1", a, ["a", "b"])
    net.put_tensor("M2", b, ["a", "b"])
    ab = net.launch()
    assert ab.labels == ["i", "k"] and ab.rowrank == 1
    assert np.allclose(ab.numpy(), np.ones((2, 2)) @ np.arange(4).reshape(2, 2))
    net.put_tensor("M1", b, ["a", "b"])
    net.put_tensor("M2", a, ["a", "b"])
    assert np.allclose(net.launch().numpy(), np.arange(4).reshape(2, 2) @ np.ones((2, 2)))
    assert a.labels == ["a", "b"]  # user tensors keep their labels
    z0 = UniTensor.zeros([2, 2], labels=["a", "b"])
    net.put_tensor("M1", z0)
    assert net.launch().norm() == 0.0


def test_launch_validation_messages(cuda):
    net = Network(MATMUL)
    net.put_tensor("M1", UniTensor.ones([2, 3], labels=["a", "b"]))
    with pytest.raises(ValueError, match="M2"):
        net.launch()
    net.put_tensor("M2", UniTensor.ones([2, 2], labels=["a", "b"]))
    with pytest.raises(ValueError, match="j"):
        net.launch()
    with pytest.raises(ValueError):
        net.put_tensor("M9", UniTensor.ones([2, 2], labels=["a", "b"]))
    with pytest.raises(ValueError):
        net.put_tensor("M1", UniTensor.ones([2, 2], labels=["a", "b"]), ["a", "zz"])
    u1 = Symmetry.u1()
    bi = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    s = UniTensor([bi, bi.redirect()], labels=["x", "y"])
    net = Network(MATMUL)
    net.put_tensor("M1", s, ["x", "y"])
    net.put_tensor("M2", s, ["x", "y"])
    net.launch()
    net.put_tensor("M2", s, ["y", "x"])
    with pytest.raises(ValueError, match="direction"):
        net.launch()


def test_optimal_order_recomputed_each_launch(cuda):
    net = Network(THREE)
    net.set_order(optimal=True)
    net.put_tensor("M1", UniTensor.ones([2, 20], labels=["a", "b"]), ["a", "b"])
    net.put_tensor("M2", UniTensor.ones([20, 20], labels=["a", "b"]), ["a", "b"])
    net.put_tensor("M3", UniTensor.ones([20, 2], labels=["a", "b"]), ["a", "b"])
    net.launch()
    assert net.get_order() == "((M1,M2),M3)"
    net.put_tensor("M1", UniTensor.ones([20, 20], labels=["a", "b"]), ["a", "b"])
    net.launch()
    assert net.get_order() == "((M2,M3),M1)"


@pytest.mark.parametrize("chi,dtype", [(128, np.float64), (64, np.complex128)])
def test_lawr_matvec_vs_oracle(cuda, chi, dtype):
    """BASELINE config C1 (chi=128 f64) and a complex variant against the oracle."""
    inp = oracle.lawr_inputs(chi, dtype=dtype, seed=31)
    want, tree = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp)
    net = Network(oracle.LAWR_NET)
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
    net.set_order(optimal=True)
    out = net.launch()
    assert net.get_order() == oracle.render_order(tree) == "(((A,L),W),R)"
    assert rel_fro(out.numpy(), want) <= 1e-12


def test_peps_small_vs_oracle_and_left_fold(cuda):
    """PEPS reading A at small size: the optimal launch equals the oracle's launch and the
    engine's own appearance-order left fold."""
    _, meta = load("network.npz")
    lines = meta["cases"][4]["net"]
    chi, D, d = 6, 3, 2
    shp = {"C0": [chi, chi], "C1": [chi, chi], "C2": [chi, chi], "C3": [chi, chi],
           "T0": [chi, D, D, chi], "T1": [chi, D, D, chi], "T2": [chi, D, D, chi], "T3": [chi, D, D, chi],
           "a": [D, D, D, D, d], "a*": [D, D, D, D, d]}
    net = Network(lines)
    arrays = {}
    for i, (nm, s) in enumerate(shp.items()):
        arrays[nm] = oracle.normal(s, seed=50 + i)
        t = UniTensor(storage.from_numpy(arrays[nm]), labels=[f"x{j}" for j in range(len(s))])
        net.put_tensor(nm, t)
    net.set_order(optimal=True)
    val = net.launch().item()
    want, tree = oracle.launch(oracle.net_slots(lines), "", arrays)
    assert net.get_order() == oracle.render_order(tree)
    want = np.asarray(want).item()  # rank-0 result
    assert abs(val - want) <= 1e-12 * max(1.0, abs(want))
    net2 = Network(lines)
    for nm in shp:
        net2.put_tensor(nm, net._bindings[nm][0])
    ref = net2.launch().item()  # appearance-order fold
    assert abs(val - ref) <= 1e-10 * max(1.0, abs(ref))


def test_launch_streams_result_to_host(cuda):
    """Network.launch(host_out=...) with chunk-uploaded operands (panel GEMMs, each panel
    streamed to the host as it completes) and without chunks: the host buffer holds the
    oracle's result after a synchronize."""
    import torch
    inp = oracle.lawr_inputs(48, seed=21)
    want, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp)
    net = Network(oracle.LAWR_NET)
    ts = {}
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(np.zeros_like(arr)), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
        ts[nm] = t
    net.set_order(optimal=True)
    host = torch.empty(want.size, dtype=torch.float64).pin_memory()
    for chunks in (1, 4):
        host.zero_()
        for nm in tree_leaves(parse_order(net.get_order())):
            ts[nm].get_block_().upload_(torch.from_numpy(np.ascontiguousarray(inp[nm])).pin_memory(), chunks=chunks)
        out = net.launch(host_out=host)
        torch.cuda.synchronize()
        got = host.numpy().reshape(want.shape)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want), chunks
        assert np.array_equal(out.numpy(), got)


def test_double_buffered_serving_loop(cuda):
    """The e2e serving loop of bench.py: two networks alternate, each refilling its inputs
    with upload_(..., after=net.done_event) (ordered only after the launch that last read
    them) while the other one computes; uneven chunk sizes; every step's host result
    equals the oracle's for that step's inputs."""
    import torch
    steps = 6
    inps = [oracle.lawr_inputs(40, seed=100 + s) for s in range(steps)]
    wants = [oracle.launch(oracle.lawr_slots(), "b, q, b2", inp)[0] for inp in inps]
    sets = []
    for _ in range(2):
        net = Network(oracle.LAWR_NET)
        ts = {}
        for nm, arr in inps[0].items():
            t = UniTensor(storage.from_numpy(np.zeros_like(arr)), labels=[f"{nm}{i}" for i in range(arr.ndim)])
            net.put_tensor(nm, t, t.labels)
            ts[nm] = t
        net.set_order(optimal=True)
        assert net.done_event is None
        sets.append((net, ts))
    pinned = [{nm: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for nm, a in inp.items()} for inp in inps]
    hosts = [torch.zeros(wants[0].size, dtype=torch.float64).pin_memory() for _ in range(steps)]
    order = tree_leaves(parse_order(sets[0][0].get_order()))
    for s in range(steps):
        net, ts = sets[s % 2]
        for nm in order:
            ts[nm].get_block_().upload_(pinned[s][nm], chunks=(1, 3, 2) if nm in ("L", "R") else 1,
                                        after=net.done_event)
        net.launch(host_out=hosts[s])
        assert net.done_event is not None
    torch.cuda.synchronize()
    for s in range(steps):
        got = hosts[s].numpy().reshape(wants[s].shape)
        assert np.linalg.norm(got - wants[s]) <= 1e-12 * np.linalg.norm(wants[s]), s


def test_upload_chunk_sizes(cuda):
    """upload_ with relative chunk sizes: boundaries on storage axis 0, all data lands."""
    import torch
    from paper_2401_01921_b200 import dense
    arr = np.random.default_rng(3).standard_normal((10, 7))
    t = storage.from_numpy(np.zeros_like(arr))
    t.upload_(torch.from_numpy(arr).pin_memory(), chunks=(1, 1, 3))
    ch = dense.pending_chunks(t)
    assert [r for r, _ in ch] == [(0, 2), (2, 4), (4, 10)]
    assert np.array_equal(t.numpy(), arr)
    with pytest.raises(ValueError):
        t.upload_(torch.from_numpy(arr).pin_memory(), chunks=(1, 0))


def test_launch_replay_program_matches_and_tracks_changes(cuda, monkeypatch):
    """Repeated dense launches replay the recorded steps (no order search, no validation
    pass, no per-step Python layout work) while the bindings keep their signature; any
    change -- in-place permute of a bound tensor, rebinding, relabelling, order change --
    falls back to the full launch and re-records. Results equal the oracle each time."""
    from paper_2401_01921_b200 import blueprint
    inp = oracle.lawr_inputs(24, seed=5)
    want, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp)
    net = Network(oracle.LAWR_NET)
    ts = {}
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
        ts[nm] = t
    net.set_order(optimal=True)
    first = net.launch()
    assert net._program is not None
    calls = []
    real = blueprint._execute
    monkeypatch.setattr(blueprint, "_execute", lambda *a: calls.append(1) or real(*a))
    for _ in range(3):
        out = net.launch()
        assert rel_fro(out.numpy(), want) <= 1e-12
        assert out.labels == first.labels and out.rowrank == first.rowrank and out.shape == first.shape
    assert not calls, "replay expected"
    assert net.get_order() == "(((A,L),W),R)"
    # in-place permute of a bound tensor (storage unchanged, logical axes swapped back by the binding order)
    L = ts["L"]
    L2 = UniTensor(storage.from_numpy(np.ascontiguousarray(inp["L"].transpose(2, 1, 0))), labels=["L2", "L1", "L0"])
    net.put_tensor("L", L2, ["L0", "L1", "L2"])
    out = net.launch()
    assert calls and rel_fro(out.numpy(), want) <= 1e-12
    calls.clear()
    out = net.launch()
    assert not calls and rel_fro(out.numpy(), want) <= 1e-12
    # mutate a bound tensor in place: A's block permuted lazily in place -> signature changes
    A = ts["A"]
    A.permute_([2, 1, 0])
    out = net.launch()  # binding order names the labels, so the result is unchanged
    assert calls and rel_fro(out.numpy(), want) <= 1e-12
    # a different dtype on rebinding: complex W
    calls.clear()
    Wc = UniTensor(storage.from_numpy(inp["W"].astype(np.complex128) * (1 + 1j)),
                   labels=[f"W{i}" for i in range(4)])
    net.put_tensor("W", Wc, Wc.labels)
    out = net.launch()
    assert calls and rel_fro(out.numpy(), want * (1 + 1j)) <= 1e-12
    calls.clear()
    out = net.launch()
    assert not calls and rel_fro(out.numpy(), want * (1 + 1j)) <= 1e-12


@pytest.mark.parametrize("seed", range(8))
def test_random_networks_vs_oracle(cuda, seed):
    """Random tree-shaped networks (3-6 tensors, ranks 1-4, dims 2-9, some open legs) with the
    optimal order: the DP order string equals the oracle's and the contracted result equals
    the oracle's launch within 1e-12 (f64; every other seed complex128)."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(3, 7))
    names = [f"T{i}" for i in range(n)]
    labels = {nm: [] for nm in names}
    dims = {}
    lab = 0
    for i in range(1, n):  # spanning tree: tensor i bonds to a random earlier tensor
        j = int(rng.integers(0, i))
        l = f"e{lab}"
        lab += 1
        labels[names[i]].append(l)
        labels[names[j]].append(l)
        dims[l] = int(rng.integers(2, 10))
    for _ in range(int(rng.integers(0, n))):  # extra loops between distinct tensors
        i, j = rng.choice(n, size=2, replace=False)
        if len(labels[names[i]]) < 4 and len(labels[names[j]]) < 4:
            l = f"e{lab}"
            lab += 1
            labels[names[i]].append(l)
            labels[names[j]].append(l)
            dims[l] = int(rng.integers(2, 6))
    opens = []
    for nm in names:  # open legs
        if len(labels[nm]) < 4 and rng.random() < 0.4:
            l = f"o{nm}"
            labels[nm].append(l)
            dims[l] = int(rng.integers(2, 6))
            opens.append(l)
    dtype = np.complex128 if seed % 2 else np.float64
    arrays = {}
    for k, nm in enumerate(names):
        shp = [dims[l] for l in labels[nm]]
        a = oracle.normal(shp, seed=100 * seed + k)
        if dtype == np.complex128:
            a = a + 1j * oracle.normal(shp, seed=100 * seed + 50 + k)
        arrays[nm] = a
    tout = ", ".join(opens)
    lines = [f"{nm}: {', '.join(labels[nm])}" for nm in names] + [f"TOUT: {tout}"]
    want, tree = oracle.launch([(nm, labels[nm]) for nm in names], tout, arrays)
    net = Network(lines)
    for nm in names:
        t = UniTensor(storage.from_numpy(arrays[nm]), labels=[f"x{i}" for i in range(arrays[nm].ndim)])
        net.put_tensor(nm, t, t.labels)
    net.set_order(optimal=True)
    out = net.launch()
    assert net.get_order() == oracle.render_order(tree)
    got = out.numpy() if opens else np.asarray(out.item())
    assert rel_fro(got, want) <= 1e-12


def test_repeated_small_launch_graph_replay_returns_fresh_results(cuda):
    """A latency-bound launch repeated on unchanged bindings is replayed from a captured CUDA
    graph after two eager replays. Every launch must still return a FRESH result (earlier
    results are not overwritten), follow in-place updates of the bound data, and stop using
    the graph when the bindings change."""
    import torch
    inp = oracle.lawr_inputs(24, seed=41)
    net = Network(oracle.LAWR_NET)
    ts = {}
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
        ts[nm] = t
    net.set_order(optimal=True)
    want, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp)
    outs = [net.launch() for _ in range(6)]
    assert net._program is not None and net._program.graph is not None
    for o in outs:
        assert rel_fro(o.numpy(), want) <= 1e-12
    assert len({o.get_block_().data_ptr for o in outs}) == len(outs)  # no aliasing between results
    # in-place update of a bound tensor's data: the graph reads the same buffer
    a2 = oracle.normal(inp["A"].shape, seed=99)
    ts["A"].get_block_().storage().copy_(torch.from_numpy(a2.reshape(-1)))
    inp2 = dict(inp, A=a2)
    want2, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp2)
    assert rel_fro(net.launch().numpy(), want2) <= 1e-12
    assert rel_fro(outs[0].numpy(), want) <= 1e-12  # earlier results untouched
    # rebinding: a new program (eager first)
    t = UniTensor(storage.from_numpy(inp["A"]), labels=["A0", "A1", "A2"])
    net.put_tensor("A", t, t.labels)
    assert rel_fro(net.launch().numpy(), want) <= 1e-12


@pytest.mark.parametrize("dt,mode", [(np.float64, 0), (np.complex128, 0), (np.complex128, 1)])
def test_contract_pair_output_order_vs_oracle(cuda, dt, mode):
    """contract_pair(out_order=...) (tnb_contract_dense_out): the same tensor, stored in the
    requested physical axis order and read back as a lazy permute."""
    from paper_2401_01921_b200 import contraction
    rng = np.random.default_rng(7)
    old = contraction._CPLX_MODE
    contraction.set_complex_mode("3M" if mode else "4M")
    try:
        for _ in range(6):
            al, bl = ["i", "k", "j", "m"], ["k", "n", "m", "p"]
            dims = {x: int(rng.integers(2, 40)) for x in "ijkmnp"}
            a = oracle.normal([dims[x] for x in al], dtype=dt, seed=int(rng.integers(1 << 30)))
            b = oracle.normal([dims[x] for x in bl], dtype=dt, seed=int(rng.integers(1 << 30)))
            oo = tuple(int(x) for x in rng.permutation(4))
            got = contract_pair(UniTensor(storage.from_numpy(a), labels=al), UniTensor(storage.from_numpy(b), labels=bl),
                                out_order=oo)
            want, wl = oracle.contract_dense(a, al, b, bl)
            assert got.labels == wl
            blk = got.get_block_()
            assert [blk.perm[x] for x in oo] == [0, 1, 2, 3]  # storage in the requested order
            assert rel_fro(got.numpy(), want) <= 1e-12
    finally:
        contraction._CPLX_MODE = old


def test_network_lays_out_long_k_intermediate(cuda):
    """A network whose root contraction is a few-tile, long-K GEMM (the PEPS closing-step
    shape at reduced size): the planner asks the right subtree for a K-major result; the
    launch (and its recorded replay) still equals the oracle."""
    from paper_2401_01921_b200 import blueprint
    lines = ["X: c0, u, c2, r, l, dn, s", "Y1: dn, dn2, c2, t", "Y2: t, c0, l, l2", "TOUT: u, r, s, dn2, l2"]
    dims = {"c0": 32, "u": 8, "c2": 32, "r": 8, "l": 8, "dn": 8, "s": 2, "dn2": 8, "l2": 8, "t": 16}
    slots = oracle.net_slots(lines)
    arrays = {n: oracle.normal([dims[x] for x in ls], seed=60 + i) for i, (n, ls) in enumerate(slots)}
    net = Network(lines)
    for n, ls in slots:
        net.put_tensor(n, UniTensor(storage.from_numpy(arrays[n]), labels=ls))
    net.set_order(contract_order="(X,(Y1,Y2))")
    tensors = {n: UniTensor(storage.from_numpy(arrays[n]), labels=ls) for n, ls in slots}
    lo, ro = blueprint._plan_children(("X", ("Y1", "Y2")), tensors)
    assert lo is None and ro is not None  # K = (c0, c2, l, dn) outermost in the intermediate
    want, _ = oracle.launch(slots, "u, r, s, dn2, l2", arrays, order="(X,(Y1,Y2))")
    for _ in range(3):  # eager, recorded, replayed
        got = net.launch()
        assert rel_fro(got.numpy(), want) <= 1e-12
