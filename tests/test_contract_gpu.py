"""a10/a11: dense pairwise contraction on DMMA vs the reference golden vectors and
the oracle (max abs <= 1e-12 on N(0,1) inputs like pkg/tests/test_contract.py:22-43;
relative Frobenius <= 1e-12 at benchmark sizes)."""
import numpy as np
import pytest

import tnkit_np as oracle
from tnb_testutil import load, rel_fro

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import UniTensor, contract, contract_pair, storage

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["4M", "3M"])
def cplx_mode(request):
    old = tnb.get_complex_mode()
    tnb.set_complex_mode(request.param)
    yield request.param
    tnb.set_complex_mode(old)


def test_golden_dense_contractions(cuda, cplx_mode):
    z, meta = load("dense.npz")
    for k, c in enumerate(meta["cases"]):
        a = UniTensor(storage.from_numpy(z[f"a{k}"]), labels=list(c["a_labels"]), name="A")
        if c["a_perm"] != list(range(len(c["a_perm"]))):
            a = a.permute(c["a_perm"])
        b = UniTensor(storage.from_numpy(z[f"b{k}"]), labels=list(c["b_labels"]), name="B")
        got = contract(a, b)
        assert got.labels == c["out_labels"]
        want = z[f"out{k}"]
        if got.rank:
            assert np.max(np.abs(got.numpy() - want)) <= 1e-12, k
        else:
            assert abs(got.item() - want[()]) <= 1e-12


def test_free_label_layout_and_ones(cuda):
    a = UniTensor.ones([2, 3, 5], labels=["i", "j", "l"], name="A")
    b = UniTensor.ones([3, 1, 5, 4], labels=["j", "k", "l", "m"], name="B")
    ab = contract(a, b)
    assert ab.labels == ["i", "k", "m"] and ab.shape == (2, 1, 4) and ab[0, 0, 0] == 15.0


def test_outer_scalar_and_identity_spine(cuda):
    ab = contract(UniTensor.ones([2], labels=["i"]), UniTensor.ones([3], labels=["j"]))
    assert ab.labels == ["i", "j"] and ab.shape == (2, 3) and np.all(ab.numpy() == 1)
    s = contract(UniTensor(storage.arange(4).reshape(2, 2), labels=["i", "j"]), UniTensor.ones([2, 2], labels=["i", "j"]))
    assert s.rank == 0 and s.item() == 6.0
    t = UniTensor(storage.arange(6).reshape(2, 3), labels=["i", "j"])
    summed = contract(t, UniTensor.ones([3], labels=["j"]))
    assert np.allclose(summed.numpy(), np.arange(6).reshape(2, 3).sum(axis=1))


def test_validation_before_arithmetic(cuda):
    from paper_2401_01921_b200 import IN, OUT, Bond, Symmetry
    ai = UniTensor([Bond(2, IN), Bond(2, OUT)], labels=["x", "y"])
    bi = UniTensor([Bond(2, IN), Bond(2, OUT)], labels=["y", "z"])
    contract(ai, bi)
    with pytest.raises(ValueError):
        contract(ai, bi.relabel(["x", "z"]))
    with pytest.raises(ValueError):
        contract(ai, UniTensor.ones([2, 2], labels=["y", "z"]))
    with pytest.raises(ValueError):
        contract(UniTensor.ones([2, 3], labels=["i", "j"]), UniTensor.ones([4, 2], labels=["j", "k"]))
    with pytest.raises(ValueError):
        contract(UniTensor.ones([2, 2], labels=["i", "k"]), UniTensor.ones([3, 2], labels=["i", "k"]))
    with pytest.raises(TypeError):
        contract(UniTensor.ones([2, 2], labels=["i", "k"], dtype=tnb.Int64),
                 UniTensor.ones([2, 2], labels=["k", "j"], dtype=tnb.Int64))


@pytest.mark.parametrize("seed", range(6))
def test_random_labelled_pairs_vs_oracle(cuda, seed):
    rng = np.random.default_rng(100 + seed)
    for _ in range(10):
        ra, rb = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        labels = [f"l{i}" for i in range(10)]
        rng.shuffle(labels)
        al = labels[:ra]
        ns = int(rng.integers(0, min(ra, rb) + 1))
        bl = al[:ns] + labels[ra:ra + rb - ns]
        rng.shuffle(bl)
        dims = {l: int(rng.integers(1, 9)) for l in set(al) | set(bl)}
        dt = np.complex128 if rng.random() < 0.3 else np.float64
        a = oracle.normal([dims[l] for l in al], dtype=dt, seed=int(rng.integers(1 << 30)))
        b = oracle.normal([dims[l] for l in bl], dtype=dt, seed=int(rng.integers(1 << 30)))
        perm = [int(x) for x in rng.permutation(ra)]
        A = UniTensor(storage.from_numpy(a), labels=list(al)).permute([al[p] for p in perm])
        got = contract(A, UniTensor(storage.from_numpy(b), labels=list(bl)))
        want, wl = oracle.contract_dense(a.transpose(perm), [al[p] for p in perm], b, bl)
        assert got.labels == wl
        g = got.numpy() if got.rank else got.item()
        assert np.max(np.abs(g - want)) <= 1e-12


@pytest.mark.parametrize("m,n,k", [(1, 1, 100000), (2048, 5120, 96), (300, 257, 1031), (7, 4096, 13),
                                   (100000, 10, 10), (4096, 3, 64)])
def test_gemm_shapes_vs_numpy(cuda, m, n, k):
    a = oracle.normal([m, k], seed=1)
    b = oracle.normal([k, n], seed=2)
    got = contract(UniTensor(storage.from_numpy(a), labels=["m", "k"]),
                   UniTensor(storage.from_numpy(b), labels=["k", "n"]))
    want = a @ b
    assert rel_fro(got.numpy() if got.rank else got.item(), want) <= 1e-13


def test_mixed_dtype_promotes(cuda):
    a = oracle.normal([8, 9], seed=3)
    b = oracle.normal([9, 5], dtype=np.complex128, seed=4)
    got = contract(UniTensor(storage.from_numpy(a), labels=["i", "k"]), UniTensor(storage.from_numpy(b), labels=["k", "j"]))
    assert got.dtype == np.complex128 and np.max(np.abs(got.numpy() - a @ b)) <= 1e-12


def test_inputs_not_mutated_and_output_fresh(cuda):
    a = UniTensor(storage.from_numpy(oracle.normal([5, 6], seed=1)), labels=["i", "j"])
    b = UniTensor(storage.from_numpy(oracle.normal([6, 7], seed=2)), labels=["j", "k"])
    a0, b0 = a.numpy().copy(), b.numpy().copy()
    c = contract_pair(a, b)
    assert np.array_equal(a.numpy(), a0) and np.array_equal(b.numpy(), b0)
    assert not c.same_data(a) and not c.same_data(b)


def test_async_upload_is_awaited_by_the_consumer(cuda):
    """upload_ copies on the engine's copy stream; a contraction issued right after it
    (on the compute stream) must see the NEW data, for dense and block-sparse operands,
    and a pending upload must not be overtaken by a later upload into the same buffer."""
    import torch
    rng = np.random.default_rng(7)
    a0, b0 = rng.standard_normal((300, 200)), rng.standard_normal((200, 100))
    a1, b1 = rng.standard_normal((300, 200)), rng.standard_normal((200, 100))
    A = UniTensor(storage.from_numpy(a0), labels=["i", "k"])
    B = UniTensor(storage.from_numpy(b0), labels=["k", "j"])
    contract(A, B)
    for _ in range(3):
        A.get_block_().upload_(torch.from_numpy(a1).pin_memory())
        B.get_block_().upload_(b1)
        got = contract(A, B).numpy()
        assert rel_fro(got, a1 @ b1) <= 1e-13
        A.get_block_().upload_(torch.from_numpy(a0).pin_memory())
        A.get_block_().upload_(torch.from_numpy(a1).pin_memory())  # WAR/WAW on one buffer
        assert rel_fro(contract(A, B).numpy(), a1 @ b1) <= 1e-13
    with pytest.raises(ValueError):
        A.get_block_().upload_(np.zeros(7))
    with pytest.raises(TypeError):
        A.get_block_().upload_(np.zeros((300, 200), dtype=np.complex128))


@pytest.mark.parametrize("dt", [np.float64, np.complex128])
def test_dispatch_paths_dot_and_half_tiles(cuda, dt, cplx_mode):
    """Every GEMM dispatch path against numpy: M*N <= 16 (dot kernel + ordered CTA reduce),
    N = 64 / M = 64 / N = 192 (128x64 and 64x128 stream-K tiles), permuted operands."""
    rng = np.random.default_rng(31)

    def arr(shape):
        x = rng.standard_normal(shape)
        if dt == np.complex128:
            x = x + 1j * rng.standard_normal(shape)
        return x.astype(dt)

    cases = [((1, 10007), (10007, 1)), ((3, 777), (777, 5)), ((16, 4096), (4096, 1)),
             ((300, 500), (500, 64)), ((64, 500), (500, 300)), ((257, 129), (129, 192))]
    for (m, k), (k2, n) in cases:
        a, b = arr((k, m)), arr((n, k2))  # stored transposed: the contraction reads permuted views
        A = UniTensor(storage.from_numpy(a), labels=["k", "m"]).permute(["m", "k"])
        B = UniTensor(storage.from_numpy(b), labels=["n", "k"]).permute(["k", "n"])
        got = contract(A, B).numpy()
        want = a.T @ b.T
        assert rel_fro(got, want) <= 1e-13, ((m, k, n), rel_fro(got, want))
    # deterministic: a second call is bit-identical
    A = UniTensor(storage.from_numpy(arr((2, 50000))), labels=["m", "k"])
    B = UniTensor(storage.from_numpy(arr((50000, 3))), labels=["k", "n"])
    assert np.array_equal(contract(A, B).numpy(), contract(A, B).numpy())


def test_small_problem_tiles(cuda):
    """chi = 128 L.A.W.R-sized steps take the 64 x 64 stream-K tiles: parity vs numpy."""
    rng = np.random.default_rng(5)
    for (m, k, n) in [(256, 128, 640), (200, 640, 100), (65, 33, 70)]:
        a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
        A = UniTensor(storage.from_numpy(a), labels=["m", "k"])
        B = UniTensor(storage.from_numpy(b), labels=["k", "n"])
        assert rel_fro(contract(A, B).numpy(), a @ b) <= 1e-13


def test_chunked_upload_pipelines_panels(cuda):
    """upload_(..., chunks=k) + contraction: panel-by-panel GEMMs (each waiting for its own
    chunk) give the same result as a plain contraction -- when the right operand's outermost
    storage axis is its first free axis (panels), and when it is not (whole wait)."""
    import torch
    rng = np.random.default_rng(17)
    a = rng.standard_normal((37, 6, 29))            # [vl, p, vr]
    l0, l1 = rng.standard_normal((2, 64, 5, 37))    # [b, w, vl]
    A = UniTensor(storage.from_numpy(a), labels=["vl", "p", "vr"])
    L = UniTensor(storage.from_numpy(l0), labels=["b", "w", "vl"])
    want = np.einsum("xpv,bwx->pvbw", a, l1)
    for k in (1, 3, 4, 64):
        L.get_block_().upload_(torch.from_numpy(l1).pin_memory(), chunks=k)
        got = contract(A, L).numpy()
        assert rel_fro(got, want) <= 1e-13, k
        L.get_block_().upload_(torch.from_numpy(l0).pin_memory(), chunks=k)
        assert rel_fro(contract(A, L).numpy(), np.einsum("xpv,bwx->pvbw", a, l0)) <= 1e-13
    # outermost storage axis contracted (b is the contracted label here): whole-tensor wait
    B = UniTensor(storage.from_numpy(l0), labels=["vr", "w", "z"])
    B.get_block_().upload_(torch.from_numpy(rng.standard_normal((64, 5, 37))).pin_memory(), chunks=4)
    A2 = UniTensor(storage.from_numpy(rng.standard_normal((3, 64))), labels=["y", "vr"])
    ref = A2.get_block_().numpy() @ B.get_block_().numpy().reshape(64, -1)
    assert rel_fro(contract(A2, B).numpy().reshape(3, -1), ref) <= 1e-13
    # lazily permuted operand: outermost storage axis is not the first free logical axis
    P = L.permute(["w", "b", "vl"])
    P.get_block_().upload_(torch.from_numpy(l1).pin_memory(), chunks=4)
    assert rel_fro(contract(A, P).numpy(), np.einsum("xpv,bwx->pvwb", a, l1)) <= 1e-13


def test_streamk_workspace_across_streams_and_graphs(cuda):
    """Eager stream-K launches share one persistent workspace (owner-reset flags); launches
    on different streams are serialised on it by an event, and a captured CUDA graph owns
    its own workspace. Interleave eager launches on two streams with graph replays on a
    third, many times, and check every result (and that the results are bit-identical to
    a lone launch: the stream-K fix-up order is fixed)."""
    import torch
    rng = np.random.default_rng(11)
    a = rng.standard_normal((384, 640))
    b = rng.standard_normal((640, 320))
    want = a @ b
    A = UniTensor(storage.from_numpy(a), labels=["i", "k"])
    B = UniTensor(storage.from_numpy(b), labels=["k", "j"])
    ref = contract_pair(A, B).numpy()
    assert np.linalg.norm(ref - want) <= 1e-12 * np.linalg.norm(want)
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    net = tnb.Network(["A: i, k", "B: k, j", "TOUT: i; j"])
    net.put_tensor("A", A)
    net.put_tensor("B", B)
    torch.cuda.synchronize()
    with torch.cuda.stream(s3):
        cn = net.compile()
    outs = []
    for it in range(20):
        for st in (s1, s2):
            with torch.cuda.stream(st):
                outs.append((st, contract_pair(A, B)))
        with torch.cuda.stream(s3):
            outs.append((s3, cn.launch()))
    torch.cuda.synchronize()
    for st, o in outs:
        got = o.numpy()
        assert np.array_equal(got, ref), "stream-K result differs across streams / graph replays"


@pytest.mark.timeout(300)
def test_stream_k_gemms_run_beside_a_long_kernel_stream(cuda):
    """The persistent stream-K GEMMs (dense and grouped block-sparse) hand partials between
    CTAs; they are launched cooperatively, so they are co-scheduled as a whole even while
    another stream keeps SMs busy with long kernels. Results stay exact and nothing hangs."""
    import torch
    import bench
    inp = oracle.lawr_inputs(96, seed=8)
    want, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp)
    net, _ = bench.make_network(tnb, oracle.LAWR_NET, inp)
    A, E = bench.c4_tensors(tnb, seed=5)
    ref_bs = [b.numpy() for b in tnb.contract(A, E).get_blocks_()]
    side = torch.cuda.Stream()
    x = torch.randn(4096, 4096, dtype=torch.float64, device=cuda)
    with torch.cuda.stream(side):
        for _ in range(12):  # ~0.1 s of DGEMMs occupying every SM, queued ahead
            y = x @ x
    for _ in range(5):
        out = net.launch().numpy()
        got_bs = [b.numpy() for b in tnb.contract(A, E).get_blocks_()]
    torch.cuda.synchronize()
    assert rel_fro(out, want) <= 1e-12
    assert all(np.array_equal(g, w) for g, w in zip(got_bs, ref_bs))
    del y


@pytest.mark.parametrize("dt", [np.float64, np.complex128])
def test_narrow_row_panel_path(cuda, dt):
    """The T1.W layout (T1[p][vr][b][w], contracted (w, p) -- the stride-1 digit w, rows
    stepping by its extent): narrow_slab_kernel's staged row panels vs numpy, for both
    orders of the contracted labels, odd / even inner extents and several outer extents."""
    rng = np.random.default_rng(77)

    def arr(shape):
        x = rng.standard_normal(shape)
        if dt == np.complex128:
            x = x + 1j * rng.standard_normal(shape)
        return x.astype(dt)

    for (p, vr, b, w, w2, q) in [(2, 64, 128, 5, 5, 2), (2, 64, 64, 4, 3, 2), (3, 8, 512, 3, 2, 5), (1, 4, 1024, 10, 16, 1),
                                 (2, 64, 64, 3, 3, 1), (2, 32, 256, 5, 5, 2)]:
        t1, W = arr((p, vr, b, w)), arr((w, w2, q, p))
        T1 = UniTensor(storage.from_numpy(t1), labels=["p", "vr", "b", "w"])
        for wl, wperm in ((["w", "w2", "q", "p"], W), (["p", "q", "w2", "w"], W.transpose(3, 2, 1, 0).copy())):
            Wt = UniTensor(storage.from_numpy(wperm), labels=wl)
            got = contract(T1, Wt)
            want = np.einsum("pvbw,wxqp->vbxq", t1, W)
            if wl[1] == "q":
                want = want.transpose(0, 1, 3, 2)
            assert rel_fro(got.numpy(), want) <= 1e-13, ((p, vr, b, w), wl)


def test_long_gathered_k_few_tiles_vs_oracle(cuda):
    """The PEPS closing-step shape at reduced chi (M = 128, N = 64, K = 65536 over four
    interleaved digits, the free s axis innermost in A): the 32-wide k-tile stream-K
    instantiation (dispatch: few output tiles, irregular K >= 2^16) against the oracle."""
    al = ["c0", "u", "c2", "r", "l", "dn", "s"]
    bl = ["dn", "dn2", "c2", "c0", "l", "l2"]
    dims = {"c0": 32, "u": 8, "c2": 32, "r": 8, "l": 8, "dn": 8, "s": 2, "dn2": 8, "l2": 8}
    a = oracle.normal([dims[x] for x in al], seed=41)
    b = oracle.normal([dims[x] for x in bl], seed=42)
    got = contract(UniTensor(storage.from_numpy(a), labels=al), UniTensor(storage.from_numpy(b), labels=bl))
    want, wl = oracle.contract_dense(a, al, b, bl)
    assert got.labels == wl == ["u", "r", "s", "dn2", "l2"]
    assert rel_fro(got.numpy(), want) <= 1e-12
