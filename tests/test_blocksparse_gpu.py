"""a12: block-sparse contraction -- device pairing table bit-exact (i, j, out) in
reference order; results within 1e-12 of the reference / oracle."""
import numpy as np
import pytest

import tnkit_np as oracle
from tnb_testutil import bonds_from_meta, load, rel_fro

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import IN, Bond, Symmetry, UniTensor, block_pairs, contract, storage
from paper_2401_01921_b200 import random as trandom

pytestmark = pytest.mark.gpu


def _payload(blocks):
    """Every block's elements, concatenated in block order (a slab's alignment padding
    between blocks is never written and holds whatever the allocator left there)."""
    import torch
    return torch.cat([b.storage().reshape(-1) for b in blocks])


def test_golden_block_sparse_cases(cuda):
    z, meta = load("blocks.npz")
    for k, c in enumerate(meta["cases"]):
        perm = c["a_perm"]
        inv = [perm.index(i) for i in range(len(perm))]
        a_labels_storage = [c["a_labels"][inv[i]] for i in range(len(perm))]
        a_bonds_storage = [c["a_bonds"][inv[i]] for i in range(len(perm))]
        a = UniTensor(bonds_from_meta(a_bonds_storage), labels=a_labels_storage, dtype=np.dtype(c["dtype"]))
        import torch
        for i in range(a.nblocks):
            a.get_block_(i).storage().copy_(torch.from_numpy(z[f"c{k}_a{i}"].reshape(-1)))
        if perm != list(range(len(perm))):
            a = a.permute(c["a_labels"])
        assert [list(q) for q in a._qns] == c["a_qns"]
        b = UniTensor(bonds_from_meta(c["b_bonds"]), labels=c["b_labels"])
        for j in range(b.nblocks):
            b.get_block_(j).storage().copy_(torch.from_numpy(z[f"c{k}_b{j}"].reshape(-1)))
        out = contract(a, b)
        assert out.labels == c["out_labels"]
        if "out_qns" not in c:
            assert abs(out.item() - z[f"c{k}_scalar"][()]) <= 1e-12
            continue
        assert [list(q) for q in out._qns] == c["out_qns"]
        for i in range(out.nblocks):
            assert np.max(np.abs(out.get_block_(i).numpy() - z[f"c{k}_out{i}"])) <= 1e-12, (k, i)
        trip = block_pairs(a, b)
        assert trip.tolist() == c["triples"], k


def _c4():
    _, meta = load("c4.npz")
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(q, d) for q, d in meta["sectors"]], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
    E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
    trandom.normal_(A, seed=meta["seed"])
    trandom.normal_(E, seed=meta["seed"] + 1)
    return A, E, meta


def test_c4_full_size_pairing_bitexact(cuda):
    A, E, meta = _c4()
    assert [list(q) for q in A._qns] == meta["a_qns"] and [list(q) for q in E._qns] == meta["e_qns"]
    assert block_pairs(A, E).tolist() == meta["triples"]


def test_c4_full_size_values(cuda):
    z, _ = load("c4.npz")
    A, E, meta = _c4()
    out = contract(A, E)
    assert out.labels == meta["out_labels"] and [list(q) for q in out._qns] == meta["out_qns"]
    ab = [b.numpy() for b in A.get_blocks_()]
    eb = [b.numpy() for b in E.get_blocks_()]
    res, trip = oracle.contract_blocks(A._qns, ab, A.labels, E._qns, eb, E.labels, out._qns)
    got = [b.numpy() for b in out.get_blocks_()]
    num = sum(np.linalg.norm(g - r) ** 2 for g, r in zip(got, res))
    den = sum(np.linalg.norm(r) ** 2 for r in res)
    assert np.sqrt(num / den) <= 1e-12
    assert np.allclose([np.linalg.norm(g) for g in got], z["norms"], rtol=1e-12, atol=0)


def test_output_flux_zero_and_lazy_permuted_operand(cuda):
    u1 = Symmetry.u1()
    mid = Bond(btype=tnb.OUT, sectors=[(2, 1), (0, 2), (-2, 1)], syms=[u1])
    leg = Bond(btype=IN, sectors=[(1, 2), (-1, 1)], syms=[u1])
    a = UniTensor([leg, leg, mid], labels=["x", "y", "s"])
    b = UniTensor([mid.redirect(), mid], labels=["s", "z"])
    trandom.normal_(a, seed=8)
    trandom.normal_(b, seed=9)
    direct = contract(a, b)
    perm = contract(a.permute(["s", "x", "y"]), b)
    assert (direct - perm.permute(direct.labels)).norm() <= 1e-13
    for i in range(direct.nblocks):
        flux = sum(q[0] if bd.btype == IN else -q[0] for bd, q in zip(direct.bonds, direct.block_qnums(i)))
        assert flux == 0


def test_blocks_without_pairs_are_zero(cuda):
    u1 = Symmetry.u1()
    b1 = Bond(btype=IN, sectors=[(0, 2), (5, 3)], syms=[u1])
    a = UniTensor([b1, b1.redirect()], labels=["i", "j"])
    b = UniTensor([b1, b1.redirect()], labels=["j", "k"])
    trandom.normal_(a, seed=1)
    trandom.normal_(b, seed=2)
    # poison the freshly allocated output: the kernel must overwrite every block
    out = contract(a, b)
    for i in range(out.nblocks):
        q = out.block_qn_indices(i)
        want = a.get_block_(q[0:1] + (q[0],)).numpy() @ b.get_block_((q[0], q[1])).numpy()
        assert np.max(np.abs(out.get_block_(i).numpy() - want)) <= 1e-12


def test_panel_masked_partition_reassembles(cuda):
    """Multi-GPU partition emulated on one GPU: each 'rank' computes only its LPT panels
    (panel mask through the C ABI); stitching the panels gives the unpartitioned result
    (the full K reduction of every panel is local). The stream-K split of the k-iterations
    depends on how much work a launch holds, so the summation order -- and the last bits --
    can differ from the single-launch result: tolerance 1e-13 relative per panel."""
    import torch
    from paper_2401_01921_b200 import contraction as C
    from paper_2401_01921_b200 import parallel as P
    from paper_2401_01921_b200.labeled import zero_flux_combos
    A, E, meta = _c4()
    full = contract(A, E)
    a_pos, b_pos, a_free, b_free, out_labels, out_bonds = C._pair_layout(A, E)
    qns = zero_flux_combos(out_bonds)
    shapes = [tuple(x.sectors[k][1] for x, k in zip(out_bonds, qn)) for qn in qns]
    ktot = P.block_pair_k(A._qns, [b.shape for b in A._blocks], a_pos, E._qns, b_pos, a_free, b_free, qns)
    for world in (2, 3, 8):
        panels, owner = P.panel_plan(shapes, len(a_free), ktot, world)
        stitched = None
        for rank in range(world):
            mask = np.array([1 if o == rank else 0 for o in owner], dtype=np.uint8)
            part = C._contract_blocks(A, E, a_pos, b_pos, a_free, b_free, out_labels, out_bonds, panel_mask=mask)
            slab = part._blocks[0]._slab
            spans = P.panel_spans(panels, [blk._off for blk in part._blocks])
            if stitched is None:
                stitched = torch.zeros_like(slab)
            for (s, n), o in zip(spans, owner):
                if o == rank:
                    stitched[s:s + n] = slab[s:s + n]
        ref = full._blocks[0]._slab
        spans = P.panel_spans(panels, [blk._off for blk in full._blocks])
        for s, n in spans:
            err = torch.linalg.norm(stitched[s:s + n] - ref[s:s + n]).item()
            assert err <= 1e-13 * max(torch.linalg.norm(ref[s:s + n]).item(), 1e-300), (s, n, err)


def test_grouped_stream_k_is_deterministic(cuda):
    """Same structure, same inputs -> bit-identical output on every call (fixed stream-K
    split, partials added in CTA order, no data atomics), eager and graph-replayed."""
    import torch
    from paper_2401_01921_b200 import graphs
    A, E, _ = _c4()
    first = _payload(contract(A, E)._blocks).clone()
    for _ in range(3):
        assert torch.equal(_payload(contract(A, E)._blocks), first)
    g = graphs.capture(lambda: contract(A, E))
    for _ in range(3):
        out = g.replay()
        torch.cuda.synchronize()
        assert torch.equal(_payload(out._blocks), first)


def test_one_shot_abi_matches_plan_execute(cuda):
    """tnb_bs_contract_masked (one call: plan + execute + pairs) and the split
    tnb_bs_plan / tnb_bs_execute / tnb_bs_plan_pairs give identical bits and triples."""
    import torch
    from paper_2401_01921_b200 import _lib, dense
    from paper_2401_01921_b200 import contraction as C
    from paper_2401_01921_b200.labeled import _slab_blocks, zero_flux_combos
    A, E, _ = _c4()
    a_pos, b_pos, a_free, b_free, out_labels, out_bonds = C._pair_layout(A, E)
    qns = zero_flux_combos(out_bonds)
    shapes = [tuple(x.sectors[k][1] for x, k in zip(out_bonds, qn)) for qn in qns]
    oblk, slab = _slab_blocks(shapes, np.dtype(np.float64), zero=False)
    trip = _lib.bs_contract(_lib.TNB_F64, A._qns, [x.storage_shape for x in A._blocks], tuple(range(3)),
                            E._qns, [x.storage_shape for x in E._blocks], tuple(range(3)), a_pos, b_pos,
                            qns, shapes, [x.data_ptr for x in A._blocks], [x.data_ptr for x in E._blocks],
                            [x.data_ptr for x in oblk], dense.stream_handle(), want_pairs=True)
    ref = contract(A, E)
    torch.cuda.synchronize()
    assert torch.equal(_payload(oblk), _payload(ref._blocks))
    assert trip.tolist() == block_pairs(A, E).tolist()


def test_contract_batched_equals_pairwise(cuda):
    """contract_batched: ONE grouped launch over the output tiles of several equal-structure
    block-sparse contractions (full C4 size); every result matches its own contract_pair
    to 1e-13 relative (same per-tile pair order; the batch changes the stream-K split, so
    partial sums are added at different k boundaries)."""
    import bench
    pairs = [bench.c4_tensors(tnb, seed=900 + 2 * i) for i in range(5)]
    outs = tnb.contract_batched(pairs)
    assert len(outs) == 5
    for (A, E), got in zip(pairs, outs):
        want = tnb.contract_pair(A, E)
        assert got.labels == want.labels and got._qns == want._qns
        for gb, wb in zip(got.get_blocks_(), want.get_blocks_()):
            g, w = gb.numpy(), wb.numpy()
            assert g.shape == w.shape
            assert np.linalg.norm(g - w) <= 1e-13 * max(np.linalg.norm(w), 1e-300)


def test_contract_batched_small_structures_and_errors(cuda):
    """Several small U1 structures: batched == pairwise; pointer tables both inline (few
    blocks) and device-staged (many items); mixed structures raise ValueError."""
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-1, 3), (0, 4), (1, 2)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    def mk(seed, V=V):
        A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
        E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
        tnb.random.normal_(A, seed=seed)
        tnb.random.normal_(E, seed=seed + 1)
        return A, E
    for n in (2, 40):  # 2 x 15 pointers: 1 KB parameter table; 40 x 15: the 8 KB one
        pairs = [mk(50 + 2 * i) for i in range(n)]
        outs = tnb.contract_batched(pairs)
        for (A, E), got in zip(pairs, outs):
            want = tnb.contract_pair(A, E)
            for gb, wb in zip(got.get_blocks_(), want.get_blocks_()):
                assert np.linalg.norm(gb.numpy() - wb.numpy()) <= 1e-13 * max(np.linalg.norm(wb.numpy()), 1e-300)
    many = [mk(300 + 2 * i) for i in range(80)]  # 80 x 15 = 1200 pointers: device table
    outs = tnb.contract_batched(many)
    for (A, E), got in zip(many[::13], outs[::13]):
        want = tnb.contract_pair(A, E)
        for gb, wb in zip(got.get_blocks_(), want.get_blocks_()):
            assert np.linalg.norm(gb.numpy() - wb.numpy()) <= 1e-13 * max(np.linalg.norm(wb.numpy()), 1e-300)
    V2 = Bond(btype=IN, sectors=[(-1, 3), (0, 5), (1, 2)], syms=[u1])
    with pytest.raises(ValueError, match="block structure"):
        tnb.contract_batched([mk(1), mk(3, V=V2)])
    with pytest.raises(TypeError):
        tnb.contract_batched([(1, 2)])


def test_contract_batched_complex_and_permuted(cuda):
    """Batched execute on complex128 blocks and on lazily permuted operands (shared perm)."""
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-2, 2), (-1, 3), (0, 5), (1, 4), (2, 1)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])

    def mk(seed, dtype):
        A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"], dtype=dtype)
        E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"], dtype=dtype)
        trandom.normal_(A, seed=seed)
        trandom.normal_(E, seed=seed + 1)
        return A, E

    for dtype in (storage.Float64, storage.Complex128):
        pairs = [mk(70 + 2 * i, dtype) for i in range(6)]
        pairs = [(A.permute(["vr", "vl", "p"]), E) for A, E in pairs]  # lazy, same perm for all
        outs = tnb.contract_batched(pairs)
        for (A, E), got in zip(pairs, outs):
            want = tnb.contract_pair(A, E)
            assert got.labels == want.labels
            for gb, wb in zip(got.get_blocks_(), want.get_blocks_()):
                w = wb.numpy()
                assert np.linalg.norm(gb.numpy() - w) <= 1e-13 * max(np.linalg.norm(w), 1e-300)


def test_contract_batched_graph_capture_large_table(cuda):
    """A batched contraction whose pointer table exceeds the kernel parameter (device table
    staged from pinned memory) captured in a CUDA graph: replays reproduce the eager result
    even after later eager calls reused the staging ring."""
    import torch
    from paper_2401_01921_b200 import graphs
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-1, 3), (0, 4), (1, 2)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])

    def mk(seed):
        A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
        E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
        trandom.normal_(A, seed=seed)
        trandom.normal_(E, seed=seed + 1)
        return A, E

    pairs = [mk(400 + 2 * i) for i in range(80)]  # 80 x 15 = 1200 pointers > 1024
    want = [o.get_blocks_()[1].numpy() for o in tnb.contract_batched(pairs)]
    holder = {}
    g = graphs.capture(lambda: holder.__setitem__("outs", tnb.contract_batched(pairs)), warmup=1)
    other = [mk(900 + 2 * i) for i in range(80)]
    for _ in range(10):  # cycle the eager staging ring past its 8 slots
        tnb.contract_batched(other)
    g.replay()
    torch.cuda.synchronize()
    for k in (0, 37, 79):
        got = holder["outs"][k].get_blocks_()[1].numpy()
        assert np.linalg.norm(got - want[k]) <= 1e-13 * np.linalg.norm(want[k])


@pytest.mark.parametrize("seed", range(16))
def test_random_block_sparse_pairs_vs_oracle(cuda, seed):
    """Randomised structures: U1 / Z2 / Z3 / U1 x Z2 bonds with random sectors and
    degeneracies, rank-3/4 operands sharing one or two legs (opposite directions), a
    random lazy permute of each operand; pairing triples bit-exact and every output block
    within 1e-12 (relative Frobenius) of the oracle's _contract_pair_blocks restatement."""
    from paper_2401_01921_b200.charges import OUT
    rng = np.random.default_rng(1000 + seed)
    sym_sets = [[Symmetry.u1()], [Symmetry.zn(2)], [Symmetry.zn(3)], [Symmetry.u1(), Symmetry.zn(2)]]
    syms = sym_sets[seed % len(sym_sets)]

    def rand_q():
        return tuple(int(rng.integers(-2, 3)) if s.modulus == 0 else int(rng.integers(0, s.modulus)) for s in syms)

    def rand_bond(btype):
        qs = [tuple(0 for _ in syms)]  # the identity charge on every bond: zero flux is reachable
        while len(qs) < int(rng.integers(2, 5)):
            q = rand_q()
            if q not in qs:
                qs.append(q)
        return Bond(btype=btype, sectors=[(q, int(rng.integers(1, 5))) for q in qs], syms=syms)

    ra, rb = int(rng.integers(3, 5)), int(rng.integers(3, 5))
    nsh = int(rng.integers(1, 3))
    a_bonds = [rand_bond(IN if rng.random() < 0.5 else OUT) for _ in range(ra)]
    shared = list(rng.choice(ra, size=nsh, replace=False))
    b_bonds = [a_bonds[i].redirect() for i in shared] + [rand_bond(IN if rng.random() < 0.5 else OUT)
                                                         for _ in range(rb - nsh)]
    a_labels = [f"a{i}" for i in range(ra)]
    b_labels = [a_labels[i] for i in shared] + [f"b{i}" for i in range(rb - nsh)]
    try:
        A = UniTensor(a_bonds, labels=a_labels)
        B = UniTensor(b_bonds, labels=b_labels)
    except ValueError:
        pytest.skip("no zero-flux block for this draw")
    trandom.normal_(A, seed=seed)
    trandom.normal_(B, seed=seed + 100)
    A = A.permute(list(rng.permutation(a_labels)))
    B = B.permute(list(rng.permutation(b_labels)))
    try:
        out = contract(A, B)
    except ValueError as e:
        assert "no valid blocks" in str(e)
        pytest.skip("output has no zero-flux block")
    a_np = [blk.numpy() for blk in A.get_blocks_()]
    b_np = [blk.numpy() for blk in B.get_blocks_()]
    want, triples = oracle.contract_blocks(A._qns, a_np, A.labels, B._qns, b_np, B.labels, out._qns)
    got_pairs = [tuple(int(x) for x in r) for r in block_pairs(A, B)]
    assert got_pairs == [tuple(t) for t in triples]
    shapes = [blk.shape for blk in out.get_blocks_()]
    want = oracle.finish_blocks(want, shapes, np.float64)
    for blk, w in zip(out.get_blocks_(), want):
        g = blk.numpy()
        assert g.shape == w.shape
        assert rel_fro(g, w) <= 1e-12 or np.linalg.norm(w) == 0 and np.abs(g).max() == 0


def test_contract_batched_mixed_dtype_conversions_stay_alive(cuda):
    """float64 x complex128 batch: every pair's A blocks are widened to complex128 on the
    fly (fresh allocations). Those must live until the one grouped launch has run; each
    result equals its own contract_pair (converted blocks were freed early)."""
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-2, 9), (-1, 17), (0, 24), (1, 15), (2, 8)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    pairs = []
    for i in range(12):
        A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"], dtype=storage.Float64)
        E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"], dtype=storage.Complex128)
        trandom.normal_(A, seed=400 + 2 * i)
        trandom.normal_(E, seed=401 + 2 * i)
        pairs.append((A, E))
    outs = tnb.contract_batched(pairs)
    for (A, E), got in zip(pairs, outs):
        want = tnb.contract_pair(A, E)
        assert got.dtype == np.complex128
        for gb, wb in zip(got.get_blocks_(), want.get_blocks_()):
            w = wb.numpy()
            assert np.linalg.norm(gb.numpy() - w) <= 1e-13 * max(np.linalg.norm(w), 1e-300)


def test_captured_graph_survives_workspace_growth_and_plan_flush(cuda):
    """A captured block-sparse graph owns its stream-K workspace and keeps its plan alive:
    after eager calls that grow the shared workspace (complex128 needs twice the partials)
    and after more than 256 new structures flush the library's plan cache, replays still
    reproduce the eager result bit for bit."""
    import torch
    from paper_2401_01921_b200 import graphs
    A, E, _ = _c4()
    first = _payload(contract(A, E)._blocks).clone()
    g = graphs.capture(lambda: contract(A, E))
    out = g.replay()
    torch.cuda.synchronize()
    assert torch.equal(_payload(out._blocks), first)
    # eager complex128 contraction: larger workspace (reallocation of the shared one)
    contract(A.astype(storage.Complex128), E)
    u1 = Symmetry.u1()
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    for n in range(1, 270):  # > 256 distinct structures: the library flushes its plan cache
        V = Bond(btype=IN, sectors=[(-1, 1 + n % 7), (0, 1 + n // 7), (1, 2)], syms=[u1])
        a = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
        e = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
        contract(a, e)
    for _ in range(3):
        out = g.replay()
        torch.cuda.synchronize()
        assert torch.equal(_payload(out._blocks), first)
    # eager calls after the flush re-plan transparently
    assert torch.equal(_payload(contract(A, E)._blocks), first)


def test_cached_structure_fast_path_follows_mutations(cuda):
    """Repeated contractions of an already-seen structure pair take the host fast path
    (cached slab descriptors / plan, lazily held outputs). In-place metadata mutations
    (put_block_, relabel_, redirect_) must invalidate it; lazily held outputs feed later
    contractions correctly; output bonds are the operands' own Bond objects."""
    import torch
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-1, 5), (0, 9), (1, 6)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])

    def mk(seed):
        A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
        E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
        trandom.normal_(A, seed=seed)
        trandom.normal_(E, seed=seed + 1)
        return A, E

    def dense_of(t):
        return np.concatenate([b.numpy().reshape(-1) for b in t.get_blocks_()])

    A, E = mk(11)
    r1 = contract(A, E)             # full path; remembers the structure pair
    r2 = contract(A, E)             # fast path
    assert np.array_equal(dense_of(r1), dense_of(r2))
    assert r2.bonds[0] is A.bonds[0] and r2.bonds[1] is E.bonds[2]
    # put_block_: a new buffer for block 3 -> the slab descriptor is stale
    blk = A.get_block(3)
    blk.storage().mul_(-2.0)
    A.put_block_(blk, 3)
    ref = contract(A.clone(), E)
    assert np.allclose(dense_of(contract(A, E)), dense_of(ref), rtol=1e-13, atol=1e-13)
    assert not np.allclose(dense_of(ref), dense_of(r1))
    # relabel_: the contracted label set changes -> a different structure
    A2, E2 = mk(21)
    contract(A2, E2)
    contract(A2, E2)
    E2.relabel_(["vr", "q", "x"])  # p no longer shared: only vr is contracted now
    got = contract(A2, E2)
    want = contract(A2.clone(), E2.clone())
    assert got.labels == want.labels == ["vl", "p", "q", "x"]
    assert np.array_equal(dense_of(got), dense_of(want))
    # lazily held outputs as inputs of the next contraction (and of a batch)
    A3, E3 = mk(31)
    out = contract(A3, E3)
    out2 = contract(A3, E3)
    X = UniTensor([V, V.redirect()], labels=["x", "y"])
    trandom.normal_(X, seed=5)
    want = contract(out.clone(), X)
    got = contract(out2, X)
    assert np.allclose(dense_of(got), dense_of(want), rtol=1e-13, atol=1e-13)
    outs = tnb.contract_batched([(out2, X), (out, X)])
    for o in outs:
        assert np.allclose(dense_of(o), dense_of(want), rtol=1e-13, atol=1e-13)
    # redirect_ of a shared bond object flips the directions -> checks fail, no stale reuse
    A4, E4 = mk(41)
    contract(A4, E4)
    contract(A4, E4)
    A4.bonds[1].redirect_()
    with pytest.raises(ValueError):
        contract(A4, E4)
    A4.bonds[1].redirect_()
    torch.cuda.synchronize()


def test_graph_owned_workspaces_are_released(cuda):
    """Each captured grouped GEMM owns its stream-K workspace (allocated at capture, tied to
    the graph); destroying the graphs releases it on the next eager launch, so repeated
    capture / destroy does not grow device memory."""
    import gc
    import torch
    from paper_2401_01921_b200 import graphs
    A, E, _ = _c4()
    contract(A, E)
    torch.cuda.synchronize()

    def cycle():
        g = graphs.capture(lambda: contract(A, E), warmup=1)
        g.replay()
        torch.cuda.synchronize()
        del g
        gc.collect()
        contract(A, E)  # eager launch: frees workspaces of destroyed graphs
        torch.cuda.synchronize()
    cycle()
    torch.cuda.empty_cache()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(12):
        cycle()
    torch.cuda.empty_cache()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < (24 << 20), (free0, free1)  # 12 x 4.9 MB would leak ~59 MB


def test_batched_twin_plan_capture_before_eager(cuda):
    """A float64 batch (>= 4 contractions) first seen INSIDE a stream capture runs on the
    parent plan (the 64 x 128-tile twin is only built eagerly); later eager calls build and
    use the twin. Graph replays and eager calls agree with the pairwise results."""
    import torch
    from paper_2401_01921_b200 import graphs
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-2, 70), (-1, 130), (0, 150), (1, 120), (2, 60)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])

    def mk(seed):
        A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
        E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
        trandom.normal_(A, seed=seed)
        trandom.normal_(E, seed=seed + 1)
        return A, E

    pairs = [mk(1300 + 2 * i) for i in range(6)]
    want = [[b.numpy() for b in tnb.contract_pair(a, e).get_blocks_()] for a, e in pairs]
    holder = {}
    g = graphs.capture(lambda: holder.__setitem__("outs", tnb.contract_batched(pairs)), warmup=0)
    g.replay()
    torch.cuda.synchronize()
    eager = tnb.contract_batched(pairs)  # builds the twin
    eager2 = tnb.contract_batched(pairs)
    g.replay()
    torch.cuda.synchronize()
    for outs in (holder["outs"], eager, eager2):
        for k, o in enumerate(outs):
            for gb, w in zip(o.get_blocks_(), want[k]):
                assert np.linalg.norm(gb.numpy() - w) <= 1e-13 * max(np.linalg.norm(w), 1e-300)
