"""(f)4: the .utn container (pkg/src/tnkit/io.py) read into / written from HBM.

Fixtures in tests/golden/utn were written by the REFERENCE's save_unitensor
(oracle/make_golden_utn.py); loads must reproduce the blocks bit for bit and saves
must reproduce the reference's files byte for byte."""
import json
import os
import struct

import numpy as np
import pytest

from paper_2401_01921_b200 import io as tio

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "utn")
CASES = ["dense", "complex_directed", "u1", "u1xz2", "int64", "u1_odd_sectors", "u1_c128"]


def _header(path):
    raw = open(path, "rb").read()
    assert raw[:5] == tio.MAGIC
    (ver,) = struct.unpack("<I", raw[5:9])
    (hlen,) = struct.unpack("<I", raw[9:13])
    return ver, raw[13:13 + hlen], raw[13 + hlen:]


@pytest.mark.parametrize("case", CASES)
def test_bond_json_round_trip_matches_reference_header(case):
    """CPU: bonds parsed from the reference's header serialise back to the same JSON."""
    ver, hraw, _ = _header(os.path.join(GOLD, case + ".utn"))
    assert ver == tio.VERSION
    h = json.loads(hraw)
    again = [tio._bond_to_json(tio._bond_from_json(d)) for d in h["bonds"]]
    assert json.dumps(again) == json.dumps(h["bonds"])


def test_bad_magic_and_version_rejected(tmp_path):
    """CPU: same checks and messages as io.py:85-90, raised before any device work."""
    bad = tmp_path / "bad.utn"
    bad.write_bytes(b"NOPE\x00" + b"\x00" * 16)
    with pytest.raises(ValueError, match="magic"):
        tio.load_unitensor(bad)
    raw = bytearray(open(os.path.join(GOLD, "dense.utn"), "rb").read())
    raw[5] = 99
    v = tmp_path / "v.utn"
    v.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="version"):
        tio.load_unitensor(v)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_load_reference_file_bitexact(cuda, case):
    z = np.load(os.path.join(GOLD, "blocks.npz"))
    meta = json.loads(str(z["meta"]))[case]
    t = tio.load_unitensor(os.path.join(GOLD, case + ".utn"))
    assert t.name == meta["name"] and t.labels == meta["labels"] and t.rowrank == meta["rowrank"]
    assert str(t.dtype) == meta["dtype"] and t.nblocks == meta["nblocks"]
    if meta["qns"] is not None:
        assert [list(q) for q in t._qns] == meta["qns"]
    for i in range(t.nblocks):
        want = z[f"{case}_b{i}"]
        got = t.get_block_(i).numpy() if t.is_sym else t.get_block_().numpy()
        assert got.dtype == want.dtype and np.array_equal(got, want), (case, i)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_save_reproduces_reference_bytes(cuda, tmp_path, case):
    src = os.path.join(GOLD, case + ".utn")
    t = tio.load_unitensor(src)
    out = tmp_path / "out.utn"
    tio.save_unitensor(t, out)
    assert open(out, "rb").read() == open(src, "rb").read()


@pytest.mark.gpu
def test_lazily_permuted_blocks_are_materialised_on_save(cuda, tmp_path):
    from paper_2401_01921_b200 import UniTensor
    t = tio.load_unitensor(os.path.join(GOLD, "dense.utn"))
    p = t.permute(["c", "a", "b"])  # lazy: save must run tnb_permute and write logical order
    f = tmp_path / "p.utn"
    p.save(f)
    q = UniTensor.load(f)
    assert q.labels == ["c", "a", "b"] and q.shape == p.shape
    assert np.array_equal(q.get_block_().numpy(), p.get_block_().contiguous().numpy())
    # block-sparse: a permuted tensor keeps its block LIST order (unitensor.py:312), so its
    # file lists qn tuples out of enumeration order and the reference's loader rejects it
    # (io.py:100-104); the engine mirrors that check and message
    s = tio.load_unitensor(os.path.join(GOLD, "u1_odd_sectors.utn")).permute(["vr", "vl", "p"])
    g = tmp_path / "s.utn"
    s.save(g)
    with pytest.raises(ValueError, match="Qn indices"):
        UniTensor.load(g)


@pytest.mark.gpu
def test_truncated_payload_rejected(cuda, tmp_path):
    raw = open(os.path.join(GOLD, "u1.utn"), "rb").read()
    cut = tmp_path / "cut.utn"
    cut.write_bytes(raw[:-9])
    with pytest.raises(ValueError, match="truncated"):
        tio.load_unitensor(cut)


@pytest.mark.gpu
def test_large_payload_multi_chunk(cuda, tmp_path, monkeypatch):
    """Payload spanning several pinned chunk buffers, not a multiple of the chunk size:
    the double-buffered read/copy pipeline reassembles it bit for bit."""
    from paper_2401_01921_b200 import UniTensor, storage
    monkeypatch.setattr(tio, "_CHUNK", 3 << 20)
    saved = list(tio._PINNED)
    tio._PINNED.clear()
    arr = np.random.default_rng(5).standard_normal((1000, 1234))  # 9.9 MB
    t = UniTensor(storage.from_numpy(arr), labels=["a", "b"], name="big")
    p = tmp_path / "big.utn"
    tio.save_unitensor(t, p)
    back = tio.load_unitensor(p)
    tio._PINNED[:] = saved
    assert back.name == "big" and np.array_equal(back.get_block_().numpy(), arr)


@pytest.mark.gpu
def test_payload_upload_download_roundtrip(cuda):
    """upload_payload_ / download_payload (packed .utn payload <-> HBM slab): round trip on a
    fresh tensor, on a lazily held contraction result (cached-structure fast path) and on a
    lazily permuted tensor (logical order, general path)."""
    import numpy as np
    import torch
    import bench
    import paper_2401_01921_b200 as tnb
    from paper_2401_01921_b200 import io as tio
    A, E = bench.c4_tensors(tnb, seed=3)
    for t in (A, tnb.contract(A, E), tnb.contract(A, E)):  # the second result: fast path, lazy blocks
        n = tio.payload_nbytes(t)
        want = np.concatenate([b.numpy().reshape(-1) for b in t.get_blocks_()])
        host = torch.empty(n, dtype=torch.uint8).pin_memory()
        t.download_payload(host)
        torch.cuda.synchronize()
        assert np.array_equal(host.numpy().view(np.float64), want)
        t2 = tnb.UniTensor(t.bonds, labels=t.labels, rowrank=t.rowrank)
        t2.upload_payload_(host)
        assert all(np.array_equal(x.numpy(), y.numpy()) for x, y in zip(t2.get_blocks_(), t.get_blocks_()))
    P = A.permute(["vr", "vl", "p"])
    n = tio.payload_nbytes(P)
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    P.download_payload(host)
    torch.cuda.synchronize()
    want = np.concatenate([b.numpy().reshape(-1) for b in P.get_blocks_()])
    assert np.array_equal(host.numpy().view(np.float64), want)


@pytest.mark.gpu
def test_payload_serving_loop_async_ordering(cuda):
    """upload_payload_ runs on the upload stream and download_payload(done=ev) on the download
    stream: a two-set serving loop whose inputs change every step (refills ordered only after
    the contraction that last read the set) returns every step's exact result."""
    import torch
    import bench
    import paper_2401_01921_b200 as tnb
    from paper_2401_01921_b200 import io as tio
    pairs = [bench.c4_tensors(tnb, seed=11 + 2 * j) for j in range(3)]
    payloads, expect = [], []
    for A, E in pairs:
        hA = torch.empty(tio.payload_nbytes(A), dtype=torch.uint8, pin_memory=True)
        hE = torch.empty(tio.payload_nbytes(E), dtype=torch.uint8, pin_memory=True)
        A.download_payload(hA)
        E.download_payload(hE)
        o = tnb.contract(A, E)
        ho = torch.empty(tio.payload_nbytes(o), dtype=torch.uint8, pin_memory=True)
        o.download_payload(ho)
        payloads.append((hA, hE))
        expect.append(ho)
    torch.cuda.synchronize()
    sets = [bench.c4_tensors(tnb, seed=99 + k) for k in range(2)]
    read = [None, None]
    outs = [torch.empty_like(expect[0]) for _ in range(9)]
    for i in range(9):
        k = i % 2
        hA, hE = payloads[i % 3]
        sets[k][0].upload_payload_(hA, after=read[k])
        sets[k][1].upload_payload_(hE, after=read[k])
        o = tnb.contract(*sets[k])
        read[k] = torch.cuda.Event()
        read[k].record()
        o.download_payload(outs[i], done=torch.cuda.Event())
    torch.cuda.synchronize()
    for i in range(9):
        assert torch.equal(outs[i], expect[i % 3]), i


@pytest.mark.gpu
def test_payload_step_captured_in_a_graph(cuda):
    """The serving step (two payload uploads, contract, payload download) captured once with
    graphs.capture replays with whatever the pinned host buffers hold at replay time."""
    import torch
    import bench
    import paper_2401_01921_b200 as tnb
    from paper_2401_01921_b200 import io as tio
    src = [bench.c4_tensors(tnb, seed=41 + 2 * j) for j in range(2)]
    A, E = bench.c4_tensors(tnb, seed=97)
    hA = torch.empty(tio.payload_nbytes(A), dtype=torch.uint8, pin_memory=True)
    hE = torch.empty(tio.payload_nbytes(E), dtype=torch.uint8, pin_memory=True)
    out0 = tnb.contract(A, E)
    hO = torch.empty(tio.payload_nbytes(out0), dtype=torch.uint8, pin_memory=True)

    def step():
        A.upload_payload_(hA)
        E.upload_payload_(hE)
        return tnb.contract(A, E).download_payload(hO)
    g = tnb.graphs.capture(step)
    for sa, se in src + src[::-1]:
        sa.download_payload(hA)
        se.download_payload(hE)
        torch.cuda.synchronize()
        want = torch.empty_like(hO)
        tnb.contract(sa, se).download_payload(want)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(hO, want)
