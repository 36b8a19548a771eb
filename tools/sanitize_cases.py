"""Small hot-path cases for compute-sanitizer runs (memcheck / racecheck / synccheck):
C1-style L.A.W.R (chi 24, f64 and c128), one U(1) block-sparse contraction (single and
batched, eager and graph-captured), permutes (t2d, wide t2d, rows, tiled), the batched
copy and the Jacobi SVD. Each result is checked against the oracle so a run under the
sanitizer is also a parity run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import tnkit_np as oracle
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import IN, Bond, Network, Symmetry, UniTensor, storage
from paper_2401_01921_b200 import random as trandom


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


torch.cuda.set_device(0)
which = sys.argv[1:] or ["lawr", "bs", "perm", "svd"]
if "lawr" in which:
    for dt in (np.float64, np.complex128):
        inp = oracle.lawr_inputs(24, dtype=dt, seed=3)
        want, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp)
        net = Network(oracle.LAWR_NET)
        for nm, arr in inp.items():
            t = UniTensor(storage.from_numpy(arr), labels=[f"x{i}" for i in range(arr.ndim)])
            net.put_tensor(nm, t, t.labels)
        net.set_order(optimal=True)
        assert rel(net.launch().numpy(), want) < 1e-12
        cn = net.compile()
        assert rel(cn.launch().numpy(), want) < 1e-12
    print("lawr ok")
if "bs" in which:
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-2, 3), (-1, 17), (0, 70), (1, 33), (2, 5)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    pairs = []
    for s in range(3):
        A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
        E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
        trandom.normal_(A, seed=10 + 2 * s)
        trandom.normal_(E, seed=11 + 2 * s)
        pairs.append((A, E))
    A, E = pairs[0]
    out = tnb.contract(A, E)
    ref, _ = oracle.contract_blocks(A._qns, [b.numpy() for b in A.get_blocks_()], A.labels, E._qns,
                                    [b.numpy() for b in E.get_blocks_()], E.labels, out._qns)
    for o, r in zip(out.get_blocks_(), ref):
        assert rel(o.numpy(), r) < 1e-12
    outs = tnb.contract_batched(pairs)
    g = tnb.graphs.capture(lambda: tnb.contract(A, E), warmup=1)
    g.replay()
    torch.cuda.synchronize()
    for o, r in zip(g.output.get_blocks_(), ref):
        assert rel(o.numpy(), r) < 1e-12
    for (a, e), o in zip(pairs, outs):
        w = tnb.contract(a, e)
        for x, y in zip(o.get_blocks_(), w.get_blocks_()):
            assert rel(x.numpy(), y.numpy()) < 1e-13
    print("bs ok")
if "perm" in which:
    for shape, p, dt in [((70, 66, 68), (2, 1, 0), np.float64), ((128, 3, 130), (2, 1, 0), np.float64),
                         ((40, 36, 5), (1, 0, 2), np.complex128), ((3, 5, 7, 2), (3, 1, 0, 2), np.float64),
                         ((66, 70), (1, 0), np.complex128)]:
        src = oracle.uniform(list(shape), dtype=dt, seed=1)
        got = storage.DenseTensor(src).permute(*p).contiguous().numpy()
        assert np.array_equal(got, oracle.permute_contiguous(src, p))
    print("perm ok")
if "svd" in which:
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(-1, 6), (0, 9), (1, 5)], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    psi = UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], rowrank=2)
    trandom.normal_(psi, seed=4)
    u, s, vh = tnb.linalg.svd(psi)
    print("svd ok")
torch.cuda.synchronize()
print("all ok")
