"""compiled (CUDA-graph) Network plans and device Lanczos."""
import numpy as np
import pytest
import torch

import tnkit_np as oracle
from tnb_testutil import rel_fro

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import Network, UniTensor, storage
from paper_2401_01921_b200.eig import ConvergenceError, LinOp, NetworkMatvec, lanczos

pytestmark = pytest.mark.gpu


def _lawr(chi, seed, dtype=np.float64):
    inp = oracle.lawr_inputs(chi, dtype=dtype, seed=seed)
    net = Network(oracle.LAWR_NET)
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
    net.set_order(optimal=True)
    return net, inp


def test_compiled_network_matches_eager_and_rebinds(cuda):
    net, inp = _lawr(48, 7)
    eager = net.launch().numpy()
    comp = net.compile()
    assert comp.order == "(((A,L),W),R)"
    assert np.array_equal(comp.launch().numpy(), eager)
    # rebinding A (the Lanczos vector) copies into the captured buffer
    a2 = oracle.normal([48, 2, 48], seed=99)
    comp.put_tensor("A", UniTensor(storage.from_numpy(a2), labels=["x", "y", "z"]))
    inp2 = dict(inp, A=a2)
    want, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", inp2)
    assert rel_fro(comp.launch().numpy(), want) <= 1e-12
    # the user's own bound tensors are untouched by compiled replays
    assert np.array_equal(net.launch().numpy(), eager)
    with pytest.raises(ValueError):
        comp.put_tensor("A", UniTensor(storage.from_numpy(oracle.normal([48, 2, 47], seed=1)), labels=["x", "y", "z"]))


def test_device_lanczos_matches_dense_eigvalsh(cuda):
    rng = np.random.default_rng(42)
    for dim, k in [(20, 1), (80, 2), (200, 3)]:
        a = rng.standard_normal((dim, dim))
        a = (a + a.T) / 2
        ad = torch.from_numpy(a).cuda()
        vals, vecs = lanczos(LinOp(dim, matvec=lambda v: ad @ v), k=k, tol=1e-12)
        assert np.allclose(vals, np.linalg.eigvalsh(a)[:k], atol=1e-10)
        for i in range(k):
            r = torch.linalg.vector_norm(ad @ vecs[:, i] - vals[i] * vecs[:, i])
            assert float(r) <= 1e-8


def test_device_lanczos_on_compiled_network(cuda):
    """H(psi) = L.psi.W.R with Hermitian environments (L = R) and a symmetric W is a
    symmetric operator; Lanczos on the graph-replayed network matches the dense
    operator's spectrum."""
    chi, D, d = 6, 3, 2
    rng = np.random.default_rng(5)
    L = rng.standard_normal((chi, D, chi))
    L = (L + L.transpose(2, 1, 0)) / 2           # L[b,w,vl] = L[vl,w,b]
    W = rng.standard_normal((D, D, d, d))
    W = (W + W.transpose(1, 0, 3, 2)) / 2         # W[w,w2,q,p] = W[w2,w,p,q]
    W = (W + W.transpose(0, 1, 3, 2)) / 2
    Wsym = (W + W.transpose(1, 0, 2, 3)) / 2
    A = rng.standard_normal((chi, d, chi))
    inp = {"L": L, "A": A, "W": Wsym, "R": L.copy()}
    net = Network(oracle.LAWR_NET)
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
    net.set_order(optimal=True)
    comp = net.compile()
    op = NetworkMatvec(comp, "A")   # out [b, q, b2] has A's [vl, p, vr] layout
    n = op.dim
    dense_h = np.zeros((n, n))
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        dense_h[:, i] = op(torch.from_numpy(e).cuda()).cpu().numpy()
    assert np.allclose(dense_h, dense_h.T, atol=1e-12)
    vals, _ = lanczos(op, k=2, tol=1e-12, seed=3)
    assert np.allclose(vals, np.linalg.eigvalsh(dense_h)[:2], atol=1e-9)


def test_lanczos_convergence_error_carries_estimate(cuda):
    a = np.diag(np.arange(1.0, 51.0))
    ad = torch.from_numpy(a).cuda()
    with pytest.raises(ConvergenceError) as e:
        lanczos(LinOp(50, matvec=lambda v: ad @ v), k=1, tol=1e-15, max_iter=3, seed=1)
    assert e.value.eigenvalues is not None


def test_device_lanczos_matches_reference_golden(cuda):
    """Engine Lanczos (graph-replayed Network matvec) vs the reference's own Ritz values
    (tests/golden/lanczos.npz, written by oracle/make_golden_lanczos.py)."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lanczos.npz"))
    inp = {k[3:]: z[k] for k in z.files if k.startswith("in_")}
    net = Network(oracle.LAWR_NET)
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
    net.set_order(optimal=True)
    op = NetworkMatvec(net.compile(), "A")
    for seed in (3, 11):
        vals, vecs = lanczos(op, k=2, tol=1e-12, seed=seed)
        assert np.allclose(vals, z[f"theta_seed{seed}"], rtol=0, atol=1e-10)
        # eigenvector residual through the engine matvec
        for j in range(2):
            v = vecs[:, j].contiguous()
            r = op(v) - vals[j] * v
            assert float(torch.linalg.vector_norm(r)) <= 1e-8 * max(1.0, abs(vals[j]))


def test_device_lanczos_complex_hermitian(cuda):
    """complex128 Hermitian operators (the reference's LinOp dtype argument): lowest Ritz
    values equal eigvalsh, eigenvectors satisfy the residual bound."""
    rng = np.random.default_rng(7)
    for dim, k in [(30, 1), (120, 2)]:
        a = rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))
        a = (a + a.conj().T) / 2
        ad = torch.from_numpy(a).cuda()
        vals, vecs = lanczos(LinOp(dim, matvec=lambda v: ad @ v, dtype=np.complex128), k=k, tol=1e-12, seed=3)
        assert np.allclose(vals, np.linalg.eigvalsh(a)[:k], atol=1e-10)
        for i in range(k):
            r = torch.linalg.vector_norm(ad @ vecs[:, i] - vals[i] * vecs[:, i])
            assert float(r) <= 1e-8


def test_device_lanczos_breakdown_restart_and_no_torch_vector_ops(cuda, monkeypatch):
    """A start vector inside a 2-dimensional invariant subspace breaks the recurrence down
    after two steps; the device Lanczos restarts with a random orthogonal vector (as the
    reference does) and still finds the 3 lowest eigenvalues. The vector work runs in
    libtnb (tnb_lanczos_step): torch's vdot / vector_norm are never called."""
    import torch
    d = np.array([-3.0, -1.0, 0.5, 1.5, 2.0, 4.0, 5.0, 7.0])
    ad = torch.diag(torch.from_numpy(d)).cuda()
    v0 = np.zeros(8)
    v0[[1, 4]] = 1.0

    def boom(*a, **k):
        raise AssertionError("torch vector op called inside lanczos")
    monkeypatch.setattr(torch, "vdot", boom)
    monkeypatch.setattr(torch.linalg, "vector_norm", boom)
    vals, vecs = lanczos(LinOp(8, matvec=lambda v: ad @ v), k=3, v0=v0, tol=1e-12, seed=2)
    assert np.allclose(vals, np.sort(d)[:3], atol=1e-12)
    for i in range(3):
        v = vecs[:, i]
        r = (ad @ v - vals[i] * v).norm().item() if False else float(np.linalg.norm((ad @ v - vals[i] * v).cpu().numpy()))
        assert r <= 1e-10
