"""Parity at the BENCHMARKED sizes: the exact launches
bench.py times, through Network.launch -> libtnb, against the oracle's numpy restatement
of Network.launch (network.py:213-244, contract.py:127-132) on the same seeded inputs.

Tolerance: relative Frobenius <= 1e-12 (BASELINE.json north_star). Oracle cost on the
box's cores: ~0.15 s (chi=1024 f64), ~1 s (chi=1024 c128), ~0.2 s per chi=512 c128
instance, ~10 s for one PEPS site at chi=256, D=8."""
import numpy as np
import pytest

import tnkit_np as oracle
from tnb_testutil import rel_fro

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import Network, UniTensor, storage, workloads

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _net(lines, arrays):
    net = Network(lines)
    for nm, arr in arrays.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"x{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
    net.set_order(optimal=True)
    return net


@pytest.mark.parametrize("dtype,mode", [(np.float64, "4M"), (np.complex128, "4M"), (np.complex128, "3M")])
def test_lawr_chi1024(cuda, dtype, mode):
    """C3 headline (f64) and the complex128 variant in both complex formulations."""
    inp = workloads.lawr_inputs(1024, dtype=dtype, seed=1234)
    ref_inp = oracle.lawr_inputs(1024, dtype=dtype, seed=1234)
    for k in inp:  # the engine's host generator reproduces the reference bits
        assert np.array_equal(inp[k], ref_inp[k])
    want, tree = oracle.launch(oracle.lawr_slots(), "b, q, b2", ref_inp)
    old = tnb.get_complex_mode()
    try:
        tnb.set_complex_mode(mode)
        net = _net(workloads.LAWR_NET, inp)
        out = net.launch()
        assert net.get_order() == oracle.render_order(tree) == "(((A,L),W),R)"
        got = out.numpy()
        assert got.shape == want.shape and got.dtype == want.dtype
        err = rel_fro(got, want)
        assert err <= TOL, err
        # a second launch (recorded-program replay path) is bit-identical
        assert np.array_equal(net.launch().numpy(), got)
    finally:
        tnb.set_complex_mode(old)


@pytest.mark.parametrize("i", [0, 37])
def test_lawr_batch_instance_chi512_c128(cuda, i):
    """C3b: instances of the 64 x chi=512 complex128 batch (seeds 5000 + 4i)."""
    seed = workloads.lawr_batch_seed(i)
    inp = workloads.lawr_inputs(512, dtype=np.complex128, seed=seed)
    want, _ = oracle.launch(oracle.lawr_slots(), "b, q, b2", oracle.lawr_inputs(512, dtype=np.complex128, seed=seed))
    out = _net(workloads.LAWR_NET, inp).launch().numpy()
    err = rel_fro(out, want)
    assert err <= TOL, err


def test_peps_site_chi256_D8(cuda):
    """C5 reading A, site 0 at the benchmarked size: the full double-layer scalar, optimal
    order (((((C0,T0),C1),(C2,T1)),a),((C3,T2),T3)),a*), against the oracle."""
    inp = workloads.peps_inputs(256, 8, 2, site=0)
    ref_inp = oracle.peps_inputs(256, 8, 2, site=0)
    for k in inp:
        assert np.array_equal(inp[k], ref_inp[k])
    want, tree = oracle.launch(oracle.net_slots(oracle.PEPS_NET), "", ref_inp)
    net = _net(workloads.PEPS_NET, inp)
    got = net.launch().item()
    assert net.get_order() == oracle.render_order(tree) == "((((((C0,T0),C1),(C2,T1)),a),((C3,T2),T3)),a*)"
    want = np.asarray(want).item()  # rank-0 result
    err = abs(got - want) / abs(want)
    assert err <= TOL, (got, want, err)


def test_peps_open_legs_chi64(cuda):
    """C5 with the optional open physical legs (s ; s'), 2x2 output, at chi=64 D=6: every
    element against the oracle (exercises the rank-5 a / a* steps with free legs)."""
    lines = list(oracle.PEPS_NET[:-3]) + ["a: u, l, dn, r, s", "a*: u', l', dn', r', s'", "TOUT: s ; s'"]
    inp = oracle.peps_inputs(64, 6, 2, site=3)
    want, tree = oracle.launch(oracle.net_slots(lines), "s ; s'", inp)
    net = _net(lines, inp)
    out = net.launch()
    assert net.get_order() == oracle.render_order(tree)
    err = rel_fro(out.numpy(), want)
    assert err <= TOL, err
