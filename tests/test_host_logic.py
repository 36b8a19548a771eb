"""Host-side (CPU) logic of the engine: charge algebra, native block enumeration,
native order DP, order-string grammar, Network parsing and validation.
All bit-exact against the reference's golden vectors or oracle restatement."""
import itertools

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import tnkit_np as oracle
from tnb_testutil import bonds_from_meta, load, oracle_bonds

from paper_2401_01921_b200 import (IN, OUT, REGULAR, Bond, Network, Symmetry, brute_force_order,
                                   contraction_cost, find_optimal_order, parse_order, render_order)
from paper_2401_01921_b200 import contraction as C
from paper_2401_01921_b200.labeled import zero_flux_combos


# -- charges / bonds (symmetry.py, bond.py) ----------------------------------------
def test_symmetry_rules():
    u1, z3 = Symmetry.u1(), Symmetry.zn(3)
    assert z3.combine(2, 2) == 1 and z3.reverse(1) == 2 and z3.normalize(-1) == 2
    assert u1.combine(-3, 5) == 2 and u1.reverse(4) == -4
    assert str(z3) == "Z3" and str(u1) == "U1" and z3 == Symmetry.zn(3) and z3 != u1
    with pytest.raises(ValueError):
        Symmetry.zn(1)


def test_golden_bond_combination():
    u1 = Symmetry.u1()
    b12 = Bond(btype=IN, sectors=[(0, 1), (1, 1)], syms=[u1]).combine(
        Bond(btype=IN, sectors=[(2, 1), (3, 1)], syms=[u1]))
    assert b12.qnums() == ((2,), (3,), (4,)) and b12.degeneracies() == (1, 2, 1)


def test_bond_validation_and_redirect():
    u1 = Symmetry.u1()
    with pytest.raises(ValueError):
        Bond(btype=REGULAR, sectors=[(0, 1)], syms=[u1])
    with pytest.raises(ValueError):
        Bond(btype=IN, sectors=[(0, 1), (0, 2)], syms=[u1])
    b = Bond(btype=IN, sectors=[(1, 2), (-1, 3)], syms=[u1])
    assert b.dim == 5 and b.sector_offsets() == (0, 2) and b.locate(3) == (1, 1)
    r = b.redirect()
    assert r.btype == OUT and r.sectors == b.sectors and r != b and r.redirect() == b


# -- a3: native zero-flux enumeration ------------------------------------------------
def test_native_zero_flux_matches_golden():
    _, meta = load("blocks.npz")
    for c in meta["enum"]:
        got = zero_flux_combos(bonds_from_meta(c["bonds"]))
        assert [list(q) for q in got] == c["qns"]
    for c in meta["cases"]:
        if "out_bonds" in c:
            assert [list(q) for q in zero_flux_combos(bonds_from_meta(c["out_bonds"]))] == c["out_qns"]


def test_native_zero_flux_c4():
    _, meta = load("c4.npz")
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=[(q, d) for q, d in meta["sectors"]], syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    assert [list(q) for q in zero_flux_combos([V, P, V.redirect()])] == meta["a_qns"]
    assert [list(q) for q in zero_flux_combos([V, P.redirect(), V.redirect()])] == meta["e_qns"]
    assert [list(q) for q in zero_flux_combos([V, V.redirect()])] == meta["out_qns"]


@st.composite
def _bond_lists(draw):
    syms = draw(st.sampled_from([[Symmetry.u1()], [Symmetry.zn(2)], [Symmetry.zn(3)],
                                 [Symmetry.u1(), Symmetry.zn(2)]]))
    rank = draw(st.integers(1, 4))
    bonds = []
    for _ in range(rank):
        charges = draw(st.lists(st.tuples(*[st.integers(-3, 3) for _ in syms]), min_size=1, max_size=4,
                                unique_by=lambda q: tuple(s.normalize(x) for s, x in zip(syms, q))))
        sectors = [(q, draw(st.integers(1, 3))) for q in charges]
        bonds.append(Bond(btype=draw(st.sampled_from([IN, OUT])), sectors=sectors, syms=syms))
    return bonds


@given(_bond_lists())
@settings(max_examples=150, deadline=None)
def test_native_zero_flux_equals_oracle(bonds):
    ob = [(1 if b.btype == IN else -1, list(b.qnums()), [s.modulus for s in b.syms]) for b in bonds]
    assert zero_flux_combos(bonds) == oracle.zero_flux_combos(ob)


# -- a14/a15: order DP and grammar ---------------------------------------------------
def test_native_order_dp_matches_reference_golden():
    _, meta = load("order.npz")
    for c in meta["cases"]:
        t = find_optimal_order(c["sets"], c["dims"])
        assert render_order(t) == c["order"], c
        assert str(contraction_cost(t, c["sets"], c["dims"])) == c["cost"]


def test_python_dp_equals_native_dp():
    _, meta = load("order.npz")
    for c in meta["cases"]:
        names = list(c["sets"])
        t = C._find_optimal_order_py(names, c["sets"], c["dims"])
        assert render_order(t) == c["order"]


def test_dp_equals_brute_force_random():
    rng = np.random.default_rng(5)
    for _ in range(30):
        nt = int(rng.integers(2, 7))
        names = [f"T{i}" for i in range(nt)]
        sets = {n: [] for n in names}
        dims, lbl = {}, 0
        for i in range(nt):
            for j in range(i + 1, nt):
                if rng.random() < 0.55:
                    sets[names[i]].append(f"e{lbl}")
                    sets[names[j]].append(f"e{lbl}")
                    dims[f"e{lbl}"] = int(rng.integers(2, 7))
                    lbl += 1
        for i in range(nt):
            if rng.random() < 0.5 or not sets[names[i]]:
                sets[names[i]].append(f"f{lbl}")
                dims[f"f{lbl}"] = int(rng.integers(2, 7))
                lbl += 1
        opt = find_optimal_order(sets, dims)
        assert contraction_cost(opt, sets, dims) == contraction_cost(brute_force_order(sets, dims), sets, dims)


def test_huge_costs_fall_back_to_exact_python_dp():
    sets = {"A": ["i", "j"], "B": ["j", "k"], "C": ["k", "l"]}
    dims = {"i": 2 ** 62, "j": 2 ** 62, "k": 2 ** 62, "l": 2 ** 62}
    t = find_optimal_order(sets, dims)
    assert render_order(t) == render_order(oracle.find_optimal_order(sets, dims))


def test_order_grammar_round_trip():
    for text in ["((M1,M2),M3)", "(M2,(M1,M3))", "(((a,b),(c,d)),e)", "T", "(a*,b')"]:
        assert render_order(parse_order(text)) == text
    assert render_order(parse_order(" ( A , ( B,C ) ) ")) == "(A,(B,C))"
    for bad in ["((M1,M2)", "(M1;M2)", "(M1,M2) x", "", "(,A)"]:
        with pytest.raises(ValueError):
            parse_order(bad)


# -- a16: Network parsing / policy (no tensors needed) --------------------------------
THREE = ["M1: i, j", "M2: j, k", "M3: k, l", "TOUT: i, l", "ORDER: ((M1,M2),M3)"]


def test_network_parse_print_and_tout_split():
    net = Network(THREE)
    text = str(net)
    assert text.splitlines()[0] == "==== Network ====" and "TOUT : i ; l" in text
    assert "ORDER : ((M1,M2),M3)" in text and "[ ] M1 : i j" in text
    n = Network(["A: i, j, k", "TOUT: i, j, k"])
    assert n._tout_row == ["i"] and n._tout_col == ["j", "k"]
    n = Network(["A: i, j", "B: j", "TOUT: i"])
    assert n._tout_row == [] and n._tout_col == ["i"]
    n = Network(["A: i, j, k", "TOUT: i, j ; k"])
    assert n._tout_row == ["i", "j"] and n._tout_col == ["k"]
    n = Network(["# heading", "", "M1: i, j  # trailing", "\r", "M2: j, k\r", "TOUT: i, k\r"])
    assert [s for s, _ in n._slots] == ["M1", "M2"]


@pytest.mark.parametrize("lines", [
    ["M1: i, j", "M1: j, k", "TOUT: i, k"], ["M1: i, j", "M2: j, k", "TOUT: i"],
    ["M1: i, j", "M2: j, k", "M3: j, l", "TOUT: i, k, l"], ["M1: i, j", "TOUT: i, j", "ORDER: (M1,M2)"],
    ["M1 i j", "TOUT:"], ["M1: i, j", "TOUT: i, j", "ORDER: ((M1)"], ["TOUT: "], ["A: i, j", "B: j, i"],
    ["A: i, j", "B: j, i", "TOUT: i"]])
def test_network_parse_errors(lines):
    with pytest.raises(ValueError):
        Network(lines)


def test_network_order_policy_and_round_trip(tmp_path):
    net = Network(THREE)
    net.set_order(optimal=False, contract_order="(M2,(M1,M3))")
    assert net.get_order() == "(M2,(M1,M3))"
    with pytest.raises(ValueError):
        net.set_order(contract_order="(M1,M2)")
    with pytest.raises(ValueError):
        net.set_order(optimal=True, contract_order="((M1,M2),M3)")
    assert Network(["M1: i, j", "M2: j, k", "TOUT: i, k"]).get_order() == "(M1,M2)"
    assert Network(["A: i", "B: i, j", "C: j, k", "D: k", "TOUT:"]).get_order() == "(((A,B),C),D)"
    for lines in (THREE, ["A: x, y, z", "TOUT: z, x ; y"], ["A: i, j", "B: j, i", "TOUT:"]):
        n = Network(lines)
        p = tmp_path / "x.net"
        n.save_file(p)
        assert Network(str(p)) == n
    # Cytnx spellings
    n = Network()
    n.FromString(THREE)
    assert n.getOrder() == "((M1,M2),M3)"
