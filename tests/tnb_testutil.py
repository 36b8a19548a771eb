"""Helpers for the parity tests: golden fixture loading and error metrics."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name))
    meta = json.loads(str(z["meta"]))
    return z, meta


def rel_fro(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    den = np.linalg.norm(want.reshape(-1))
    num = np.linalg.norm((got - want).reshape(-1))
    return num / den if den > 0 else num


def bonds_from_meta(meta_bonds):
    from paper_2401_01921_b200 import IN, OUT, Bond
    from paper_2401_01921_b200.charges import symmetry_from_str
    out = []
    for b in meta_bonds:
        syms = [symmetry_from_str(s) for s in b["syms"]]
        out.append(Bond(btype=IN if b["btype"] == 1 else OUT, sectors=[(tuple(q), d) for q, d in b["sectors"]],
                        syms=syms))
    return out


def oracle_bonds(meta_bonds):
    """(btype, [qnum tuples], sym_n list) for oracle.zero_flux_combos."""
    out = []
    for b in meta_bonds:
        syms = [0 if s == "U1" else int(s[1:]) for s in b["syms"]]
        out.append((b["btype"], [tuple(q) for q, _ in b["sectors"]], syms))
    return out
