"""Benchmark workload recipes (BASELINE.json configs).

Synthetic, seeded inputs with the reference generators' exact bits (PCG64 via
``dense.host_normal``): there is no dataset in this domain. Used by bench.py's
GPU leg and by examples; the CPU oracle keeps its own independent copy.
"""
import numpy as np

from . import dense

# C1/C3: DMRG one-site effective Hamiltonian L.A.W.R (labels from tnkit dmrg.py:93, :192)
LAWR_NET = ["L: b, w, vl", "A: vl, p, vr", "W: w, w2, q, p", "R: b2, w2, vr", "TOUT: b, q, b2"]

# C5 reading A: PEPS double layer with a CTM environment
PEPS_NET = ["C0: c0t0, c0t3", "C1: c1t1, c1t0", "C2: c2t2, c2t1", "C3: c3t3, c3t2",
            "T0: c1t0, u, u', c0t0", "T1: c2t1, r, r', c1t1", "T2: c3t2, dn, dn', c2t2", "T3: c0t3, l, l', c3t3",
            "a: u, l, dn, r, s", "a*: u', l', dn', r', s", "TOUT:"]


def lawr_inputs(chi, d=2, D=5, dtype=np.float64, seed=1234):
    """L[chi,D,chi], A[chi,d,chi], W[D,D,d,d], R[chi,D,chi] ~ N(0,1), seeds seed+0..3."""
    return {"L": dense.host_normal([chi, D, chi], dtype=dtype, seed=seed),
            "A": dense.host_normal([chi, d, chi], dtype=dtype, seed=seed + 1),
            "W": dense.host_normal([D, D, d, d], dtype=dtype, seed=seed + 2),
            "R": dense.host_normal([chi, D, chi], dtype=dtype, seed=seed + 3)}


def lawr_label_sets():
    return {"L": ["b", "w", "vl"], "A": ["vl", "p", "vr"], "W": ["w", "w2", "q", "p"], "R": ["b2", "w2", "vr"]}


def lawr_dims(chi, d=2, D=5):
    return {"b": chi, "vl": chi, "vr": chi, "b2": chi, "w": D, "w2": D, "p": d, "q": d}


def peps_shapes(chi=256, D=8, d=2):
    return {"C0": [chi, chi], "C1": [chi, chi], "C2": [chi, chi], "C3": [chi, chi],
            "T0": [chi, D, D, chi], "T1": [chi, D, D, chi], "T2": [chi, D, D, chi], "T3": [chi, D, D, chi],
            "a": [D, D, D, D, d], "a*": [D, D, D, D, d]}


def c4_sectors(total=2048, qmax=10, sigma2=18.0):
    """21 U(1) sectors -qmax..qmax, sizes ~ exp(-q^2/(2 sigma^2)), largest-remainder to `total`."""
    qs = list(range(-qmax, qmax + 1))
    w = np.exp(-np.array(qs, dtype=np.float64) ** 2 / sigma2)
    x = total * w / w.sum()
    n = np.maximum(1, np.floor(x)).astype(np.int64)
    rem = total - int(n.sum())
    for k in np.argsort(-(x - np.floor(x)), kind="stable")[:rem]:
        n[k] += 1
    return [(q, int(c)) for q, c in zip(qs, n)]


def peps_inputs(chi=256, D=8, d=2, site=0):
    """C5 site `site`: every slot N(0,1) from its own seed 9000 + 16*site + slot index, so the
    32 sites of the batch are distinct, independently reproducible networks."""
    return {nm: dense.host_normal(shp, seed=9000 + 16 * site + k)
            for k, (nm, shp) in enumerate(peps_shapes(chi, D, d).items())}


def lawr_batch_seed(i):
    """C3b instance i: L, A, W, R = normal(seed .. seed+3) (seeds S+4i)."""
    return 5000 + 4 * i
