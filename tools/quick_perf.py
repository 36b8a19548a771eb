"""Quick device timings of the hot-path kernels (development aid, not the bench)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

import tnkit_np as oracle
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import Network, UniTensor, storage, contract


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.min(ts))


def main():
    torch.cuda.set_device(0)
    # permute sweep
    for shape, dt in [((64,) * 4, np.float64), ((64,) * 4, np.complex128), ((16,) * 6, np.float64), ((16,) * 6, np.complex128)]:
        src = storage.uniform(list(shape), dtype=dt, seed=1)
        nbytes = 2 * src.size * src.itemsize
        import itertools
        perms = [p for p in itertools.permutations(range(len(shape)))][1:24] if len(shape) == 4 else \
            [tuple(int(x) for x in np.random.default_rng(i).permutation(6)) for i in range(8)]
        res = []
        for p in perms:
            med, mn = timeit(lambda: src.permute(*p).contiguous())
            res.append(nbytes / med / 1e6)
        print(f"permute {shape} {np.dtype(dt).name}: GB/s median {np.median(res):.0f} min {np.min(res):.0f} max {np.max(res):.0f}")
        print("   per-perm:", " ".join(f"{x:.0f}" for x in res))
    # LAWR
    for chi, dt in [(1024, np.float64), (1024, np.complex128), (128, np.float64), (512, np.complex128)]:
        inp = oracle.lawr_inputs(chi, dtype=dt, seed=3)
        net = Network(oracle.LAWR_NET)
        for nm, arr in inp.items():
            t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
            net.put_tensor(nm, t, t.labels)
        net.set_order(optimal=True)
        macs = {128: 4.3581e7, 512: 2.7106e9, 1024: 2.1580e10}[chi]
        flop = macs * (8 if dt == np.complex128 else 2)
        for mode in (["4M", "3M"] if dt == np.complex128 else ["4M"]):
            tnb.set_complex_mode(mode)
            med, mn = timeit(lambda: net.launch(), reps=5)
            print(f"LAWR chi={chi} {np.dtype(dt).name} {mode}: {med:.3f} ms  {flop / med / 1e9:.0f} GFLOP/s")
        tnb.set_complex_mode("4M")
        # per-step breakdown
        L = net._bindings["L"][0].relabel(["b", "w", "vl"]); A = net._bindings["A"][0].relabel(["vl", "p", "vr"])
        W = net._bindings["W"][0].relabel(["w", "w2", "q", "p"]); R = net._bindings["R"][0].relabel(["b2", "w2", "vr"])
        t1 = tnb.contract_pair(A, L); t2 = tnb.contract_pair(t1, W)
        for name, fn in [("step1 A.L", lambda: tnb.contract_pair(A, L)), ("step2 T1.W", lambda: tnb.contract_pair(t1, W)),
                         ("step3 T2.R", lambda: tnb.contract_pair(t2, R))]:
            med, mn = timeit(fn, reps=5)
            print(f"    {name}: {med:.3f} ms")
    # C4
    from paper_2401_01921_b200 import IN, Bond, Symmetry
    from paper_2401_01921_b200 import random as trandom
    u1 = Symmetry.u1()
    V = Bond(btype=IN, sectors=oracle.c4_sectors(), syms=[u1])
    P = Bond(btype=IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    A = UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
    E = UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
    trandom.normal_(A, seed=1); trandom.normal_(E, seed=2)
    med, mn = timeit(lambda: contract(A, E), reps=20)
    print(f"C4 block-sparse: {med*1000:.1f} us  {2*1.6907e8/med/1e6:.0f} GFLOP/s")
    t0 = time.perf_counter()
    for _ in range(20):
        contract(A, E)
    torch.cuda.synchronize()
    print(f"C4 host wall per call: {(time.perf_counter()-t0)/20*1e6:.0f} us")


if __name__ == "__main__":
    main()
