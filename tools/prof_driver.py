"""Small driver for ncu captures: one workload, a few iterations (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

import tnkit_np as oracle
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import Network, UniTensor, storage


def lawr(chi, dt, iters):
    inp = oracle.lawr_inputs(chi, dtype=dt, seed=3)
    net = Network(oracle.LAWR_NET)
    for nm, arr in inp.items():
        t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
    net.set_order(optimal=True)
    for _ in range(iters):
        net.launch()
    torch.cuda.synchronize()


def permute(shape, dt, perms, iters):
    src = storage.uniform(list(shape), dtype=dt, seed=1)
    for _ in range(iters):
        for p in perms:
            src.permute(*p).contiguous()
    torch.cuda.synchronize()


def c4(iters):
    sys.path.insert(0, ROOT)
    import bench
    A, E = bench.c4_tensors(tnb)
    for _ in range(iters):
        tnb.contract(A, E)
    torch.cuda.synchronize()


def peps_step(iters):
    """The C5 a* step: A(256,8,256,8,8,8,2) x B(8,8,256,256,8,8) -> (8,8,2,8,8) (M=128, N=64)."""
    a = storage.normal([256, 8, 256, 8, 8, 8, 2], seed=1)
    b = storage.normal([8, 8, 256, 256, 8, 8], seed=2)
    A = UniTensor(a, labels=["c1", "l", "c2", "dn", "u", "r", "s"])
    B = UniTensor(b, labels=["u2", "r2", "c1", "c2", "l", "dn"])
    for _ in range(iters):
        tnb.contract(A, B)
    torch.cuda.synchronize()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    what = sys.argv[1]
    if what == "lawr":
        lawr(int(sys.argv[2]), np.complex128 if sys.argv[3] == "c128" else np.float64, int(sys.argv[4]))
    elif what == "permute":
        perms = [tuple(int(c) for c in p) for p in sys.argv[4].split(",")]
        permute(tuple(int(x) for x in sys.argv[2].split("x")), np.complex128 if sys.argv[3] == "c128" else np.float64,
                perms, int(sys.argv[5]))
    elif what == "peps_step":
        peps_step(int(sys.argv[2]))
    elif what == "c4":
        c4(int(sys.argv[2]))
    print("done")


def c4_batch(n, iters):
    sys.path.insert(0, ROOT)
    import bench
    pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(n)]
    for _ in range(iters):
        tnb.contract_batched(pairs)
    torch.cuda.synchronize()


if __name__ == "__main__" and sys.argv[1] == "c4_batch":
    c4_batch(int(sys.argv[2]), int(sys.argv[3]))


def lanczos_probe(chi, iters):
    sys.path.insert(0, ROOT)
    import bench
    from paper_2401_01921_b200 import eig
    inp = oracle.hermitian_lawr_inputs(chi, seed=7)
    net, _ = bench.make_network(tnb, oracle.LAWR_NET, inp)
    op = eig.NetworkMatvec(net.compile(), "A")
    try:
        eig.lanczos(op, k=1, tol=1e-14, max_iter=iters, seed=3)
    except eig.ConvergenceError:
        pass
    torch.cuda.synchronize()


if __name__ == "__main__" and sys.argv[1] == "lanczos":
    lanczos_probe(int(sys.argv[2]), int(sys.argv[3]))


def peps_site(iters):
    sys.path.insert(0, ROOT)
    import bench
    from paper_2401_01921_b200 import workloads as WL
    net, _ = bench.make_network(tnb, WL.PEPS_NET, WL.peps_inputs(256, 8, 2, site=0))
    for _ in range(iters):
        net.launch()
    torch.cuda.synchronize()


if __name__ == "__main__" and sys.argv[1] == "peps_site":
    peps_site(int(sys.argv[2]))
