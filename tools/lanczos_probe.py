"""Dev aid: where a device-Lanczos iteration spends its time (chi=1024 L.A.W.R)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import bench, paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import eig
import tnkit_np as ORACLE
inp = ORACLE.hermitian_lawr_inputs(1024, seed=7)
net, _ = bench.lawr_network(tnb, inp)
op = eig.NetworkMatvec(net.compile(), "A")
v = torch.randn(op.dim, dtype=torch.float64, device="cuda")
Qt = torch.randn(31, op.dim, dtype=torch.float64, device="cuda")
w = op(v)
def t(f, name):
    for _ in range(3): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20): f()
    torch.cuda.synchronize(); print(name, "ms %.3f" % ((time.perf_counter() - t0) / 20 * 1e3))
t(lambda: op(v), "matvec")
t(lambda: w - Qt.T @ (Qt @ w), "reorth(31)")
t(lambda: float(torch.vdot(v, w)), "vdot+sync")
t(lambda: float(torch.dot(v, w)), "dot+sync")
t(lambda: float((v * w).sum()), "mul-sum+sync")
t(lambda: float(torch.linalg.vector_norm(w)), "norm+sync")
import scipy.linalg
al, be = np.random.rand(30), np.random.rand(29)
t0 = time.perf_counter()
for _ in range(20): scipy.linalg.eigh_tridiagonal(al, be, select="i", select_range=(0, 0))
print("eigh_tridiagonal(30) ms %.3f" % ((time.perf_counter() - t0) / 20 * 1e3))
import cProfile, pstats
def run():
    try:
        eig.lanczos(op, k=1, tol=1e-14, max_iter=30, seed=3)
    except eig.ConvergenceError:
        pass
run(); torch.cuda.synchronize()
t0 = time.perf_counter(); run(); torch.cuda.synchronize(); print("lanczos 30 it ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile(); pr.enable(); run(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
