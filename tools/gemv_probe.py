"""Dev aid: fp64 tall-skinny GEMV variants for the Lanczos reorthogonalisation."""
import time, torch
n = 2 * 1024 * 1024
b = torch.randn(31, n, dtype=torch.float64, device="cuda")
w = torch.randn(n, dtype=torch.float64, device="cuda")
c = torch.randn(31, dtype=torch.float64, device="cuda")
def t(f, name):
    for _ in range(3): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): f()
    torch.cuda.synchronize(); print(name, "ms %.3f" % ((time.perf_counter() - t0) / 10 * 1e3))
t(lambda: b @ w, "b @ w (gemv)")
t(lambda: (b * w).sum(1), "(b*w).sum(1)")
t(lambda: torch.einsum("rsk,sk->rs", b.view(31, 512, -1), w.view(512, -1)).sum(1), "split einsum")
t(lambda: b.T @ c, "b.T @ c (gemv)")
t(lambda: c @ b, "c @ b (gemv)")
t(lambda: (b * c[:, None]).sum(0), "(b*c).sum(0)")
