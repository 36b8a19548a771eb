"""cuBLAS DGEMM / ZGEMM probe (measurement only; never on the product path)."""
import torch, json
res = {}
for dt, name in ((torch.float64, "dgemm"), (torch.complex128, "zgemm")):
    n = 8192 if dt == torch.float64 else 4096
    a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    flop = 2 * n**3 * (4 if dt == torch.complex128 else 1)
    res[name] = flop / best / 1e9
print(json.dumps({"cublas_tflops": res}))
