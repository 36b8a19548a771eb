"""Dev aid: host->device bandwidth with 1/2/4 concurrent copy streams (pinned source)."""
import torch, time
torch.cuda.set_device(0)
N = 100 << 20
x = torch.empty(N, dtype=torch.uint8).pin_memory()
y = torch.empty(N, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = N // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                y[i * chunk:(i + 1) * chunk].copy_(x[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print("streams", ns, "H2D GB/s %.1f" % (N / dt / 1e9))
for ns in (1, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = N // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                x[i * chunk:(i + 1) * chunk].copy_(y[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print("streams", ns, "D2H GB/s %.1f" % (N / dt / 1e9))
