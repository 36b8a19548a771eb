"""Host->device bandwidth on the box: one pinned 100 MB copy vs split over 2 / 4 streams (dev aid)."""
import torch

torch.cuda.set_device(0)
n = 100 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for _ in range(2):
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[k * n // ns:(k + 1) * n // ns].copy_(h[k * n // ns:(k + 1) * n // ns], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for _ in range(5):
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[k * n // ns:(k + 1) * n // ns].copy_(h[k * n // ns:(k + 1) * n // ns], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    print(f"{ns} streams: {5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
# D2H
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    h.copy_(d, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"D2H: {5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
