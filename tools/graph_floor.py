import torch, time
torch.cuda.set_device(0)
x = torch.zeros(1024, device="cuda")
for nk in (1, 3, 5, 10):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        x.add_(1)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        for _ in range(nk):
            x.add_(1)
    torch.cuda.synchronize()
    torch.cuda._sleep(20000000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{nk} tiny kernels per graph: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per replay")
