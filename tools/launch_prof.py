"""Dev aid: host-side cProfile of an eager L.A.W.R Network.launch at chi=128."""
import cProfile, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import bench, paper_2401_01921_b200 as tnb
net, _ = bench.lawr_network(tnb, bench.WL.lawr_inputs(128, dtype=np.float64, seed=1))
for _ in range(20):
    net.launch()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    net.launch()
torch.cuda.synchronize()
print("wall us per launch", (time.perf_counter() - t0) / 200 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    net.launch()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
