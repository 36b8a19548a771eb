"""Dev aid: event timeline of one e2e L.A.W.R step (chunk landings on the upload stream,
panel completions on the compute stream) -- every torch.cuda.Event the engine records is
made a timing event and logged."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

LOG = []
_Ev = torch.cuda.Event


class TEvent(_Ev):
    def __new__(cls, enable_timing=False, blocking=False, interprocess=False):
        return super().__new__(cls, enable_timing=True, blocking=blocking, interprocess=interprocess)

    def record(self, stream=None):
        super().record(stream)
        s = stream if stream is not None else torch.cuda.current_stream()
        LOG.append((self, s.cuda_stream))


torch.cuda.Event = TEvent
import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import dense
from paper_2401_01921_b200 import workloads as WL

torch.cuda.set_device(0)
chi = 1024
inp = WL.lawr_inputs(chi, dtype=np.float64, seed=1)
net, tensors = bench.lawr_network(tnb, inp)
pinned = {nm: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for nm, a in inp.items()}
probe = net.launch().get_block_().contiguous().storage()
out_host = torch.empty(probe.shape, dtype=probe.dtype, pin_memory=True)
first_use = tnb.tree_leaves(tnb.parse_order(net.get_order()))
# per-tensor chunk weights, e.g.  A=1 L=1,2,3,3 R=3,1
pat = {"A": "4", "L": "4", "R": "4", "W": "1"}
for a in sys.argv[1:]:
    k, v = a.split("=")
    pat[k] = v
chunks = {k: (int(v) if "," not in v else tuple(float(x) for x in v.split(","))) for k, v in pat.items()}
print("chunks", chunks)


def step():
    for nm in first_use:
        tensors[nm].get_block_().upload_(pinned[nm], chunks=chunks[nm])
    net.launch(host_out=out_host)


for _ in range(3):
    step()
torch.cuda.synchronize()
names = {torch.cuda.current_stream().cuda_stream: "compute", dense.upload_stream().cuda_stream: "upload",
         dense.download_stream().cuda_stream: "download"}
tot = []
for rep in range(5):
    LOG.clear()
    if rep == 4:
        tnb._lib.ktimer_reset()
        tnb._lib.ktimer_enable(True)
    t0 = TEvent()
    t0.record()
    step()
    t1 = TEvent()
    t1.record()
    torch.cuda.synchronize()
    tot.append(t0.elapsed_time(t1))
    if rep == 4:
        print(" ".join(f"{names.get(s, s)[0]}{t0.elapsed_time(ev):.3f}" for ev, s in LOG[1:-1]))
tnb._lib.ktimer_enable(False)
print("step ms median", sorted(tot)[2], "gemm launches (n, ms)", tnb._lib.ktimer_read(tnb._lib.KF_GEMM)[:2],
      "skinny", tnb._lib.ktimer_read(tnb._lib.KF_GEMM_SKINNY)[:2])
