"""Quick A/B timing for library variants (TNB_LIB_PATH): single C4, 64 x C4 batched (bs
kernel time), and the chi=1024 f64 L.A.W.R launch (GEMM kernel time + whole-launch events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import bench
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import workloads as WL


def ktime(fn, fam, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tnb._lib.ktimer_reset()
    tnb._lib.ktimer_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # a sleeping kernel first: the host queues all n calls before the GPU reaches them, so the
    # events see device time, not the host's per-call overhead
    torch.cuda._sleep(int(os.environ.get("TNB_AB_SLEEP", "20000000")))
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    tnb._lib.ktimer_enable(False)
    k, ms, _ = tnb._lib.ktimer_read(fam)
    return ms / n, e0.elapsed_time(e1) / n


torch.cuda.set_device(0)
what = sys.argv[1:] or ["bs", "lawr"]
tag = os.path.basename(os.environ.get("TNB_LIB_PATH", "libtnb.so"))
if "bs" in what:
    A, E = bench.c4_tensors(tnb)
    pairs = [bench.c4_tensors(tnb, seed=777 + 2 * i) for i in range(64)]
    t1, _ = ktime(lambda: tnb.contract(A, E), tnb._lib.KF_BS_GEMM)
    tb, _ = ktime(lambda: tnb.contract_batched(pairs), tnb._lib.KF_BS_GEMM, 5)
    f = 2 * bench.C4_MACS
    print(f"[{tag}] bs single {t1 * 1e3:.1f} us ({f / t1 / 1e9 / 37.06:.3f})  batch64 {tb:.3f} ms "
          f"({64 * f / tb / 1e9 / 37.06:.3f})")
if "lawr" in what:
    for dt in (np.float64, np.complex128):
        net, _ = bench.make_network(tnb, WL.LAWR_NET, WL.lawr_inputs(1024, dtype=dt))
        g, w = ktime(net.launch, tnb._lib.KF_GEMM)
        macs, _ = bench.lawr_macs(tnb, 1024)
        fl = macs * (8 if dt == np.complex128 else 2)
        print(f"[{tag}] lawr1024 {np.dtype(dt).name} gemm {g:.3f} ms launch {w:.3f} ms ({fl / w / 1e9:.0f} GF/s)")
if "c1" in what:
    net, _ = bench.make_network(tnb, WL.LAWR_NET, WL.lawr_inputs(128))
    g, w = ktime(net.launch, tnb._lib.KF_GEMM, 50)
    cn = net.compile()
    _, wg = ktime(cn.launch, tnb._lib.KF_GEMM, 50)
    print(f"[{tag}] C1 chi128: gemm {g * 1e3:.1f} us/launch, eager launch {w * 1e3:.1f} us, graph {wg * 1e3:.1f} us")
