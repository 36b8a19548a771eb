"""T1.W narrow step at chi = 1024 (and c128): kernel time of the row-panel kernel vs the
per-lane gather kernel (TNB_NO_SLAB=1 in a second process) (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import UniTensor, contract, storage

torch.cuda.set_device(0)
tag = "gather" if os.environ.get("TNB_NO_SLAB") else "slab"
for dt in (np.float64, np.complex128):
    chi, D, d = 1024, 5, 2
    rng = np.random.default_rng(1)
    t1 = rng.standard_normal((d, chi, chi, D)).astype(dt)
    W = rng.standard_normal((D, D, d, d)).astype(dt)
    T1 = UniTensor(storage.from_numpy(t1), labels=["p", "vr", "b", "w"])
    Wt = UniTensor(storage.from_numpy(W), labels=["w", "w2", "q", "p"])
    for _ in range(3):
        contract(T1, Wt)
    torch.cuda.synchronize()
    tnb._lib.ktimer_reset()
    tnb._lib.ktimer_enable(True)
    n = 20
    for _ in range(n):
        contract(T1, Wt)
    torch.cuda.synchronize()
    tnb._lib.ktimer_enable(False)
    k, ms, _ = tnb._lib.ktimer_read(tnb._lib.KF_GEMM_SKINNY)
    byts = 2 * t1.nbytes
    print(f"[{tag}] {np.dtype(dt).name} T1.W chi={chi}: {ms / max(k, 1) * 1e3:.1f} us/launch "
          f"({byts / (ms / max(k, 1)) / 1e6:.0f} GB/s, {byts / (ms / max(k, 1)) / 1e6 / 6547:.2f} of HBM)")
# reference point: a device-to-device copy of the same bytes, same loop
x = torch.empty(2 * 1024 * 1024 * 5, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    y.copy_(x)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 20
print(f"torch copy of {x.nbytes / 1e6:.0f} MB: {t * 1e3:.1f} us ({2 * x.nbytes / t / 1e6:.0f} GB/s)")
