"""T1.W step alone at chi=1024 f64 / c128: slab-narrow vs the previous narrow kernel (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import torch

import tnkit_np as oracle
import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import UniTensor, storage

torch.cuda.set_device(0)
for dt in (np.float64, np.complex128):
    chi = 1024
    t1 = oracle.normal([2, chi, chi, 5], dtype=dt, seed=1)
    w = oracle.normal([5, 5, 2, 2], dtype=dt, seed=2)
    T1 = UniTensor(storage.from_numpy(t1), labels=["p", "vr", "b", "w"])
    W = UniTensor(storage.from_numpy(w), labels=["w", "w2", "q", "p"])
    out = tnb.contract(T1, W)
    want, _ = oracle.contract_dense(t1, ["p", "vr", "b", "w"], w, ["w", "w2", "q", "p"])
    err = np.linalg.norm(out.numpy() - want) / np.linalg.norm(want)
    for _ in range(3):
        tnb.contract(T1, W)
    torch.cuda.synchronize()
    tnb._lib.ktimer_reset()
    tnb._lib.ktimer_enable(True)
    for _ in range(20):
        tnb.contract(T1, W)
    torch.cuda.synchronize()
    tnb._lib.ktimer_enable(False)
    k, ms, _ = tnb._lib.ktimer_read(tnb._lib.KF_GEMM_SKINNY)
    nb = (t1.nbytes + want.nbytes)
    print(f"{np.dtype(dt).name}: {ms / k * 1e3:.1f} us per T1.W launch, {nb / (ms / k) / 1e6:.0f} GB/s, rel err {err:.1e}")
