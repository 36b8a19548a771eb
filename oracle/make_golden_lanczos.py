"""Lanczos golden values from the REFERENCE (tnkit.linalg.lanczos, build container only).

The operator is the Hermitian L.A.W.R effective Hamiltonian of oracle.hermitian_lawr_inputs
(chi = 8) applied through the reference's own Network; tests/golden/lanczos.npz holds the
reference's lowest-2 Ritz values for seeds 3 and 11 and the inputs.  Usage:
    python oracle/make_golden_lanczos.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, HERE)
from tnkit import Network, UniTensor, storage  # noqa: E402
from tnkit.linalg import LinOp, lanczos  # noqa: E402

import tnkit_np as oracle  # noqa: E402

inp = oracle.hermitian_lawr_inputs(8, seed=7)
net = Network(oracle.LAWR_NET)
for nm, arr in inp.items():
    t = UniTensor(storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
    net.put_tensor(nm, t, t.labels)
net.set_order(optimal=True)
shape = inp["A"].shape


def mv(v):
    a = UniTensor(storage.from_numpy(np.asarray(v).reshape(shape)), labels=[f"A{i}" for i in range(3)])
    net.put_tensor("A", a, a.labels)
    return np.ascontiguousarray(net.launch().get_block_().view()).reshape(-1)


out = {f"in_{k}": v for k, v in inp.items()}
for seed in (3, 11):
    theta, _ = lanczos(LinOp(int(np.prod(shape)), matvec=mv), k=2, tol=1e-12, seed=seed)
    out[f"theta_seed{seed}"] = np.asarray(theta)
np.savez_compressed(os.path.join(os.path.dirname(HERE), "tests", "golden", "lanczos.npz"), **out)
print("wrote lanczos.npz", {k: v for k, v in out.items() if k.startswith("theta")})
