import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import test_linalg_gpu as T
from paper_2401_01921_b200 import UniTensor, storage, linalg as L
rng = np.random.default_rng(3)
for m, n in [(7, 9), (9, 7), (33, 33), (64, 130), (8, 8), (2, 3), (3, 2)]:
    a = rng.standard_normal((m, n))
    t = UniTensor(storage.from_numpy(a), labels=["r", "c"], rowrank=1)
    s, u, v = L.svd(t)
    U, S, V = u.get_block_().numpy(), s.get_block_().numpy(), v.get_block_().numpy()
    print((m, n), "rec", np.linalg.norm(U @ S @ V - a) / np.linalg.norm(a), "UtU", np.linalg.norm(U.T @ U - np.eye(U.shape[1])),
          "VVt", np.linalg.norm(V @ V.T - np.eye(V.shape[0])))
