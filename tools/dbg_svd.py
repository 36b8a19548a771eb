import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import test_linalg_gpu as T
from paper_2401_01921_b200 import linalg, contract
z, meta = T._z()
name = "two_site_u1_c128"
t = T._build_input(name, z, meta[name])
s, u, v = linalg.svd(t)
A = T._dense_np(t); U = T._dense_np(u); S = T._dense_np(s); V = T._dense_np(v)
Um = U.reshape(-1, U.shape[-1]); Vm = V.reshape(V.shape[0], -1)
rec = (Um @ S @ Vm).reshape(A.shape)
print("numpy rec err", np.linalg.norm(rec - A) / np.linalg.norm(A))
us = contract(u.set_name("U"), s.set_name("S"))
print("U.S err", np.linalg.norm(T._dense_np(us).reshape(-1, S.shape[1]) - Um @ S) / np.linalg.norm(Um @ S))
r2 = contract(us, v)
print("(US).V err", np.linalg.norm(T._dense_np(r2) - rec) / np.linalg.norm(rec))
sc = s.astype(np.complex128)
us2 = contract(u, sc.set_name("S"))
print("U.S(c128) err", np.linalg.norm(T._dense_np(us2).reshape(-1, S.shape[1]) - Um @ S) / np.linalg.norm(Um @ S))
