"""Dev aid: page-cache read rates for the .utn loader (single vs parallel preads)."""
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = "/tmp/utn_probe.bin"
N = 6138848
with open(path, "wb") as f:
    f.write(np.random.default_rng(0).bytes(N + 1000))
buf = torch.empty(N, dtype=torch.uint8, pin_memory=True)
mv = memoryview(buf.numpy())
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))


def best(fn, k=30):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, sorted(ts)[k // 2] * 1e3


fd = os.open(path, os.O_RDONLY)
print("single preadv ms (best, median)", best(lambda: os.preadv(fd, [mv], 100)))
with open(path, "rb") as f:
    def rd():
        f.seek(100)
        f.readinto(mv)
    print("readinto ms", best(rd))
for nt in (2, 4, 8):
    pool = ThreadPoolExecutor(nt)
    piece = (N + nt - 1) // nt

    def par():
        fs = [pool.submit(os.preadv, fd, [mv[a:a + piece]], 100 + a) for a in range(0, N, piece)]
        for x in fs:
            x.result()
    print(f"pool {nt} threads ms", best(par))
npbuf = np.empty(N, np.uint8)
print("numpy fromfile ms", best(lambda: np.fromfile(path, dtype=np.uint8, count=N, offset=100)))
st = torch.empty(N, dtype=torch.uint8, device="cuda")


def h2d():
    st.copy_(buf, non_blocking=True)
    torch.cuda.synchronize()
print("h2d ms", best(h2d))

pool = ThreadPoolExecutor(4)
piece = 1 << 20


def par_then_copy():
    fs = [pool.submit(os.preadv, fd, [mv[a:min(a + piece, N)]], 100 + a) for a in range(0, N, piece)]
    for x in fs:
        x.result()
    st.copy_(buf, non_blocking=True)
    torch.cuda.synchronize()


def par_piecewise():
    fs = [(a, pool.submit(os.preadv, fd, [mv[a:min(a + piece, N)]], 100 + a)) for a in range(0, N, piece)]
    for a, x in fs:
        x.result()
        st[a:min(a + piece, N)].copy_(buf[a:min(a + piece, N)], non_blocking=True)
    torch.cuda.synchronize()


ev = torch.cuda.Event()


def par_piecewise_ev():
    fs = [(a, pool.submit(os.preadv, fd, [mv[a:min(a + piece, N)]], 100 + a)) for a in range(0, N, piece)]
    for a, x in fs:
        x.result()
        st[a:min(a + piece, N)].copy_(buf[a:min(a + piece, N)], non_blocking=True)
    ev.record()
    ev.synchronize()


print("parallel read then one copy ms", best(par_then_copy))
print("parallel read, piecewise copies ms", best(par_piecewise))
print("parallel read, piecewise copies + event ms", best(par_piecewise_ev))

import mmap
cr = torch.cuda.cudart()
print("cudart has", [a for a in dir(cr) if "Host" in a])
import ctypes
libcudart = None
for nm in ("libcudart.so.12", "libcudart.so"):
    try:
        libcudart = ctypes.CDLL(nm)
        break
    except OSError:
        pass
print("libcudart", libcudart)


def mm_register_copy():
    with open(path, "rb") as f:
        m = mmap.mmap(f.fileno(), 0, prot=mmap.PROT_READ)
        addr = ctypes.addressof(ctypes.c_char.from_buffer_copy(b"x"))  # placeholder
        buf_t = (ctypes.c_char * len(m))
        p = ctypes.c_void_p(ctypes.cast(ctypes.c_char_p(None), ctypes.c_void_p).value)
        mv2 = memoryview(m)
        arr = np.frombuffer(mv2, dtype=np.uint8)
        ptr = arr.ctypes.data
        rc = libcudart.cudaHostRegister(ctypes.c_void_p(ptr), ctypes.c_size_t(len(m)), ctypes.c_uint(8))  # ReadOnly
        if rc != 0:
            raise RuntimeError(f"cudaHostRegister rc {rc}")
        rc = libcudart.cudaMemcpyAsync(ctypes.c_void_p(st.data_ptr()), ctypes.c_void_p(ptr + 100), ctypes.c_size_t(N),
                                       ctypes.c_int(1), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        libcudart.cudaHostUnregister(ctypes.c_void_p(ptr))
        del arr, mv2
        m.close()
        return rc


try:
    print("mmap+register+copy ms", best(mm_register_copy))
    back = st.cpu().numpy()
    ref = np.fromfile(path, dtype=np.uint8, count=N, offset=100)
    print("mmap path correct", np.array_equal(back, ref))
except Exception as e:
    print("mmap register failed", e)
