"""Probe: can pinning the caller's pageable rows in place (cudaHostRegister) beat
staging them through a pinned ring?  Times register + H2D + unregister of a touched
1.6 GB numpy buffer, in whole and in 64 MB chunks, against a plain pageable copy."""
import ctypes
import time

import numpy as np
import torch

N = 1600 << 20
try:
    cudart = ctypes.CDLL("libcudart.so")
except OSError:
    import glob
    import os
    cand = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    cand += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = ctypes.CDLL(cand[0])
torch.cuda.init()
h = np.ones(N, dtype=np.uint8)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
ptr = h.ctypes.data


def reg(p, nbytes):
    t = time.perf_counter()
    rc = cudart.cudaHostRegister(ctypes.c_void_p(p), ctypes.c_size_t(nbytes), 0)
    return rc, time.perf_counter() - t


def unreg(p):
    t = time.perf_counter()
    rc = cudart.cudaHostUnregister(ctypes.c_void_p(p))
    return rc, time.perf_counter() - t


for rep in range(3):
    rc, tr = reg(ptr, N)
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(torch.from_numpy(h), non_blocking=True)
    torch.cuda.synchronize()
    tc = time.perf_counter() - t
    rc2, tu = unreg(ptr)
    print(f"whole: register rc={rc} {tr*1e3:.1f} ms, copy {tc*1e3:.1f} ms, unregister rc={rc2} {tu*1e3:.1f} ms")

C = 64 << 20
for rep in range(3):
    tr = tu = 0.0
    for o in range(0, N, C):
        rc, x = reg(ptr + o, C)
        tr += x
    for o in range(0, N, C):
        rc, x = unreg(ptr + o)
        tu += x
    print(f"chunks of 64 MB: register {tr*1e3:.1f} ms, unregister {tu*1e3:.1f} ms")

for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(torch.from_numpy(h))
    torch.cuda.synchronize()
    print(f"pageable copy (driver staging): {(time.perf_counter() - t)*1e3:.1f} ms")
