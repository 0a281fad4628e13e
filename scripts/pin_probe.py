"""How fast can the host expert pool (90 GB pinned for Mixtral-8x7B) be
allocated?  torch's pin_memory (cudaHostAlloc, 4 KB pages faulted by one
thread) vs mmap + MADV_HUGEPAGE + parallel first touch + cudaHostRegister.

    python scripts/pin_probe.py [GB]
"""

import ctypes
import json
import mmap
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 16.0
nbytes = int(gb * (1 << 30))
res = {"gb": gb}

t = time.perf_counter()
a = torch.empty(nbytes // 2, dtype=torch.bfloat16, pin_memory=True)
res["torch_pin_memory_s"] = time.perf_counter() - t
del a

libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                      ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
libc.munmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
MADV_HUGEPAGE = 14
for huge in (True, False):
    t = time.perf_counter()
    ptr = libc.mmap(None, nbytes, mmap.PROT_READ | mmap.PROT_WRITE,
                    mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    if huge:
        libc.madvise(ptr, nbytes, MADV_HUGEPAGE)
    th = len(os.sched_getaffinity(0))
    chunk = (nbytes + th - 1) // th

    def touch(i):
        a0 = i * chunk
        n = min(chunk, nbytes - a0)
        if n > 0:
            ctypes.memset(ptr + a0, 0, n)

    with ThreadPoolExecutor(th) as ex:
        list(ex.map(touch, range(th)))
    t_touch = time.perf_counter() - t
    rt = torch.cuda.cudart()
    r = rt.cudaHostRegister(ptr, nbytes, 1)  # cudaHostRegisterPortable
    t_reg = time.perf_counter() - t - t_touch
    key = "mmap_huge" if huge else "mmap_4k"
    res[key] = {"touch_s": t_touch, "register_s": t_reg, "rc": int(r)}
    # is torch treating it as pinned, and how fast is a copy?
    buf = (ctypes.c_uint16 * (nbytes // 2)).from_address(ptr)
    import numpy as np
    ht = torch.from_numpy(np.ctypeslib.as_array(buf))
    res[key]["torch_is_pinned"] = bool(ht.is_pinned())
    d = torch.empty(1 << 28, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(8):
        d.copy_(ht[i * (1 << 28):(i + 1) * (1 << 28)], non_blocking=True)
    torch.cuda.synchronize()
    res[key]["h2d_gbs"] = 8 * (1 << 29) / (time.perf_counter() - t) / 1e9
    rt.cudaHostUnregister(ptr)
    libc.munmap(ptr, nbytes)
print(json.dumps(res))
