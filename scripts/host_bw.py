"""Host-tier bandwidth probe (development aid): stream-read ceiling of the
host memory vs the slow-tier SwiGLU GEMV (daop_host_expert_ffn), per thread
count, on pinned and pageable buffers.  python scripts/host_bw.py"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_10375_b200 import _lib  # noqa: E402

d, ffn = 4096, 14336
nthreads = len(os.sched_getaffinity(0))
print("host threads", nthreads, "cpu", open("/proc/cpuinfo").read().count("processor"))
buf = torch.empty(3 * d * ffn, dtype=torch.bfloat16, pin_memory=True)
buf.view(torch.int16).random_(-100, 100)
pg = torch.empty(3 * d * ffn, dtype=torch.bfloat16)
pg.copy_(buf)
cs = ctypes.c_double(0)
x = np.random.default_rng(0).integers(0, 1 << 15, size=d, dtype=np.uint16)
y = np.empty(d, dtype=np.float32)
for th in sorted({1, 2, 4, 8, nthreads, 2 * nthreads}):
    for name, b in (("pinned", buf), ("pageable", pg)):
        nb = b.numel() * 2
        _lib.call("daop_host_stream_read", b.data_ptr(), nb, th, ctypes.addressof(cs))
        t = time.perf_counter()
        for _ in range(3):
            _lib.call("daop_host_stream_read", b.data_ptr(), nb, th, ctypes.addressof(cs))
        rd = 3 * nb / (time.perf_counter() - t) / 1e9
        p = b.data_ptr()
        w1, w3, w2 = p, p + d * ffn * 2, p + 2 * d * ffn * 2
        _lib.call("daop_host_expert_ffn", x.ctypes.data, 1, w1, w3, w2, d, ffn, y.ctypes.data, 0, th)
        t = time.perf_counter()
        for _ in range(3):
            _lib.call("daop_host_expert_ffn", x.ctypes.data, 1, w1, w3, w2, d, ffn, y.ctypes.data,
                      0, th)
        dt = (time.perf_counter() - t) / 3
        print(f"threads {th:3d} {name:8s} read {rd:6.1f} GB/s   expert GEMV {dt*1e3:6.2f} ms "
              f"= {nb / dt / 1e9:6.1f} GB/s", flush=True)
caps = np.zeros(2, dtype=np.int32)
_lib.call("daop_host_caps", caps.ctypes.data, caps.ctypes.data + 4)
print("caps: avx512_bf16", bool(caps[0] & 1), "amx", bool(caps[0] & 2))
p = buf.data_ptr()
w1, w3, w2 = p, p + d * ffn * 2, p + 2 * d * ffn * 2
for n in (16, 64, 128, 256):
    xs = np.random.default_rng(1).integers(0, 1 << 14, size=(n, d), dtype=np.uint16)
    ys = np.empty((n, d), dtype=np.float32)
    _lib.call("daop_host_expert_ffn", xs.ctypes.data, n, w1, w3, w2, d, ffn, ys.ctypes.data, 0, 0)
    t = time.perf_counter()
    for _ in range(3):
        _lib.call("daop_host_expert_ffn", xs.ctypes.data, n, w1, w3, w2, d, ffn, ys.ctypes.data,
                  0, 0)
    dt = (time.perf_counter() - t) / 3
    print(f"batched expert n={n:4d}: {dt*1e3:7.2f} ms  {2*n*3*d*ffn/dt/1e12:6.2f} TFLOP/s  "
          f"{3*d*ffn*2/dt/1e9:6.1f} GB/s of weights", flush=True)
