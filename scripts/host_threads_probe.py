"""Host-tier expert GEMV time vs worker threads (one 8x7B expert, n = 1)."""
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import _lib  # noqa: E402
from paper_2501_10375_b200.daop import HostExpertPool, host_expert_ffn  # noqa: E402

d, ffn = 4096, 14336
pool = HostExpertPool(P.ModelShape(1, 8, 1), d, ffn, seed=0)
x = np.random.default_rng(0).integers(0, 1 << 14, (1, d)).astype(np.uint16)
caps = np.zeros(2, dtype=np.int32)
_lib.call("daop_host_caps", caps.ctypes.data, caps.ctypes.data + 4)
print("affinity", len(os.sched_getaffinity(0)), "caps", caps.tolist(), "cpus", os.cpu_count())
os.system("lscpu | grep -E 'Model name|Thread|Core|Socket|NUMA node|L3' ")
grains = [(0, 0), (32, 16), (64, 32), (16, 8)]
for gu, gd in grains:
  _lib.call("daop_host_set_grain", gu, gd)
  print("grain", gu, gd)
  for th in (12, 14, 15, 16, 0):
    for r in range(2):
        host_expert_ffn(pool, 0, r, x, th)
    ts = []
    for i in range(16):  # rotate experts so nothing is cache-resident
        a = time.perf_counter()
        host_expert_ffn(pool, 0, i % 8, x, th)
        ts.append(time.perf_counter() - a)
    med = statistics.median(ts) * 1e3
    print("  threads %2d: %.3f ms  %.1f GB/s  (min %.3f max %.3f)" %
          (th, med, 352.3 / med, min(ts) * 1e3, max(ts) * 1e3))

# batched experts (prefill slow tier, AMX tiles when n >= 16)
for gu, gd in ((0, 0), (32, 16)):
    _lib.call("daop_host_set_grain", gu, gd)
    for n in (16, 64, 256):
        xb = np.random.default_rng(1).integers(0, 1 << 14, (n, d)).astype(np.uint16)
        host_expert_ffn(pool, 0, 0, xb)
        ts = []
        for i in range(8):
            a = time.perf_counter()
            host_expert_ffn(pool, 0, i % 8, xb)
            ts.append(time.perf_counter() - a)
        med = statistics.median(ts) * 1e3
        print("grain %s n %3d: %.3f ms  %.1f TFLOP/s" %
              ("chunked" if gu else "static ", n, med, 6 * n * d * ffn / med / 1e9))
