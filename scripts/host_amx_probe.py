"""(historical A/B: the prefetch was reverted -- the AMX experts are compute-bound)
Host-tier AMX expert time (prefill-sized token batches) with and without the
software prefetch of the next weight block (DAOP_HOST_PREFETCH=0/1; run once
per setting: the switch is read once per process).  Development aid; any host."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2501_10375_b200 import _lib  # noqa: E402

d, ffn, NE = 4096, 14336, 6
rng = np.random.default_rng(0)
W = [(rng.integers(0, 1 << 15, size=(ffn, d), dtype=np.uint16) & 0x3f7f,
      rng.integers(0, 1 << 15, size=(ffn, d), dtype=np.uint16) & 0x3f7f,
      rng.integers(0, 1 << 15, size=(d, ffn), dtype=np.uint16) & 0x3f7f) for _ in range(NE)]
res = {}
for n in (16, 58, 128, 256):
    x = (rng.integers(0, 1 << 15, size=(n, d), dtype=np.uint16) & 0x3f7f)
    y = np.empty((n, d), dtype=np.float32)
    ts = []
    for rep in range(3):
        for e in range(NE):
            w1, w3, w2 = W[e]
            t0 = time.perf_counter()
            _lib.call("daop_host_expert_ffn", x.ctypes.data, n, w1.ctypes.data, w3.ctypes.data,
                      w2.ctypes.data, d, ffn, y.ctypes.data, 0, 0)
            ts.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.median(ts[NE:]))
    res[n] = (round(ms, 2), round(3 * ffn * d * 2 / ms / 1e6, 1))
print(f"prefetch={os.environ.get('DAOP_HOST_PREFETCH', '1')} ms per expert (GB/s of weights):", res,
      flush=True)
