"""Does the GPU pulling expert weights over PCIe from the pinned pool slow the
host tier's expert GEMV (shared host DRAM)?  Host experts alone, H2D copies
alone, then both at once (development aid, GPU box)."""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.daop import HostExpertPool, host_expert_ffn  # noqa: E402

L, E, D, FFN = 4, 8, 4096, 14336
pool = HostExpertPool(P.ModelShape(L, E, 2), D, FFN, seed=0, device=torch.device("cuda"))
xs = np.random.default_rng(0).standard_normal((1, D)).astype(np.float32)
dst = torch.empty(pool.slot_elems, dtype=torch.bfloat16, device="cuda")
side = torch.cuda.Stream()


def host_loop(n, out):
    t0 = time.perf_counter()
    for i in range(n):
        host_expert_ffn(pool, 1, i % E, xs)
    out.append((time.perf_counter() - t0) / n * 1e3)


def h2d_loop(n, out):
    with torch.cuda.stream(side):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(n):
            dst.copy_(pool.buf[2 * E + i % E], non_blocking=True)
        b.record()
    b.synchronize()
    out.append(n * pool.slot_elems * 2 / (a.elapsed_time(b) / 1e3) / 1e9)


for _ in range(2):
    r = []
    host_loop(8, r)
    print(f"host expert alone: {r[-1]:.2f} ms ({pool.slot_elems * 2 / r[-1] / 1e6:.0f} GB/s)")
    r = []
    h2d_loop(16, r)
    print(f"H2D alone: {r[-1]:.1f} GB/s")
    rh, rc = [], []
    th = threading.Thread(target=h2d_loop, args=(60, rc))
    th.start()
    time.sleep(0.05)
    host_loop(16, rh)
    th.join()
    print(f"together: host expert {rh[-1]:.2f} ms ({pool.slot_elems * 2 / rh[-1] / 1e6:.0f} GB/s), "
          f"H2D {rc[-1]:.1f} GB/s", flush=True)
