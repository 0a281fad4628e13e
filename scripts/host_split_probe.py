"""Does a pinned-host -> HBM DMA stream slow the host-tier expert GEMV?
If not, a slow expert can be split: part of its rows computed on the host,
the rest DMA'd to HBM and computed on the GPU, both reading host DRAM."""
import statistics
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.daop import HostExpertPool, host_expert_ffn  # noqa: E402

d, ffn = 4096, 14336
pool = HostExpertPool(P.ModelShape(1, 4, 1), d, ffn, seed=0)
x = np.random.default_rng(0).integers(0, 1 << 15, (1, d)).astype(np.uint16) & 0x3fff
src = pool.slot(0, 3)
dst = torch.empty_like(src, device="cuda")


def host_times(n=8):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        host_expert_ffn(pool, 0, 0, x)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


host_expert_ffn(pool, 0, 0, x)
print("host alone  %.3f ms" % host_times())
s = torch.cuda.Stream()
for th in (16, 12, 8):
    stop = False
    nbytes = [0]

    def dma():
        with torch.cuda.stream(s):
            while not stop:
                dst.copy_(src, non_blocking=True)
                s.synchronize()
                nbytes[0] += src.numel() * 2
    t = threading.Thread(target=dma)
    t0 = time.perf_counter()
    t.start()
    time.sleep(0.05)
    ts = []
    for _ in range(8):
        a = time.perf_counter()
        host_expert_ffn(pool, 0, 0, x, th)
        ts.append(time.perf_counter() - a)
    stop = True
    t.join()
    el = time.perf_counter() - t0
    print("threads %2d: host with DMA %.3f ms, DMA %.1f GB/s" %
          (th, statistics.median(ts) * 1e3, nbytes[0] / el / 1e9))
    ts = []
    for _ in range(8):
        a = time.perf_counter()
        host_expert_ffn(pool, 0, 0, x, th)
        ts.append(time.perf_counter() - a)
    print("threads %2d: host alone %.3f ms" % (th, statistics.median(ts) * 1e3))
torch.cuda.synchronize()
a = time.perf_counter()
for _ in range(4):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
print("DMA alone %.1f GB/s" % (4 * src.numel() * 2 / (time.perf_counter() - a) / 1e9))
