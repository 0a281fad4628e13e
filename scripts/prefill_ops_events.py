"""configs[3] prefill layer (8 x 4096 tokens, Mixtral-8x7B): CUDA-event time of
each op inside back-to-back layers, and of the router / gather / combine run
alone back to back (development aid, GPU box).  HBM bytes per op are the
algorithmic ones."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

d, ffn, E, k, T = 4096, 14336, 8, 2, 32768
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
h = m.input_hidden(T, stream=5)
hist = torch.zeros((8, E), dtype=torch.int32, device="cuda")
names = ["router", "permute+gather", "up", "down", "combine"]
acc = {n: [] for n in names}


def layer(record):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k, hist=hist, tokens_per_seq=4096,
                   hist_seq_stride=E)
    ev[1].record()
    pr = ops.permute(r["topk_idx"], E, r["x"])
    ev[2].record()
    act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab, m.n_slots,
                             m.slot_elems, d, ffn)
    ev[3].record()
    y = ops.expert_gemm_down(act, pr["offsets"], m.slot_of[0], m.slab, m.n_slots, m.slot_elems,
                             d, ffn)
    ev[4].record()
    ops.combine(h, y, pr["inv"], r["topk_w"])
    ev[5].record()
    if record is not None:
        record.append(ev)
    return r, pr, y


for _ in range(2):
    layer(None)
recs = []
for _ in range(6):
    layer(recs)
torch.cuda.synchronize()
for ev in recs:
    for i, n in enumerate(names):
        acc[n].append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
tot = sum(np.median(v) for v in acc.values())
print("inside back-to-back layers (us, median):",
      {n: round(float(np.median(v)), 1) for n, v in acc.items()}, f"sum {tot / 1e3:.3f} ms")
import threading  # noqa: E402
import time  # noqa: E402

import pynvml  # noqa: E402

pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)


def clocks(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_MEM)))
        time.sleep(0.002)


r, pr, y = layer(None)
by = {"router": 537e6 + 268e6 + 2 * T * E * 4 + T * k * 8,
      "permute+gather": 2 * 268e6, "combine": 537e6 * 2 + T * k * d * 4}
fns = (("router", lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], k, hist=hist,
                                      tokens_per_seq=4096, hist_seq_stride=E)),
       ("permute+gather", lambda: ops.permute(r["topk_idx"], E, r["x"])),
       ("combine", lambda: ops.combine(h, y, pr["inv"], r["topk_w"])))
for when in ("right after the GEMMs", "after 3 s idle", "after 3 s idle"):
    if when != "right after the GEMMs":
        torch.cuda.synchronize()
        time.sleep(3.0)
    else:
        layer(None)
    alone = {}
    for n, fn in fns:
        samples, stop = [], threading.Event()
        th = threading.Thread(target=clocks, args=(stop, samples))
        th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        us = e0.elapsed_time(e1) / 20 * 1e3
        sm = int(np.median([a for a, _ in samples])) if samples else -1
        mem = int(np.median([b for _, b in samples])) if samples else -1
        alone[n] = (round(us, 1), round(by[n] / us / 1e6, 2), f"sm {sm} MHz mem {mem} MHz")
    print(f"alone, 20 back to back, {when} (us, TB/s algorithmic):", alone, flush=True)
