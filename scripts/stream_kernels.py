"""Steady-state timing of the HBM-bound prefill kernels (router, permutation
gather, combine) at BASELINE configs[3] (8 x 4096 tokens, Mixtral-8x7B),
CUDA events per launch, an L2 flush (256 MB write) before each launch.

    python scripts/stream_kernels.py [reps]
Prints per-kernel median us and GB/s of algorithmic bytes (development aid).
"""

import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
T, d, E, k = 32768, 4096, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, 512, seed=0, resident_layers=[])
h = m.input_hidden(T, stream=5)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return ts


res = {}
ops.set_router_mode(True, bulk=True)
res["router_bulk"] = (timed(lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)), T * d * 6)
for pf in (0, 1):
    ops.set_router_mode(True, prefetch=pf, bulk=False)
    res[f"router_single_pf{pf}"] = (timed(lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1],
                                                             k)), T * d * 6)
ops.set_router_mode(False)
res["router_two_pass"] = (timed(lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)),
                          T * d * 6)
ops.set_router_mode(True, prefetch=int(os.environ.get("DAOP_PF", "1")), bulk=True)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
x, idx, w = r["x"], r["topk_idx"], r["topk_w"]
res["permute_only"] = (timed(lambda: ops.permute(idx, E)), T * k * 16)
for var, ctas in ((0, 2), (0, 4), (0, 8), (1, 0)):
    ops.set_stream_mode(gather=var, gather_ctas_per_sm=ctas or 2)
    res[f"permute+gather_v{var}_c{ctas}"] = (timed(lambda: ops.permute(idx, E, x)), T * d * 2 * 3)
ops.set_stream_mode(0, 0, 2, 4)
pr = ops.permute(idx, E, x)
y = torch.randn((T * k, d), device="cuda")
for var, st in ((0, 2), (0, 3), (0, 4), (1, 0)):
    ops.set_stream_mode(combine=var, combine_stages=st or 4, gather_ctas_per_sm=2)
    res[f"combine_v{var}_s{st}"] = (timed(lambda: ops.combine(h, y, pr["inv"], w)), T * d * 4 * 4)
ops.set_stream_mode(0, 0, 2, 4)
out = {}
for key, (ts, nbytes) in res.items():
    med = statistics.median(ts)
    out[key] = {"us_median": round(med, 1), "us_min": round(min(ts), 1),
                "gbs": round(nbytes / med / 1e3, 1)}
print(json.dumps(out, indent=1))
