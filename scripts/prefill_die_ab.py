"""A/B of the per-die GEMM schedule on the whole configs[3] prefill layer
(router, permutation, grouped GEMMs, combine), alternating plain / per-die on
the same box (development aid, GPU box)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import _lib  # noqa: E402
from paper_2501_10375_b200.engine import MoEBlockEngine  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

d, ffn, E, k, T = 4096, 14336, 8, 2, 32768
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
eng = MoEBlockEngine(m)
h = m.input_hidden(T, stream=5)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
res = {"plain": [], "per-die": []}
for rep in range(3):
    for name, arg in (("plain", 0), ("per-die", -1)):
        _lib.call("daop_set_gemm_die_table", 0, arg)
        for _ in range(2):
            eng.prefill(h, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            eng.prefill(h, 0)
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / n)
        print(f"rep {rep} {name:8s} {res[name][-1]:7.3f} ms/layer", flush=True)
for k_, v in res.items():
    print(f"{k_:8s} median {np.median(v):7.3f} ms/layer")
