"""configs[3] prefill layer with the GEMMs' persisting-L2 set-aside on vs off
(daop_set_gemm_mode bit 11), interleaved on one box: per-op CUDA-event times
(development aid, GPU box)."""
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
    record.append(ev)


for rep in range(3):
    for tag, mode in (("set-aside on", 1 << 11), ("set-aside off", 0)):
        ops.set_gemm_mode(mode)
        recs = []
        for _ in range(2):
            layer([])
        for _ in range(6):
            layer(recs)
        torch.cuda.synchronize()
        acc = {n: np.median([ev[i].elapsed_time(ev[i + 1]) * 1e3 for ev in recs])
               for i, n in enumerate(names)}
        tot = recs[0][0].elapsed_time(recs[-1][5]) / len(recs)
        print(f"rep {rep} {tag:14s} layer {tot:.3f} ms  ops (us):",
              {n: round(float(v), 1) for n, v in acc.items()}, flush=True)
ops.set_gemm_mode(0)
