"""Prefill-sized batches: dense (512-row pair tiles) vs skinny (weights as the
M side, 64-token blocks) grouped GEMMs on one Mixtral-8x7B layer, by T."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

m = MoEModel(P.ModelShape(2, 8, 2), 4096, 14336, seed=0, resident_layers=[0])
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(n):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / n


for T in (128, 192, 256, 320, 384, 512, 768, 1024):
    h = m.input_hidden(T, stream=9)
    r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], 2)
    pr = ops.permute(r["topk_idx"], 8, r["x"])
    cnt = (pr["offsets"][1:] - pr["offsets"][:-1]).tolist()
    args = (pr["offsets"], m.slot_of[0], m.slab, m.n_slots, m.slot_elems, 4096, 14336)

    def dense():
        a = ops.expert_gemm_up(pr["x_perm"], *args)
        ops.expert_gemm_down(a, *args)

    def skinny():
        a = ops.expert_gemm_up_skinny(pr["x_perm"], *args, nt=64)
        ops.expert_gemm_down_skinny(a, *args, nt=64)
    print(f"T {T:5d} rows/expert max {max(cnt):4d}: dense {timed(dense):.3f} ms  "
          f"skinny {timed(skinny):.3f} ms", flush=True)
