"""8x22B (EP, one GPU) prefill GEMM groups with the per-die schedule: the up
and down GEMMs on the layer's own permuted rows, CUDA-event timed per
(group_up, group_down) (development aid, GPU box)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

d, ffn, E, k, T = 6144, 16384, 8, 2, 32768
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
h = m.input_hidden(T, stream=5)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
pr = ops.permute(r["topk_idx"], E, r["x"])
act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab, m.n_slots,
                         m.slot_elems, d, ffn)


def timed(fn, n=int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for g in (16, 32, 64):
        ms = timed(lambda: ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab,
                                               m.n_slots, m.slot_elems, d, ffn, g))
        print(f"rep {rep} up   group {g:4d}: {ms:7.3f} ms", flush=True)
    for g in (-4, -8, -16):
        ms = timed(lambda: ops.expert_gemm_down(act, pr["offsets"], m.slot_of[0], m.slab,
                                                 m.n_slots, m.slot_elems, d, ffn, g))
        print(f"rep {rep} down group {g:4d}: {ms:7.3f} ms", flush=True)
