"""Skinny GEMMs alone at one batch size (profiling aid): python scripts/skinny_probe.py B"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
d, ffn, E, k = 4096, 14336, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
h = m.input_hidden(B, stream=9)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
pr = ops.permute(r["topk_idx"], E, r["x"])
so = m.slot_of[0]
for _ in range(3):
    act = ops.expert_gemm_up_skinny(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots,
                                    m.slot_elems, d, ffn)
    y = ops.expert_gemm_down_skinny(act, pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d,
                                    ffn)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
for _ in range(20):
    act = ops.expert_gemm_up_skinny(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots,
                                    m.slot_elems, d, ffn)
e[1].record()
for _ in range(20):
    y = ops.expert_gemm_down_skinny(act, pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d,
                                    ffn)
e[2].record()
torch.cuda.synchronize()
up, dn = e[0].elapsed_time(e[1]) / 20 * 1e3, e[1].elapsed_time(e[2]) / 20 * 1e3
print(f"b={B}: up {up:.1f} us ({8 * 2 * ffn * d * 2 / up / 1e3:.0f} GB/s)  "
      f"down {dn:.1f} us ({8 * ffn * d * 2 / dn / 1e3:.0f} GB/s)")
