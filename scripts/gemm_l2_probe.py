"""L2 reuse probe for the grouped GEMMs (development aid).  Under ncu:

    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
        -k regex:grouped_gemm python scripts/gemm_l2_probe.py

8 experts x 8192 rows (Mixtral prefill 8 x 4096 tokens, k = 2).  Ideal DRAM
reads: up 0.54 GB x + 1.88 GB W1|W3; down 0.94 GB W2 + 1.88 GB act per
n-group pass.  mode = kernel | policy << 4 | demote << 8.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import model as M, ops  # noqa: E402

d, ffn, E = 4096, 14336, 8
m = M.MoEModel(P.ModelShape(1, E, 2), d, ffn, seed=0, resident_layers=[0])
so = m.slot_of[0]
rows = E * 8192
x = torch.empty((rows, d), dtype=torch.bfloat16, device="cuda")
ops.fill_uniform_bf16(x, 1, 7, 1.0)
act = torch.empty((rows, ffn), dtype=torch.bfloat16, device="cuda")
ops.fill_uniform_bf16(act, 1, 8, 1.0)
off = torch.arange(E + 1, dtype=torch.int64, device="cuda") * 8192
CASES = [("up", 0, 64, 0), ("up", 0, 64, 1), ("up", 2, 64, 1), ("up", 0, 128, 1),
         ("down", 2, -8, 0), ("down", 2, -8, 2), ("down", 3, -8, 2), ("down", 3, -16, 2),
         ("down", 2, -4, 2)]
if __name__ == "__main__":
    for which, pol, g, dem in CASES:
        ops.set_gemm_mode((pol << 4) | (dem << 8))
        for _ in range(2):
            if which == "up":
                ops.expert_gemm_up(x, off, so, m.slab, m.n_slots, m.slot_elems, d, ffn, g)
            else:
                ops.expert_gemm_down(act, off, so, m.slab, m.n_slots, m.slot_elems, d, ffn, g)
        torch.cuda.synchronize()
        print(which, pol, g, dem, flush=True)
    ops.set_gemm_mode(0)
