import sys
import torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import model as M, ops
d, ffn, E = 4096, 14336, 8
m = M.MoEModel(P.ModelShape(1, E, 2), d, ffn, seed=0, resident_layers=[0])
so = m.slot_of[0]
x = torch.empty((E * 8192, d), dtype=torch.bfloat16, device="cuda")
ops.fill_uniform_bf16(x, 1, 7, 1.0)
act = torch.empty((E * 8192, ffn), dtype=torch.bfloat16, device="cuda")
ops.fill_uniform_bf16(act, 1, 8, 1.0)
off = torch.arange(E + 1, dtype=torch.int64, device="cuda") * 8192
for dem in (4, 5, 0, 4, 1, 5):
    ops.set_gemm_mode((0 << 4) | (dem << 8))
    for _ in range(2):
        ops.expert_gemm_up(x, off, so, m.slab, m.n_slots, m.slot_elems, d, ffn, 64)
    torch.cuda.synchronize()
for pol, g, dem in ((2, -8, 4), (2, -8, 6), (3, -8, 6), (2, -8, 0), (3, -16, 6)):
    ops.set_gemm_mode((pol << 4) | (dem << 8))
    for _ in range(2):
        ops.expert_gemm_down(act, off, so, m.slab, m.n_slots, m.slot_elems, d, ffn, g)
    torch.cuda.synchronize()
