"""Gathered up GEMM vs dense (debug aid, GPU box): python scripts/gather_probe.py MODE"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

mode = int(sys.argv[1], 0) if len(sys.argv) > 1 else 0
d, ffn, E, T = 512, 1024, 8, int(sys.argv[2]) if len(sys.argv) > 2 else 700
print("start", flush=True)
m = MoEModel(P.ModelShape(2, E, 2), d, ffn, seed=8, resident_layers=[0])
torch.cuda.synchronize()
print("model", flush=True)
h = m.input_hidden(T, stream=5)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], 2)
pr = ops.permute(r["topk_idx"], E, r["x"])
so = m.slot_of[0]
ops.set_gemm_mode(mode)
ref = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn)
torch.cuda.synchronize()
print("dense ok", flush=True)
got = ops.expert_gemm_up_gather(r["x"], pr["perm"], 2, pr["offsets"], so, m.slab, m.n_slots,
                                m.slot_elems, d, ffn)
torch.cuda.synchronize()
n = int(pr["offsets"][-1])
print("gather done; equal:", torch.equal(got[:n], ref[:n]),
      "mismatch rows:", int((got[:n] != ref[:n]).any(1).sum()), flush=True)
