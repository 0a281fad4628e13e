"""Minimal launch sequences for ncu captures (never a timing source)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200.engine import MoEBlockEngine
from paper_2501_10375_b200.model import MoEModel

what = sys.argv[1] if len(sys.argv) > 1 else "decode"
import os
from paper_2501_10375_b200 import ops
ops.set_gemm_mode(int(os.environ.get("DAOP_GEMM_MODE", "0")))
d, ffn, E, k = 4096, 14336, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
eng = MoEBlockEngine(m)
if what == "daop_prefill256":  # 256-token prompt, 4 full decoder layers, all experts resident
    import numpy as np
    from paper_2501_10375_b200.daop import DaopEngine, HostExpertPool
    shape = P.ModelShape(4, E, k)
    pool = HostExpertPool(shape, d, ffn, seed=0, device=torch.device("cuda"))
    de = DaopEngine(shape, d, ffn, np.full((4, E), 0.25), 1.0, P.PolicyConfig("daop"), seed=0,
                    host_pool=pool, attention=True, max_seq=512)
    de.prefill_graphs = os.environ.get("DAOP_PF_GRAPH", "1") == "1"
    hp = de.model.input_hidden(256, stream=400)
    for _ in range(3):
        de.prefill(hp)
elif what == "attn_prefill":  # 256-token prompt through one attention layer (tcgen05 + mma.sync)
    from paper_2501_10375_b200.attention import AttentionStack
    att = AttentionStack(1, d, 32, 8, max_seq=512)
    hp = m.input_hidden(256, stream=6)
    for _ in range(3):
        att.prefill(hp, 0, 0)
elif what == "decode":
    hs = [m.input_hidden(1, stream=9, step=i)[0] for i in range(8)]
    for i in range(8):
        eng.decode(hs[i])
else:
    T = 32768
    h = m.input_hidden(T, stream=5)
    g = int(os.environ.get("DAOP_GROUP", "0"))
    for _ in range(2):
        eng.prefill(h, 0, group_up=g, group_down=g)
torch.cuda.synchronize()
print("done", what)
