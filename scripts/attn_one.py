"""Attention decode: repeated calls with progress output (debug aid, GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_10375_b200.attention import AttentionStack  # noqa: E402

ctx = int(sys.argv[1])
att = AttentionStack(2, 4096, 32, 8, max_seq=ctx + 64, seed=0)
h = torch.randn(4096, device="cuda")
out = torch.empty_like(h)
for i, (layer, pos) in enumerate([(0, ctx + j) for j in range(5)] + [(j % 2, ctx) for j in range(6)]):
    att.decode(h, layer, pos, out=out)
    torch.cuda.synchronize()
    print(i, layer, pos, float(out.abs().sum()), flush=True)
