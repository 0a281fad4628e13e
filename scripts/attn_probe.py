"""Attention decode kernels on the Mixtral-8x7B shape (development aid, GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_10375_b200.attention import AttentionStack  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
att = AttentionStack(2, 4096, 32, 8, max_seq=ctx + 64, seed=0)
h = torch.randn(4096, device="cuda")
out = torch.empty_like(h)
for i in range(5):
    att.decode(h, 0, ctx + i, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 200
b = att.bytes_per_token_layer(ctx + 1)
for graph in (False, True):
    if graph:  # launch-cost free: the layers back to back in one graph
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(20):
                att.decode(h, i % 2, ctx, out=out)
        g.replay()
        torch.cuda.synchronize()
    e0.record()
    if graph:
        for _ in range(n // 20):
            g.replay()
    else:
        for i in range(n):
            att.decode(h, i % 2, ctx, out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(f"attention decode layer at ctx {ctx} ({'graph' if graph else 'eager'}): {us:.1f} us, "
          f"{b / us / 1e3:.0f} GB/s")
