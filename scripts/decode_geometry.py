"""Decode-kernel ring geometry sweep on a given shape (development aid, GPU box).

    python scripts/decode_geometry.py d ffn variant...
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

d, ffn = int(sys.argv[1]), int(sys.argv[2])
variants = [int(v) for v in sys.argv[3:]] or [0]
E, k = 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
bufs = ops.DecodeBuffers(d, ffn, E, k, "cuda")
hs = [m.input_hidden(1, stream=9, step=i)[0] for i in range(16)]
nbytes = 2 * 3 * d * ffn * 2 + 2 * E * d * 2
for v in variants:
    try:
        for i in range(5):
            ops.decode_layer(hs[i], m.norm[0], m.gate[0], m.gate[1], m.fast[0], m.slot_of[0],
                             m.slab, m.slot_elems, d, ffn, k, bufs, variant=v)
        torch.cuda.synchronize()
        ref = bufs.h_out.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 300
        e0.record()
        for i in range(n):
            ops.decode_layer(hs[i % 16], m.norm[0], m.gate[0], m.gate[1], m.fast[0],
                             m.slot_of[0], m.slab, m.slot_elems, d, ffn, k, bufs, variant=v)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        print(f"variant {v:2d}: {us:7.1f} us  {nbytes / us / 1e3:7.1f} GB/s", flush=True)
    except Exception as exc:  # unsupported geometry for this shape
        print(f"variant {v:2d}: {exc}", flush=True)
