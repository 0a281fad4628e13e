"""Router at decode-batch sizes (T = 16 / 64 / 128), 20 launches replayed
as one CUDA graph: the CTA-per-token kernel vs the bulk-copy router forced
to small T (daop_set_router_mode bit 3).  Development aid, GPU box."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import _lib, ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

for d in (4096, 6144):
    m = MoEModel(P.ModelShape(2, 8, 2), d, 512, seed=0, resident_layers=[])
    for T in (16, 64, 128):
        h = m.input_hidden(T, stream=5)
        res = {}
        for mode in (1, 1 | 8):
            _lib.call("daop_set_router_mode", mode)

            def fn():
                return ops.router(h, m.norm[0], m.gate[0], m.gate[1], 2)
            for _ in range(5):
                fn()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            res["small" if mode == 1 else "bulk"] = round(a.elapsed_time(b) / 20 * 1e3, 1)
        print(d, T, res, flush=True)
_lib.call("daop_set_router_mode", 1)
