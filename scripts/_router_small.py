import sys, statistics
sys.path.insert(0, ".")
import torch
import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import ops, _lib
from paper_2501_10375_b200.model import MoEModel
for d in (4096, 6144):
    m = MoEModel(P.ModelShape(2, 8, 2), d, 512, seed=0, resident_layers=[])
    for T in (16, 64, 128):
        h = m.input_hidden(T, stream=5)
        res = {}
        for mode in (1, 1 | 8):
            _lib.call("daop_set_router_mode", mode)
            fn = lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], 2)
            for _ in range(5): fn()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20): fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record(); torch.cuda.synchronize()
            res[mode] = round(a.elapsed_time(b) / 20 * 1e3, 1)
        print(d, T, res, flush=True)
_lib.call("daop_set_router_mode", 1)
