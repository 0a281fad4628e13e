"""Do the prefill GEMMs' persisting-L2 settings slow the HBM-bound prefill
kernels (router, permutation + gather, combine) that follow them?  Times them
alone before any GEMM, after one up GEMM, and after resetting the persisting
lines (development aid, GPU box)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

d, ffn, E, k, T = 4096, 14336, 8, 2, 32768
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
h = m.input_hidden(T, stream=5)
hist = torch.zeros((8, E), dtype=torch.int32, device="cuda")
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k, hist=hist, tokens_per_seq=4096,
               hist_seq_stride=E)
pr = ops.permute(r["topk_idx"], E, r["x"])
y = torch.randn(pr["x_perm"].shape[0], d, device="cuda")
fns = (("router+hist", lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], k, hist=hist,
                                           tokens_per_seq=4096, hist_seq_stride=E)),
       ("router", lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)),
       ("permute+gather", lambda: ops.permute(r["topk_idx"], E, r["x"])),
       ("combine", lambda: ops.combine(h, y, pr["inv"], r["topk_w"])))


def run(tag):
    res = {}
    for n, fn in fns:
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[n] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    print(f"{tag:42s}", res, flush=True)


from paper_2501_10375_b200 import _lib  # noqa: E402

run("before any GEMM")
_lib.call("daop_set_gemm_mode", 1 << 11)  # persisting set-aside ON (tuning bit)
ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab, m.n_slots, m.slot_elems, d,
                   ffn)
torch.cuda.synchronize()
run("after one up GEMM, set-aside on")
_lib.call("daop_set_gemm_mode", 0)  # default: set-aside off (the next GEMM resets it to 0)
ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab, m.n_slots, m.slot_elems, d,
                   ffn)
torch.cuda.synchronize()
run("after an up GEMM with the set-aside at 0")
