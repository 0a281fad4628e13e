"""Per-die tile schedule of the prefill GEMMs (daop_set_gemm_die_table) vs the
plain schedule: candidate SM -> die tables, bit-identity of act / y, time per
launch (development aid, GPU box).

    python scripts/gemm_die_probe.py [iters]      # iters = 0: one launch per config (ncu)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import _lib, ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cands = sys.argv[2].split(",") if len(sys.argv) > 2 else ["off", "auto", "off", "auto"]
# optional rasterisation groups: "up1/up2/..,down1/down2/.." (0 = library default)
groups = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "0"]
ups = [int(g) for g in groups[0].split("/")]
downs = [int(g) for g in groups[1].split("/")]
d, ffn, E, k, T = 4096, 14336, 8, 2, 32768
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
h = m.input_hidden(T, stream=5)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
pr = ops.permute(r["topk_idx"], E, r["x"])
n = torch.cuda.get_device_properties(0).multi_processor_count
sm = np.arange(n)
tables = {"half": (sm >= n // 2), "tpcalt": ((sm >> 1) & 1) == 1, "quarter": ((sm >> 2) & 1) == 1,
          "gpc18": ((sm // 18) & 1) == 1}


def set_table(c):
    if c == "off":
        _lib.call("daop_set_gemm_die_table", 0, 0)
    elif c == "auto":
        _lib.call("daop_set_gemm_die_table", 0, -1)
    else:
        t = tables[c].astype(np.int32)
        _lib.call("daop_set_gemm_die_table", t.ctypes.data, len(t))


def up(g=0):
    return ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab, m.n_slots,
                              m.slot_elems, d, ffn, g)


def down(a, g=0):
    return ops.expert_gemm_down(a, pr["offsets"], m.slot_of[0], m.slab, m.n_slots,
                                m.slot_elems, d, ffn, g)


set_table("off")
a_ref = up()
y_ref = down(a_ref)
torch.cuda.synchronize()
for c in cands:
    set_table(c)
    for gu, gd in zip(ups, downs):
        a = up(gu)
        y = down(a_ref, gd)
        torch.cuda.synchronize()
        same = torch.equal(a, a_ref) and torch.equal(y, y_ref)
        tag = f"{c:8s} groups {gu:4d} {gd:4d}"
        if iters == 0:
            print(f"{tag} bit-identical {same}", flush=True)
            continue
        res = []
        for fn in (lambda: up(gu), lambda: down(a_ref, gd)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fn()
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / iters)
        print(f"{tag} up {res[0]:7.3f} ms  down {res[1]:7.3f} ms  bit-identical {same}", flush=True)
set_table("off")
