"""Grouped-GEMM tuning sweep (development aid; bench.py is the contract).

    python scripts/gemm_sweep.py time   # CUDA-event timing, 6 back-to-back calls per config
    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
        -k regex:grouped_gemm python scripts/gemm_sweep.py once   # one call per config

Configs: (which, policy, group).  policy per csrc/grouped_gemm.cu GemmParams.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import model as M, ops  # noqa: E402

UP = [(pol, g) for pol in (0, 4, 5, 6) for g in (32, 64, 128)]
DOWN = [(pol, g) for pol in (2, 3, 4, 5) for g in (-4, -8, -16)]

mode = sys.argv[1] if len(sys.argv) > 1 else "time"
d, ffn, E, k, T = 4096, 14336, 8, 2, 32768
m = M.MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
h = m.input_hidden(T, stream=5)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
pr = ops.permute(r["topk_idx"], E, r["x"])
so = m.slot_of[0]
act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn)


def up(g):
    return ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots, m.slot_elems,
                              d, ffn, g)


def down(g):
    return ops.expert_gemm_down(act, pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn,
                                g)


def timed(fn, iters):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


fl_up, fl_dn = 2 * T * k * d * 2 * ffn, 2 * T * k * d * ffn
passes = 1 if mode == "once" else 2
for which, cfgs, fn, fl in (("up", UP, up, fl_up), ("down", DOWN, down, fl_dn)):
    for pol, g in [c for i in range(passes) for c in (cfgs if i == 0 else cfgs[::-1])]:
        ops.set_gemm_mode(pol << 4)
        if mode == "once":
            fn(g)
            torch.cuda.synchronize()
            print(which, pol, g, flush=True)
        else:
            ms = timed(lambda: fn(g), 6)
            print(f"{which:5s} policy={pol} group={g:4d} {ms:7.3f} ms {fl / ms / 1e9:6.0f} TF/s",
                  flush=True)
ops.set_gemm_mode(0)
