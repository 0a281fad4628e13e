"""Sustained grouped-GEMM sweep (development aid, run on the GPU box):
L2 policy x rasterisation group for the up / down GEMMs of one
Mixtral-8x7B prefill layer (8 x 4096 tokens), each config timed over N
back-to-back launches with CUDA events while NVML samples the SM clock.

    python scripts/gemm_power_sweep.py [N] [configs...]   config = which:policy:group
"""
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
CONFIGS = sys.argv[2:] or ["up:0:64", "up:4:64", "up:5:64", "down:2:-8", "down:4:-8",
                           "down:3:-8", "down:4:-4", "down:6:-8"]
d, ffn, E, k = 4096, 14336, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
T = 32768
h = m.input_hidden(T, stream=5)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
pr = ops.permute(r["topk_idx"], E, r["x"])
act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab, m.n_slots,
                         m.slot_elems, d, ffn)
torch.cuda.synchronize()

import pynvml  # noqa: E402
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)


def clocks(stop, out):
    while not stop.is_set():
        out.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
        time.sleep(0.005)


from paper_2501_10375_b200.engine import MoEBlockEngine  # noqa: E402
eng = MoEBlockEngine(m)

# cuBLAS reference on the same per-expert shapes (bf16 out, no SwiGLU)
off = pr["offsets"].tolist()
xs = [pr["x_perm"][off[e]:off[e + 1]] for e in range(E)]
acts = [act[off[e]:off[e + 1]] for e in range(E)]
w13 = [m.slab[m.slot(0, e)][: 2 * ffn * d].view(2 * ffn, d) for e in range(E)]
w2 = [m.slab[m.slot(0, e)][2 * ffn * d:].view(d, ffn) for e in range(E)]

for cfg in CONFIGS:
    which, pol, grp = cfg.split(":")[:3]
    extra = int(cfg.split(":")[3]) if cfg.count(":") >= 3 else 0  # demote | persist-off bits
    ops.set_gemm_mode((int(pol) << 4) | (extra << 8))
    grp = int(grp)

    def run():
        if which == "cublas_up":
            for e in range(E):
                torch.matmul(xs[e], w13[e].t())
        elif which == "cublas_down":
            for e in range(E):
                torch.matmul(acts[e], w2[e].t())
        elif which == "prefill":  # the whole layer through the engine, default groups
            eng.prefill(h, 0)
        elif which == "prefill_sep":  # the same layer with the separate combine pass
            rr = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
            pp = ops.permute(rr["topk_idx"], E, rr["x"])  # dense: materialised x_perm
            aa = ops.expert_gemm_up(pp["x_perm"], pp["offsets"], m.slot_of[0], m.slab,
                                    m.n_slots, m.slot_elems, d, ffn)
            yy = ops.expert_gemm_down(aa, pp["offsets"], m.slot_of[0], m.slab, m.n_slots,
                                      m.slot_elems, d, ffn)
            ops.combine(h, yy, pp["inv"], rr["topk_w"])
        elif which == "up":
            ops.expert_gemm_up(pr["x_perm"], pr["offsets"], m.slot_of[0], m.slab, m.n_slots,
                               m.slot_elems, d, ffn, grp)
        else:
            ops.expert_gemm_down(act, pr["offsets"], m.slot_of[0], m.slab, m.n_slots,
                                 m.slot_elems, d, ffn, grp)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    time.sleep(1.0)  # let the clock recover between configs
    samples, stop = [], threading.Event()
    th = threading.Thread(target=clocks, args=(stop, samples))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N):
        run()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / N
    fl = 2.0 * T * k * d * ffn * (2 if which.endswith("up") else 3 if which.startswith("prefill")
                                  else 1)
    print(f"{cfg:12s} {ms:7.3f} ms  {fl / ms / 1e9:7.1f} TF/s  sm {statistics.median(samples):.0f} MHz",
          flush=True)
ops.set_gemm_mode(0)
