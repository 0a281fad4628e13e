import sys, statistics, time, threading
sys.path.insert(0, ".")
import torch
import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import ops
from paper_2501_10375_b200.model import MoEModel
import pynvml
pynvml.nvmlInit(); hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
d, ffn, E, k, T = 4096, 14336, 8, 2, 32768
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
h = m.input_hidden(T, stream=5)
r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
pr = ops.permute(r["topk_idx"], E, r["x"])
so = m.slot_of[0]
act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn)
torch.cuda.synchronize()
def up(): ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn)
def down(): ops.expert_gemm_down(act, pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn)
for name, fn in (("up", up), ("down", down)):
    for exp in (0, 1 << 18, (1 << 18) | (5 << 20), 5 << 20, (1 << 18) | (3 << 20)):
        ops.set_gemm_mode(exp)
        for _ in range(3): fn()
        torch.cuda.synchronize(); time.sleep(0.5)
        smp, stop = [], threading.Event()
        def poll():
            while not stop.is_set():
                smp.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000)); time.sleep(0.005)
        th = threading.Thread(target=poll); th.start()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): fn()
        b.record(); torch.cuda.synchronize(); stop.set(); th.join()
        print(name, exp, round(a.elapsed_time(b) / 20, 3), "ms", "sm", statistics.median(x[0] for x in smp), "W", round(statistics.median(x[1] for x in smp)), flush=True)
ops.set_gemm_mode(0)
import ctypes
from paper_2501_10375_b200 import _lib
