import sys, torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200.engine import MoEBlockEngine
from paper_2501_10375_b200.model import MoEModel
d, ffn, E, k = 4096, 14336, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
eng = MoEBlockEngine(m)
for b in (1, 8, 16, 32, 64, 128, 256):
    h = m.input_hidden(b, stream=9)
    for _ in range(3): r = eng.prefill(h, 0)
    torch.cuda.synchronize()
    act = int((r["offsets"][1:] - r["offsets"][:-1] > 0).sum())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): eng.prefill(h, 0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    by = act * 3 * d * ffn * 2
    print(f"b={b:4d} active experts {act}: {ms*1e3:8.1f} us  {b/ms*1e3:9.0f} tok/s  weights {by/ms/1e9:6.0f} GB/s", flush=True)
