"""Batched decode through one Mixtral-8x7B MoE layer: step time by batch,
eager launches and one CUDA graph per step (development aid, GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.engine import MoEBlockEngine  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

d, ffn, E, k = 4096, 14336, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
eng = MoEBlockEngine(m)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sizes = [int(a) for a in sys.argv[1:]] or [1, 8, 16, 32, 64, 128, 256]
for b in sizes:
    h = m.input_hidden(b, stream=9)
    for _ in range(3):
        r = eng.prefill(h, 0)
    torch.cuda.synchronize()
    act = int((r["offsets"][1:] - r["offsets"][:-1] > 0).sum())
    e0.record()
    for _ in range(20):
        eng.prefill(h, 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eng.prefill(h, 0)
        with torch.cuda.graph(g):
            for _ in range(10):
                eng.prefill(h, 0)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    gms = e0.elapsed_time(e1) / 40
    by = act * 3 * d * ffn * 2
    print(f"b={b:4d} active experts {act}: eager {ms*1e3:7.1f} us, graph {gms*1e3:7.1f} us "
          f"{b/gms*1e3:9.0f} tok/s  weights {by/gms/1e6:5.0f} GB/s", flush=True)
