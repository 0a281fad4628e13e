import sys, time, torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200.ep import PeerEP, ep_model
m = ep_model(P.ModelShape(2, 8, 2), 6144, 16384, 0, 1, seed=0)
h = m.input_hidden(64, stream=300)
ctx = PeerEP(m, 0, 64, 0, 1)
for _ in range(10): ctx.layer(h)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); a.record()
for _ in range(50): ctx.layer(h)
b.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("gpu ms/step", a.elapsed_time(b) / 50, "host submit ms/step", (t1 - t0) / 50 * 1e3, "wall", (t2 - t0) / 50 * 1e3)
