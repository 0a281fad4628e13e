"""Where the end-to-end decode call spends its time (development aid, GPU box)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200.engine import MoEBlockEngine
from paper_2501_10375_b200.model import MoEModel
d, ffn = 4096, 14336
m = MoEModel(P.ModelShape(2, 8, 2), d, ffn, seed=0, resident_layers=[0])
eng = MoEBlockEngine(m)
hh = torch.empty(d, dtype=torch.float32, pin_memory=True)
hh.copy_(m.input_hidden(1, stream=9)[0].cpu())
for _ in range(20):
    eng.decode_host(hh)
def wall(fn, n=500):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e6
from paper_2501_10375_b200 import _lib
for spin in (1, 0, 1):
    _lib.call("daop_graph_step_mode", spin)
    print(f"decode_host (graph, spin={spin}) us/step", wall(lambda: eng.decode_host(hh)))
_lib.call("daop_graph_step_mode", 0)
st = torch.cuda.current_stream().cuda_stream
ex = eng._host_graphs[0][1]
hs = eng._h_host.data_ptr()
print("raw daop_graph_step us/step", wall(lambda: _lib.LIB.daop_graph_step(ex, st, hs, hs, 0)))
g = eng._graphs_keepalive[0]
def replay_sync():
    g.replay(); torch.cuda.current_stream().synchronize()
print("graph replay + sync us", wall(replay_sync))
# copies only
hd = torch.empty(d, device="cuda"); ho = torch.empty(d + 4, device="cuda")
oh = torch.empty(d + 4, pin_memory=True)
g2 = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    hd.copy_(hh, non_blocking=True); oh.copy_(ho, non_blocking=True)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
with torch.cuda.graph(g2):
    hd.copy_(hh, non_blocking=True); oh.copy_(ho, non_blocking=True)
def copies():
    g2.replay(); torch.cuda.current_stream().synchronize()
print("graph H2D+D2H only + sync us", wall(copies))
def kern_only():
    eng.decode(eng._h_dev, 0); torch.cuda.current_stream().synchronize()
print("decode launch + sync (no graph, no copies) us", wall(kern_only))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200): eng.decode(eng._h_dev, 0)
e1.record(); torch.cuda.synchronize(); print("kernel back-to-back us", e0.elapsed_time(e1) / 200 * 1e3)

# launch + sync floor: an empty graph-captured kernel
z = torch.zeros(1, device="cuda")
g3 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    z.add_(1)
torch.cuda.synchronize()
with torch.cuda.graph(g3):
    z.add_(1)
def empty():
    g3.replay(); torch.cuda.current_stream().synchronize()
print("empty graph replay + sync us", wall(empty))

# persistent decode server: no launch, no stream sync per call
# (no torch.cuda.synchronize() while it is open: the server kernel only ends
# when closed or idle)
with eng.decode_server() as srv:
    for _ in range(20):
        srv.step(hh)
    t = time.perf_counter()
    for _ in range(1000):
        srv.step(hh)
    print("decode server us/step", (time.perf_counter() - t) / 1000 * 1e6)

# where the server's per-call time goes (GPU globaltimer stamps)
tr = torch.zeros((1200, 4), dtype=torch.int64, device="cuda")
_lib.call("daop_server_trace", tr.data_ptr(), 1200)
with eng.decode_server() as srv:
    for _ in range(1100):
        srv.step(hh)
_lib.call("daop_server_trace", 0, 0)
torch.cuda.synchronize()
t = tr[100:1100].cpu().double()
import numpy as np
seen, rel, done = t[:, 0], t[:, 1], t[:, 2]
print("server: doorbell->released %.2f us, released->body done %.2f us, call period %.2f us" % (
    float((rel - seen).median()) / 1e3, float((done - rel).median()) / 1e3,
    float((seen[1:] - seen[:-1]).median()) / 1e3))
