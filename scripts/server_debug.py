"""Debug: decode server vs launch-per-call host path vs device path, per step."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2501_10375_b200 as P
from paper_2501_10375_b200.engine import MoEBlockEngine
from paper_2501_10375_b200.model import MoEModel
d, ffn = int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 14336
m = MoEModel(P.ModelShape(2, 8, 2), d, ffn, seed=2, resident_layers=[0])
eng = MoEBlockEngine(m)
hs = [m.input_hidden(1, stream=70, step=i)[0].cpu().contiguous() for i in range(6)]
dev = []
for h in hs:
    b = eng.decode(h.cuda())
    dev.append((b.h_out.clone(), b.sel.clone()))
ref = []
for h in hs:
    out, sel = eng.decode_host(h)
    ref.append((out.clone(), sel.clone()))
ref2 = []
for h in hs:
    out, sel = eng.decode_host(h)
    ref2.append((out.clone(), sel.clone()))
srv_out = []
with eng.decode_server() as srv:
    for i, h in enumerate(hs):
        out, sel = srv.step(h)
        srv_out.append((out.clone(), sel.clone()))
for i in range(6):
    a = dev[i][0].cpu()
    print(i, "sel dev/host/host2/srv", dev[i][1].tolist(), ref[i][1].tolist(), ref2[i][1].tolist(),
          srv_out[i][1].tolist(),
          "max|host-dev|", (ref[i][0] - a).abs().max().item(),
          "max|host2-host|", (ref2[i][0] - ref[i][0]).abs().max().item(),
          "max|srv-host|", (srv_out[i][0] - ref[i][0]).abs().max().item(),
          "n diff srv", int((srv_out[i][0] != ref[i][0]).sum()))
