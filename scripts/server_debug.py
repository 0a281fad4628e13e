"""Debug: decode server vs launch-per-call host path, per step: which rows
differ (grouped by the CTA that owns them: rows_per_cta = ceil(d / 148)) and
whether the differing values equal the previous step's output (stale)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2501_10375_b200 as P
from paper_2501_10375_b200.engine import MoEBlockEngine
from paper_2501_10375_b200.model import MoEModel
d, ffn = int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 14336
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
m = MoEModel(P.ModelShape(2, 8, 2), d, ffn, seed=2, resident_layers=[0])
eng = MoEBlockEngine(m)
hs = [m.input_hidden(1, stream=70, step=i)[0].cpu().contiguous() for i in range(n)]
ref = []
for h in hs:
    out, sel = eng.decode_host(h)
    ref.append((out.clone(), sel.clone()))
srv_out = []
with eng.decode_server() as srv:
    for i, h in enumerate(hs):
        out, sel = srv.step(h)
        srv_out.append((out.clone(), sel.clone()))
rpc = (d + 147) // 148
bad = 0
for i in range(n):
    diff = (srv_out[i][0] != ref[i][0]).nonzero().flatten()
    if len(diff) == 0:
        continue
    bad += 1
    ctas = sorted(set((diff // rpc).tolist()))
    prev = ref[i - 1][0] if i else None
    stale = int((srv_out[i][0][diff] == prev[diff]).sum()) if prev is not None else -1
    print(f"step {i}: {len(diff)} rows differ in {len(ctas)} CTAs {ctas[:20]}; "
          f"sel {srv_out[i][1].tolist()} vs {ref[i][1].tolist()}; equal to prev step: {stale}")
print(f"{bad}/{n} steps differ")
