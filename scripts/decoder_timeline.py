"""Where a full decoder layer's decode time goes (Mixtral-8x7B, ctx 512):
global-timer spans of the last layer's QKV GEMV, attention core, O-proj and
MoE decode kernel (per-CTA stamps, daop_attn_timeline / daop_decode_timeline),
relative to the previous layer's MoE end (development aid, GPU box)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import _lib  # noqa: E402
from paper_2501_10375_b200.attention import AttentionStack  # noqa: E402
from paper_2501_10375_b200.engine import MoEBlockEngine  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402

L, D, CTX = 6, 4096, 512
m = MoEModel(P.ModelShape(L, 8, 2), D, 14336, seed=0)
eng = MoEBlockEngine(m)
att = AttentionStack(L, D, 32, 8, max_seq=CTX + 64, seed=0)
h = m.input_hidden(1, stream=3)[0]
for i in range(3):
    eng.decode_token(h.clone(), start=4, daop=True, attn=att, pos=CTX + i)
torch.cuda.synchronize()
for rep in range(3):
    _lib.call("daop_attn_timeline", 1, 0)
    _lib.call("daop_decode_timeline", 1, 0, 0)
    eng.decode_token(h.clone(), start=4, daop=True, attn=att, pos=CTX + 5)
    torch.cuda.synchronize()
    at = np.zeros((3, 256, 2), dtype=np.uint64)
    _lib.call("daop_attn_timeline", 0, at.ctypes.data)
    dt = np.zeros((1024, 16), dtype=np.uint64)
    _lib.call("daop_decode_timeline", 0, dt.ctypes.data, 1024)
    spans = {}
    for k, name in enumerate(("qkv", "core", "oproj")):
        st, en = at[k, :, 0], at[k, :, 1]
        ok = st > 0
        spans[name] = (int(st[ok].min()), int(en[en > 0].max()))
    ms, me = dt[:, 12], dt[:, 13]
    spans["moe"] = (int(ms[ms > 0].min()), int(me[me > 0].max()))
    # the QKV kernel starts (PDL) during the previous MoE kernel and waits for it
    t0 = spans["qkv"][0]
    print(f"rep {rep}: last decoder layer (us from QKV start):",
          {k: (round((a - t0) / 1e3, 2), round((b - t0) / 1e3, 2)) for k, (a, b) in spans.items()},
          flush=True)
