"""Where a DAOP prefill layer's time goes (T = 256, Mixtral-8x7B shape)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.attention import AttentionStack  # noqa: E402
from paper_2501_10375_b200.daop import DaopEngine  # noqa: E402

L, T = int(sys.argv[1]) if len(sys.argv) > 1 else 8, 256
att = AttentionStack(L, 4096, 32, 8, max_seq=512)
h = torch.randn(T, 4096, device="cuda")
att.prefill(h, 0, 0)
torch.cuda.synchronize()
t0 = time.perf_counter()
for l in range(L):
    att.prefill(h, l, 0)
torch.cuda.synchronize()
print(f"attention prefill: {(time.perf_counter() - t0) / L * 1e3:.3f} ms per layer")
shape = P.ModelShape(L, 8, 2)
for attn in (False, True):
    eng = DaopEngine(shape, 4096, 14336, np.full((L, 8), 0.25), 1.0, P.PolicyConfig("daop"),
                     seed=0, attention=attn, max_seq=512)
    hp = eng.model.input_hidden(T, stream=400)
    first = eng.prefill(hp)
    torch.cuda.synchronize()
    print(f"  first call attention={attn}: {first.ms / L:.3f} ms per layer")
    t0 = time.perf_counter()
    pre = eng.prefill(hp)
    torch.cuda.synchronize()
    print(f"DaopEngine.prefill attention={attn}: {pre.ms / L:.3f} ms per layer "
          f"(wall {(time.perf_counter() - t0) / L * 1e3:.3f})")
    del eng
