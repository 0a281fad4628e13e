"""Expert-parallel (PeerEP) prefill layer, Mixtral-8x22B shape, 32K tokens,
one GPU: launch sequence for an ncu launch list (development aid; bench.py
`ep` is the measurement)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.ep import PeerEP, ep_model  # noqa: E402

m = ep_model(P.ModelShape(2, 8, 2), 6144, 16384, 0, 1, seed=0)
h = m.input_hidden(32768, stream=300)
ctx = PeerEP(m, 0, 32768, 0, 1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    ctx.layer(h)
torch.cuda.synchronize()
print("done")
