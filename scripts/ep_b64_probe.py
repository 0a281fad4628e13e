"""Expert-parallel (PeerEP) batched decode step, b = 64, Mixtral-8x22B shape,
one GPU: launch list for ncu (development aid; bench.py `ep.decode_b64` is the
measurement)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.ep import PeerEP, ep_model  # noqa: E402

m = ep_model(P.ModelShape(2, 8, 2), 6144, 16384, 0, 1, seed=0)
h = m.input_hidden(64, stream=300)
ctx = PeerEP(m, 0, 64, 0, 1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    ctx.layer(h)
torch.cuda.synchronize()
print("done")
