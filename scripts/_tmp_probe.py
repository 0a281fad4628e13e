import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import _lib, ops
from paper_2501_10375_b200.model import MoEModel
d, ffn, E, k = 4096, 14336, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
bufs = ops.DecodeBuffers(d, ffn, E, k, "cuda")
hs = [m.input_hidden(1, stream=9, step=i)[0] for i in range(8)]
for i in range(20):
    ops.decode_layer(hs[i % 8], m.norm[0], m.gate[0], m.gate[1], m.fast[0], m.slot_of[0], m.slab, m.slot_elems, d, ffn, k, bufs)
torch.cuda.synchronize()
tlb = np.zeros((148, 16), dtype=np.uint64)
_lib.call("daop_decode_timeline", 2, 0, 0)
torch.cuda.synchronize()
for i in range(3):
    ops.decode_layer(hs[i % 8], m.norm[0], m.gate[0], m.gate[1], m.fast[0], m.slot_of[0], m.slab, m.slot_elems, d, ffn, k, bufs)
torch.cuda.synchronize()
_lib.call("daop_decode_timeline", 0, tlb.ctypes.data, 148)
t = tlb.astype(np.int64)
rel = (t[:, :12] - t[:, :1])
for i, nm in enumerate(["start", "phase0 end", "ph1", "act", "end", "rms", "x+gates", "z summed", "sel+stream", "softmax", "topk", "finish_sel"]):
    print(f"  {nm:10s} median {np.median(rel[:, i]):10.0f} cycles")
