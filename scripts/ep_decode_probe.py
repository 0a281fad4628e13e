import sys, time
import torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import ops, _lib
from paper_2501_10375_b200.ep import PeerEPDecode, ep_model
d, ffn, E, K = 6144, 16384, 8, 2
m = ep_model(P.ModelShape(2, E, K), d, ffn, 0, 1, seed=0)
dec = PeerEPDecode(m, 0, 1)
hs = [m.input_hidden(1, stream=400, step=i)[0] for i in range(32)]
def timeit(fn, n=200):
    for i in range(5): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for i in range(n): fn(i)
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3, (t1 - t0) / n * 1e6
def dec_only(i):
    ops.decode_layer(hs[i % 32], m.norm[0], m.gate[0], m.gate[1], m.fast[0], m.slot_of[0], m.slab, m.slot_elems, d, ffn, K, dec.bufs)
print("decode only (gpu us, host us)", timeit(dec_only))
def dec_share(i):
    dec_only(i); dec.epoch += 1
    _lib.call("daop_ep_decode_share", dec.peers.data_ptr(), 0, 1, K, d, dec.bufs.y.data_ptr(), dec.bufs.is_fast.data_ptr(), dec.epoch, ops._s())
print("decode+share", timeit(dec_share))
print("full layer", timeit(lambda i: dec.layer(hs[i % 32])))
print("fused decode kernel only", timeit(lambda i: dec.stream(hs[i % 32])))
def fin(i):
    dec.finish()
dec.stream(hs[0])
print("finish only", timeit(fin))
