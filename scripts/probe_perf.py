"""Quick kernel timing probe (development aid; bench.py is the contract)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import model as M, ops

def ev_time(fn, iters=50, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

what = sys.argv[1] if len(sys.argv) > 1 else "all"
d, ffn, E, k = 4096, 14336, 8, 2
if what in ("decode", "all"):
    m = M.MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
    bufs = ops.DecodeBuffers(d, ffn, E, k, "cuda")
    hs = [m.input_hidden(1, stream=9, step=i)[0] for i in range(16)]
    it = [0]
    var = [0]
    mode = [0]
    pp = torch.softmax(torch.randn(E, device="cuda"), 0)
    def step():
        ops.decode_layer(hs[it[0] % 16], m.norm[0], m.gate[0], m.gate[1], m.fast[0], m.slot_of[0],
                         m.slab, m.slot_elems, d, ffn, k, bufs, variant=var[0],
                         mode=mode[0], pred_prev=pp if mode[0] else None,
                         weights_from_pred=bool(mode[0]))
        it[0] += 1
    from paper_2501_10375_b200 import _lib
    for v, md in ((0, 0), (0, 1), (9, 1)):
        var[0] = v
        mode[0] = md
        try:
            ms = ev_time(step, iters=200, warm=10)
        except Exception as exc:  # noqa: BLE001
            print(f"decode_layer variant={v}: {exc}", flush=True)
            continue
        b = 704_774_144
        tlb = np.zeros((148, 16), dtype=np.uint64)
        _lib.call("daop_decode_timeline", 1, 0, 0)
        torch.cuda.synchronize(); step(); torch.cuda.synchronize()
        _lib.call("daop_decode_timeline", 0, tlb.ctypes.data, 148)
        t = tlb.astype(np.int64)
        rel = (t - t[:, :1]) / 1.9e3   # SM cycles relative to each CTA's start, ~us at 1.9 GHz
        ph = {nm: np.median(rel[:, i]) for i, nm in ((1, "ph0"), (2, "ph1"), (3, "act"), (4, "end"))}
        print(f"decode_layer mode={md} variant={v}: {ms*1e3:.1f} us  {b/ms/1e6:.1f} GB/s  phase ends (us, median CTA): "
              + " ".join(f"{k} {x:.1f}" for k, x in ph.items()) + f"  max end {rel[:, 4].max():.1f}",
              flush=True)
if what in ("prefill", "all"):
    from paper_2501_10375_b200.engine import MoEBlockEngine
    T = 32768
    m = M.MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
    eng = MoEBlockEngine(m)
    h = m.input_hidden(T, stream=5)
    r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
    pr = ops.permute(r["topk_idx"], E, r["x"])
    so = m.slot_of[0]
    act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn)
    y = ops.expert_gemm_down(act, pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn)
    st = {
        "router": lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], k),
        "permute+gather": lambda: ops.permute(r["topk_idx"], E, r["x"]),
        "gemm up": lambda: ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn),
        "gemm down": lambda: ops.expert_gemm_down(act, pr["offsets"], so, m.slab, m.n_slots, m.slot_elems, d, ffn),
        "combine": lambda: ops.combine(h, y, pr["inv"], r["topk_w"]),
        "prefill layer": lambda: eng.prefill(h, 0),
    }
    for name, fn in st.items():
        print(f"{name:16s} {ev_time(fn, 10, 3):8.3f} ms", flush=True)
