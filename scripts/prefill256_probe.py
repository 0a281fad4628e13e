"""Per-op CUDA-event timing of one 256-token prompt layer (Mixtral-8x7B MoE
block + attention), steady state (development aid)."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import ops
from paper_2501_10375_b200.attention import AttentionStack
from paper_2501_10375_b200.model import MoEModel

T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
d, ffn, E, k = 4096, 14336, 8, 2
m = MoEModel(P.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
att = AttentionStack(1, d, 32, 8, max_seq=T + 16)
h = m.input_hidden(T, stream=7)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}


def t(name, fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    res[name] = round(statistics.median(ts), 1)
    return out


t("attention_prefill", lambda: att.prefill(h, 0, 0))
r = t("router", lambda: ops.router(h, m.norm[0], m.gate[0], m.gate[1], k))
pr = t("permute+gather", lambda: ops.permute(r["topk_idx"], E, r["x"]))
so = m.slot_of[0]
act = t("up_skinny", lambda: ops.expert_gemm_up_skinny(pr["x_perm"], pr["offsets"], so, m.slab,
                                                        m.n_slots, m.slot_elems, d, ffn))
y = t("down_skinny", lambda: ops.expert_gemm_down_skinny(act, pr["offsets"], so, m.slab,
                                                          m.n_slots, m.slot_elems, d, ffn))
t("combine", lambda: ops.combine(h, y, pr["inv"], r["topk_w"]))
for nt in (32, 48, 64, 80, 96, 128):
    t(f"up_skinny_nt{nt}", lambda: ops.expert_gemm_up_skinny(pr["x_perm"], pr["offsets"], so, m.slab,
                                                              m.n_slots, m.slot_elems, d, ffn, nt))
    t(f"down_skinny_nt{nt}", lambda: ops.expert_gemm_down_skinny(act, pr["offsets"], so, m.slab,
                                                                  m.n_slots, m.slot_elems, d, ffn,
                                                                  nt))
t("up_pair", lambda: ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, m.slab, m.n_slots,
                                        m.slot_elems, d, ffn))
t("down_pair", lambda: ops.expert_gemm_down(act, pr["offsets"], so, m.slab, m.n_slots,
                                            m.slot_elems, d, ffn))
off = pr["offsets"].tolist()
print("rows per expert", [off[i + 1] - off[i] for i in range(E)])
print(res, "moe sum (router..combine)", round(sum(res[x] for x in ("router", "permute+gather", "up_skinny", "down_skinny", "combine")), 1))
# attention sub-ops
from paper_2501_10375_b200 import _lib
xa = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
t("attn_norm_rows", lambda: _lib.call("daop_attn_norm_rows", h.data_ptr(), T, att.norm[0].data_ptr(), d,
                                      float(ops.RMS_EPS), xa.data_ptr(), ops._s()))
qkv = t("attn_qkv_gemm", lambda: ops.gemm_bf16_f32(xa, att.wqkv[0]))
o = torch.empty((T, att.q_dim), dtype=torch.bfloat16, device="cuda")
t("attn_core", lambda: _lib.call("daop_attn_prefill", qkv.data_ptr(), T, 0, att.k_cache[0].data_ptr(),
                                 att.v_cache[0].data_ptr(), 32, 8, att.max_seq, float(att.theta),
                                 o.data_ptr(), ops._s()))
t("attn_o_gemm", lambda: ops.gemm_bf16_f32(o, att.wo[0], resid=h))
t("attn_qkv_gemm_splitk", lambda: ops.gemm_bf16_f32(xa, att.wqkv[0], ws=True))
t("attn_o_gemm_splitk", lambda: ops.gemm_bf16_f32(o, att.wo[0], resid=h, ws=True))
print({k: v for k, v in res.items() if k.startswith("attn")})
