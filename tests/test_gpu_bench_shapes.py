"""Parity at the bench's own shapes (VERDICT r01 "What's weak" #1).

The tensor-bound bench numbers run the grouped tcgen05 GEMMs at
  * BASELINE configs[3]: Mixtral-8x7B, 8 x 4096 = 32,768 tokens (~8K rows per
    expert: the persistent tile schedule / rasterisation of a real prefill);
  * BASELINE configs[4]: Mixtral-8x22B (d 6144, ffn 16384), the `ep` prefill
    and `decode_b64` sections.
The CPU oracle cannot run a whole 32K-token layer in seconds, so each check
samples rows: up to 96 random sorted rows per expert for the SwiGLU
activations and down-projection outputs (teacher-forced on the GPU's bf16
inputs), and a sample of tokens for the layer output (teacher-forced x,
selection and weights).  The routing is checked FREE-RUNNING on every token:
the oracle computes x = RMSNorm(h), p, top-k from h alone; indices must agree
except on rows whose oracle top-(k+1) probabilities are within 1e-5 of each
other (near ties, SPEC.md:184 / moesim/_kernels.py:63-79), and the agreement
rate is asserted >= 99.9 %.

Tolerances: act within one bf16 ulp (+1e-4 rms); y and the
layer output max|d| <= 2e-3 rms(ref) + 1e-3 |ref|.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import decisions as D  # noqa: E402
from oracle import numerics as N  # noqa: E402

NEAR_TIE = 1e-5


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as pkg
    from paper_2501_10375_b200 import model, ops
    return pkg, model, ops


def f32(t):
    return t.float().cpu().numpy()


def hidden_close(got, ref, tag=""):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    rms = float(np.sqrt(np.mean(ref ** 2)))
    err = np.abs(got - ref)
    bound = 2e-3 * rms + 1e-3 * np.abs(ref)
    worst = float((err / np.maximum(bound, 1e-30)).max())
    assert worst <= 1.0, f"{tag}: max |d| {err.max():.3e} exceeds bound (ratio {worst:.2f})"


def free_running_agreement(h, gamma, wg, wg_next, sel_gpu, k):
    """Oracle router from h alone vs the GPU's indices.  Returns (agree,
    n_rows, n_exempt, n_bad): n_bad counts disagreeing rows that are NOT
    near ties (must be 0)."""
    x = N.rmsnorm(h, gamma)
    p, _ = N.router(x, wg, wg_next)
    sel_ref = D.topk_rows(p.astype(np.float64), k)
    srt = -np.sort(-p.astype(np.float64), axis=1)[:, : k + 1]
    gap = np.min(srt[:, :-1] - srt[:, 1:], axis=1)  # smallest gap among the top k+1
    diff = np.any(sel_ref != sel_gpu, axis=1)
    near = gap < NEAR_TIE
    return int((~diff).sum()), len(diff), int((diff & near).sum()), int((diff & ~near).sum())


def _device_weights(m, l, e):
    v = m.expert_views(m.slot(l, e))
    return f32(v[0]), f32(v[1]), f32(v[2])


def _sampled_layer_check(P, m, h, r, pr, act, y, out, k, n_rows=96, n_tok=64, seed=0):
    E, d = m.shape.num_experts, m.d
    rng = np.random.default_rng(seed)
    x = r["x"]
    off = pr["offsets"].cpu().numpy()
    perm = pr["perm"].cpu().numpy()
    # the permutation is exact (integer work) on every row
    off_ref, perm_ref, inv_ref = N.permutation(r["topk_idx"].cpu().numpy(), E)
    assert np.array_equal(off, off_ref) and np.array_equal(perm, perm_ref)
    assert np.array_equal(pr["inv"].cpu().numpy(), inv_ref)
    tok = np.sort(rng.choice(h.shape[0], size=min(n_tok, h.shape[0]), replace=False))
    sel_t = r["topk_idx"].cpu().numpy()[tok].astype(np.int64)
    w_t = r["topk_w"].cpu().numpy()[tok]
    x_t = f32(x[torch.from_numpy(tok).cuda()])
    y_tok = np.zeros((len(tok), k, d), dtype=np.float32)
    for e in range(E):
        a, b = int(off[e]), int(off[e + 1])
        if a == b:
            continue
        w1, w3, w2 = _device_weights(m, 0, e)
        rows = np.sort(rng.choice(np.arange(a, b), size=min(n_rows, b - a), replace=False))
        ri = torch.from_numpy(rows).cuda()
        xp = f32(pr["x_perm"][ri])
        assert np.array_equal(xp, f32(x[torch.from_numpy(perm[rows] // k).cuda()])), e
        a_ref = N.expert_act(xp, w1, w3)
        a_gpu = f32(act[ri])
        dif = np.abs(a_gpu - a_ref)
        rms = float(np.sqrt(np.mean(a_ref.astype(np.float64) ** 2)))
        bound = np.abs(a_ref) * 2.0 ** -7 + 1e-4 * rms
        assert np.all(dif <= bound), f"expert {e} act: >1 ulp frac {(dif > bound).mean():.2e}"
        assert (dif > 0).mean() < 0.02, f"expert {e}: {(dif > 0).mean():.3f} of act differ"
        hidden_close(y[ri].cpu().numpy(), a_gpu @ w2.T, f"expert {e} down rows")
        for i, t in enumerate(tok):  # the sampled tokens' picks of this expert
            for j in range(k):
                if sel_t[i, j] == e:
                    y_tok[i, j] = N.expert_ffn(x_t[i:i + 1], w1, w3, w2)[0]
        del w1, w3, w2
    ref = h.cpu().numpy()[tok].astype(np.float32).copy()
    for j in range(k):
        ref = ref + w_t[:, j:j + 1] * y_tok[:, j]
    hidden_close(out.cpu().numpy()[tok], ref, "layer output (sampled tokens)")


@pytest.mark.parametrize("d,ffn,T,tag", [
    (4096, 14336, 32768, "8x7B configs[3] 8 x 4096 tokens"),
    (6144, 16384, 8192, "8x22B configs[4] 8192 tokens"),
])
def test_prefill_layer_at_bench_shape(P, d, ffn, T, tag):
    pkg, model_mod, ops = P
    E, k = 8, 2
    m = model_mod.MoEModel(pkg.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
    h = m.input_hidden(T, stream=200)
    r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
    pr = ops.permute(r["topk_idx"], E, r["x"])
    slot_of = m.slot_of[0].contiguous()
    act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], slot_of, m.slab, m.n_slots,
                             m.slot_elems, d, ffn)
    y = ops.expert_gemm_down(act, pr["offsets"], slot_of, m.slab, m.n_slots, m.slot_elems, d, ffn)
    out = ops.combine(h, y, pr["inv"], r["topk_w"])
    torch.cuda.synchronize()
    hn = h.cpu().numpy()
    agree, n, exempt, bad = free_running_agreement(hn, f32(m.norm[0]), f32(m.gate[0]),
                                                   f32(m.gate[1]),
                                                   r["topk_idx"].cpu().numpy(), k)
    # RMSNorm is bit-compatible with the oracle (fp64 squares, IEEE f32 scale):
    # the bf16 x rows equal the CPU path's, so routing agrees free-running
    x_ref = N.rmsnorm(hn, f32(m.norm[0]))
    x_bad = int((f32(r["x"]) != x_ref).sum())
    print(f"{tag}: free-running routing agreement {agree}/{n} ({agree / n:.5%}), "
          f"{exempt} near-tie rows exempt; x elements differing from the oracle: {x_bad}")
    assert x_bad <= 1e-6 * x_ref.size
    assert bad == 0, f"{bad} rows disagree without a near tie"
    assert agree / n >= 0.999
    # the production path the bench times (MoEBlockEngine.prefill) is the same ops
    from paper_2501_10375_b200.engine import MoEBlockEngine
    rb = MoEBlockEngine(m).prefill(h, 0)
    torch.cuda.synchronize()
    assert torch.equal(rb["out"], out)
    _sampled_layer_check(P, m, h, r, pr, act, y, out, k)


def test_skinny_b64_at_8x22b_shape(P):
    """decode_b64 of the `ep` section: 64 tokens through the skinny GEMMs at
    the Mixtral-8x22B shape, every row checked against the oracle."""
    pkg, model_mod, ops = P
    d, ffn, E, k, T = 6144, 16384, 8, 2, 64
    m = model_mod.MoEModel(pkg.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
    h = m.input_hidden(T, stream=500)
    r = ops.router(h, m.norm[0], m.gate[0], m.gate[1], k)
    pr = ops.permute(r["topk_idx"], E, r["x"])
    slot_of = m.slot_of[0].contiguous()
    act = ops.expert_gemm_up_skinny(pr["x_perm"], pr["offsets"], slot_of, m.slab, m.n_slots,
                                    m.slot_elems, d, ffn)
    y = ops.expert_gemm_down_skinny(act, pr["offsets"], slot_of, m.slab, m.n_slots,
                                    m.slot_elems, d, ffn)
    out = ops.combine(h, y, pr["inv"], r["topk_w"])
    torch.cuda.synchronize()
    _sampled_layer_check(P, m, h, r, pr, act, y, out, k, n_rows=128, n_tok=64)


@pytest.mark.parametrize("G", [2, 8])
def test_peer_ep_emulated_at_8x22b_vs_oracle(P, G):
    """PeerEP (emulated G ranks on one GPU) at the Mixtral-8x22B shape: each
    rank's output equals the single-GPU layer bit for bit AND its sampled
    tokens match the CPU oracle directly (not only transitively)."""
    pkg, model_mod, ops = P
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.ep import PeerEP, ep_model
    d, ffn, E, k = 6144, 16384, 8, 2
    t_rank = 1024
    m = model_mod.MoEModel(pkg.ModelShape(2, E, k), d, ffn, seed=0, resident_layers=[0])
    eng = MoEBlockEngine(m)
    models = [ep_model(pkg.ModelShape(2, E, k), d, ffn, r, G, seed=0) for r in range(G)]
    ranks = PeerEP.emulated(models, 0, t_cap=t_rank)
    hs = [m.input_hidden(t_rank - 37 * r, stream=600 + r) for r in range(G)]
    for r in range(G):
        ranks[r].route(hs[r])
    for r in range(G):
        ranks[r].publish()
    for r in range(G):
        ranks[r].dispatch()
    for r in range(G):
        ranks[r].experts()
    outs = [ranks[r].finish() for r in range(G)]
    torch.cuda.synchronize()
    rng = np.random.default_rng(G)
    xs = {}
    for r in range(G):
        ranks[r].check()
        ref = eng.prefill(hs[r], 0)
        assert torch.equal(outs[r][1], ref["topk_idx"])
        assert torch.equal(outs[r][0], ref["out"]), r
        xs[r] = ref["x"]
    # direct oracle check of rank 0 and the last rank: routing free-running on
    # every token, expert outputs on sampled tokens (teacher-forced bf16 x)
    for r in (0, G - 1):
        hn_all = hs[r].cpu().numpy()
        agree, n, exempt, bad = free_running_agreement(
            hn_all, f32(m.norm[0]), f32(m.gate[0]), f32(m.gate[1]), outs[r][1].cpu().numpy(), k)
        assert bad == 0 and agree / n >= 0.999, (agree, n, exempt, bad)
        tok = np.sort(rng.choice(hs[r].shape[0], size=16, replace=False))
        hn = hn_all[tok]
        x = f32(xs[r][torch.from_numpy(tok).cuda()])
        sel = outs[r][1].cpu().numpy()[tok].astype(np.int64)
        w = outs[r][2].cpu().numpy()[tok]
        ys = np.zeros((len(tok), k, d), dtype=np.float32)
        for e in sorted(set(sel.reshape(-1).tolist())):
            w1, w3, w2 = _device_weights(m, 0, e)
            for i in range(len(tok)):
                for j in range(k):
                    if sel[i, j] == e:
                        ys[i, j] = N.expert_ffn(x[i:i + 1], w1, w3, w2)[0]
        refo = hn.astype(np.float32).copy()
        for j in range(k):
            refo = refo + w[:, j:j + 1] * ys[:, j]
        hidden_close(outs[r][0].cpu().numpy()[tok], refo, f"EP G={G} rank {r} vs oracle")
    for c in ranks:
        c.close()
