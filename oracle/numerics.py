"""Oracle (TEST INFRASTRUCTURE ONLY): numpy fp32 restatement of the MoE block.

The reference executes no numerics ("Combination weights at the MoE output
are not simulated numerically"; "No numerical execution of
experts"), so this module is PARITY UNPINNED by any reference
vector: it restates the builder-defined contract of DESIGN.md §3 (SURVEY.md
Appendix B), which follows PAPER.md:110-114 (gate on the post-attention
hidden state), PAPER.md:234,319,329 (next-layer prediction from x_l) and the
Mixtral top-2 renormalisation.

Contract (per layer l, residual h fp32 (T, d)):
    x      = bf16( (h * rsqrt(mean(h^2) + eps)) * gamma_l )
    z      = x . Wg_l^T          (fp32 accumulate)       p  = softmax(z)
    z_hat  = x . Wg_{l+1}^T      (l + 1 < L)             p^ = softmax(z_hat)
    sel    = topk(p, k)          (ties -> lower index; decisions.topk_rows)
    w_j    = p[sel_j] / sum_j p[sel_j]
    a      = bf16( silu(x . W1_e^T) * (x . W3_e^T) )      (fp32 accumulate)
    y_e    = a . W2_e^T                                   (fp32 accumulate)
    h'     = h + sum_{j=0..k-1} w_j y_{sel_j}             (fixed j order)
"""

from __future__ import annotations

import numpy as np

from . import rng
from .decisions import topk_rows

RMS_EPS = 1e-5


# ------------------------------------------------------------------ weights


class OracleModel:
    """Lazily generated random-init weights (bit-identical to the CUDA init)."""

    def __init__(self, num_layers, num_experts, top_k, d_model, d_ff, seed=0):
        self.L, self.E, self.k = num_layers, num_experts, top_k
        self.d, self.ffn, self.seed = d_model, d_ff, seed
        self.scale_in = float(np.float32(1.0 / np.sqrt(d_model)))
        self.scale_ff = float(np.float32(1.0 / np.sqrt(d_ff)))

    def gate(self, layer):
        return rng.tensor_bf16(self.seed, rng.make_tag(rng.KIND_GATE, layer),
                               (self.E, self.d), self.scale_in)

    def norm(self, layer):
        return rng.norm_weight(self.seed, layer, self.d)

    def w1(self, layer, e):
        return rng.tensor_bf16(self.seed, rng.make_tag(rng.KIND_EXPERT, layer, e, 0),
                               (self.ffn, self.d), self.scale_in)

    def w3(self, layer, e):
        return rng.tensor_bf16(self.seed, rng.make_tag(rng.KIND_EXPERT, layer, e, 1),
                               (self.ffn, self.d), self.scale_in)

    def w2(self, layer, e):
        return rng.tensor_bf16(self.seed, rng.make_tag(rng.KIND_EXPERT, layer, e, 2),
                               (self.d, self.ffn), self.scale_ff)


def input_hidden(seed: int, stream: int, step: int, t: int, d: int) -> np.ndarray:
    """Synthetic residual-stream input h (T, d) fp32, unit variance U(-√3, √3)."""
    tag = rng.make_tag(rng.KIND_INPUT, stream, step)
    return rng.tensor_f32(seed, tag, (t, d), float(np.float32(np.sqrt(3.0))))


# ------------------------------------------------------------------ blocks


def rmsnorm(h: np.ndarray, gamma: np.ndarray) -> np.ndarray:
    h = h.astype(np.float32)
    ms = (h.astype(np.float64) ** 2).mean(axis=-1, keepdims=True).astype(np.float32)
    r = np.float32(1.0) / np.sqrt(ms + np.float32(RMS_EPS))
    return rng.round_bf16((h * r) * gamma.astype(np.float32))


def softmax(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.float32)
    m = z.max(axis=-1, keepdims=True)
    ez = np.exp(z - m)
    return ez / ez.sum(axis=-1, keepdims=True)


def router(x, wg_true, wg_pred=None):
    """Fused-router contract: probs of the own gate and of the next layer's gate
    from ONE read of x."""
    p = softmax(x.astype(np.float32) @ wg_true.T.astype(np.float32))
    ph = None
    if wg_pred is not None:
        ph = softmax(x.astype(np.float32) @ wg_pred.T.astype(np.float32))
    return p, ph


def renorm_weights(p_rows: np.ndarray, sel: np.ndarray) -> np.ndarray:
    g = np.take_along_axis(p_rows, sel, axis=1).astype(np.float32)
    return g / g.sum(axis=1, keepdims=True)


def silu(a: np.ndarray) -> np.ndarray:
    return a / (np.float32(1.0) + np.exp(-a))


def expert_act(x, w1, w3):
    """a = bf16(silu(x W1^T) * (x W3^T)) -- the SwiGLU intermediate."""
    g = x.astype(np.float32) @ w1.T
    u = x.astype(np.float32) @ w3.T
    return rng.round_bf16(silu(g) * u)


def expert_ffn(x, w1, w3, w2):
    return expert_act(x, w1, w3) @ w2.T


def permutation(topk_idx: np.ndarray, num_experts: int):
    """Stable token->expert permutation by histogram + exclusive scan.

    Rows (t, j) sorted by (expert, t, j).  Returns (offsets (E+1,), perm
    (T*k,) flat source index t*k+j for each sorted position, inv (T, k)
    sorted position of each (t, j)).
    """
    t, k = topk_idx.shape
    flat = topk_idx.reshape(-1).astype(np.int64)
    hist = np.bincount(flat, minlength=num_experts)
    offsets = np.zeros(num_experts + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(hist)
    perm = np.argsort(flat, kind="stable").astype(np.int64)
    inv = np.empty(t * k, dtype=np.int64)
    inv[perm] = np.arange(t * k)
    return offsets, perm, inv.reshape(t, k)


def combine(h, y_sorted, inv, w):
    """h' = h + sum_j w_j y[inv[t, j]] in fixed j order."""
    out = h.astype(np.float32).copy()
    for j in range(inv.shape[1]):
        out = out + w[:, j:j + 1] * y_sorted[inv[:, j]]
    return out


def moe_layer(model: OracleModel, layer: int, h: np.ndarray, sel=None, w=None,
              x=None):
    """One MoE block on all tokens with every expert exact on current input.

    sel / w may be injected (teacher forcing with the GPU's decisions);
    x may be injected (teacher forcing with the GPU's normalised input).
    Returns dict(x, p, p_hat, sel, w, out).
    """
    if x is None:
        x = rmsnorm(h, model.norm(layer))
    wg_pred = model.gate(layer + 1) if layer + 1 < model.L else None
    p, ph = router(x, model.gate(layer), wg_pred)
    if sel is None:
        sel = topk_rows(p.astype(np.float64), model.k)
    if w is None:
        w = renorm_weights(p, sel)
    offsets, perm, inv = permutation(sel, model.E)
    y = np.zeros((sel.size, model.d), dtype=np.float32)
    for e in range(model.E):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if a == b:
            continue
        rows = perm[a:b] // model.k
        y[a:b] = expert_ffn(x[rows], model.w1(layer, e), model.w3(layer, e),
                            model.w2(layer, e))
    out = combine(h, y, inv, w)
    return {"x": x, "p": p, "p_hat": ph, "sel": sel, "w": w, "out": out}


def daop_decode_token(model: OracleModel, h: np.ndarray, sel_per_layer, start: int,
                      weights_from_pred: bool = True, engine: str = "daop", pre=None):
    """One decode token through all layers with the engine's decisions injected
    (teacher forcing).  Below `start` (or for fiddler) picks run on the current
    x_l with true-gate weights; from `start` on (daop) weights come from the
    prediction carried on layer l-1 and slow picks -- flagged by the caller --
    use the stale x_{l-1} (policies.py:325-330).

    sel_per_layer: list of (experts, slow_flags) per layer; pre(h, l) (optional)
    is the non-MoE block applied before layer l's MoE block.  Returns h'."""
    h = h.astype(np.float32)[None, :]
    x_prev, ph_prev = None, None
    for l in range(model.L):
        if pre is not None:
            h = pre(h[0], l)[None, :].astype(np.float32)
        x = rmsnorm(h, model.norm(l))
        wg_next = model.gate(l + 1) if l + 1 < model.L else None
        p, ph = router(x, model.gate(l), wg_next)
        experts, slow = sel_per_layer[l]
        plan_l = engine == "daop" and l >= start
        src = ph_prev if (plan_l and weights_from_pred) else p
        g = src[0, experts].astype(np.float32)
        w = g / g.sum()
        out = h.copy()
        for j, e in enumerate(experts):
            xin = x_prev if (plan_l and slow[j]) else x
            out = out + w[j] * expert_ffn(xin, model.w1(l, e), model.w3(l, e), model.w2(l, e))
        h, x_prev, ph_prev = out, x, ph
    return h[0]


# ------------------------------------------------------------------ non-MoE block (attention)
# Builder-defined restatement of csrc/attention.cu (the reference prices this
# block as t_nonmoe, moesim/simulator.py:291).  Parity is
# within tolerance (fp32 reductions in a different order).

KIND_ATTN = 5
NORM_LAYER_OFFSET = 4096
HEAD_DIM = 128


class OracleAttention:
    def __init__(self, d, n_heads=32, n_kv=8, theta=1e6, seed=0):
        self.d, self.n_heads, self.n_kv, self.theta, self.seed = d, n_heads, n_kv, theta, seed
        self.q_dim, self.kv_dim = n_heads * HEAD_DIM, n_kv * HEAD_DIM
        self.s_in = float(np.float32(1.0 / np.sqrt(d)))
        self.s_o = float(np.float32(1.0 / np.sqrt(self.q_dim)))

    def norm(self, layer):
        return rng.norm_weight(self.seed, layer + NORM_LAYER_OFFSET, self.d)

    def _cached(self, key, make):
        cache = self.__dict__.setdefault("_cache", {})
        if key not in cache:
            cache[key] = make()
        return cache[key]

    def wqkv(self, layer):  # generated once per layer (token-by-token oracle runs)
        return self._cached(("qkv", layer), lambda: rng.tensor_bf16(
            self.seed, rng.make_tag(KIND_ATTN, layer, 0, 0),
            (self.q_dim + 2 * self.kv_dim, self.d), self.s_in))

    def wo(self, layer):
        return self._cached(("o", layer), lambda: rng.tensor_bf16(
            self.seed, rng.make_tag(KIND_ATTN, layer, 0, 1), (self.d, self.q_dim), self.s_o))


def rope(x: np.ndarray, pos: int, theta: float) -> np.ndarray:
    """Rotate-half RoPE of (..., 128) fp32 vectors at position pos."""
    half = HEAD_DIM // 2
    i = np.arange(half, dtype=np.float32)
    inv = (np.float32(1.0) / np.power(np.float32(theta), (2 * i) / np.float32(HEAD_DIM))).astype(np.float32)
    ang = (np.float32(pos) * inv).astype(np.float32)
    c, s = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
    a, b = x[..., :half], x[..., half:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1).astype(np.float32)


def attention_decode(att: OracleAttention, layer: int, h: np.ndarray, pos: int,
                     k_cache: np.ndarray, v_cache: np.ndarray):
    """One decode token; k_cache / v_cache (n_kv, >= pos+1, 128) float32 views
    of the bf16 cache (entries < pos used as given; pos is written here).
    Returns (h_out, xa, k_cache, v_cache)."""
    xa = rmsnorm(h[None, :], att.norm(layer))[0]
    w64 = att._cached(("qkv64", layer), lambda: att.wqkv(layer).astype(np.float64))
    qkv = (w64 @ xa.astype(np.float64)).astype(np.float32)
    q = qkv[: att.q_dim].reshape(att.n_heads, HEAD_DIM)
    k = qkv[att.q_dim: att.q_dim + att.kv_dim].reshape(att.n_kv, HEAD_DIM)
    v = qkv[att.q_dim + att.kv_dim:].reshape(att.n_kv, HEAD_DIM)
    q = rope(q, pos, att.theta)
    k = rope(k, pos, att.theta)
    k_cache = k_cache.copy()
    v_cache = v_cache.copy()
    k_cache[:, pos] = rng.round_bf16(k)
    v_cache[:, pos] = rng.round_bf16(v)
    group = att.n_heads // att.n_kv
    o = np.zeros((att.n_heads, HEAD_DIM), dtype=np.float64)
    for hd in range(att.n_heads):
        g = hd // group
        sc = (k_cache[g, : pos + 1].astype(np.float64) @ q[hd].astype(np.float64)) / np.sqrt(HEAD_DIM)
        p = np.exp(sc - sc.max())
        p /= p.sum()
        o[hd] = p @ v_cache[g, : pos + 1].astype(np.float64)
    o_b = rng.round_bf16(o.reshape(-1).astype(np.float32))
    wo64 = att._cached(("o64", layer), lambda: att.wo(layer).astype(np.float64))
    y = (wo64 @ o_b.astype(np.float64)).astype(np.float32)
    return h.astype(np.float32) + y, xa, k_cache, v_cache
