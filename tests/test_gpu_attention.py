"""Non-MoE block (attention with a KV cache, decode b = 1) vs the oracle
restatement (oracle/numerics.py attention_decode), teacher-forced on the
GPU's own cache contents; tolerance as for the hidden states."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import numerics as N  # noqa: E402
from oracle import rng as R  # noqa: E402


def bf16_f32(t):
    return R.bf16_bits_to_f32(t.view(torch.int16).cpu().numpy().view(np.uint16))


def close(got, ref, tag):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    rms = float(np.sqrt(np.mean(ref ** 2)))
    err = np.abs(got - ref)
    bound = 2e-3 * rms + 1e-3 * np.abs(ref)
    assert (err <= bound).all(), f"{tag}: max |d| {err.max():.3e} (rms {rms:.3e})"


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as pkg
    from paper_2501_10375_b200 import attention
    return pkg, attention


@pytest.mark.parametrize("d,heads,kv,positions", [
    (1024, 8, 2, [0, 1, 2, 3]),          # first tokens: one tile, one split
    (1024, 8, 2, [700, 1601]),           # several tiles and splits, ragged tail
    (4096, 32, 8, [0, 1, 333]),          # Mixtral-8x7B attention shape
])
def test_attention_decode_parity(P, d, heads, kv, positions):
    pkg, A = P
    att = A.AttentionStack(2, d, heads, kv, max_seq=2048, seed=3)
    oatt = N.OracleAttention(d, heads, kv, theta=att.theta, seed=3)
    # earlier positions: random cache contents (teacher forcing of the history)
    g = torch.Generator(device="cuda").manual_seed(1)
    att.k_cache[1].copy_(torch.randn(att.k_cache[1].shape, generator=g, device="cuda"))
    att.v_cache[1].copy_(torch.randn(att.v_cache[1].shape, generator=g, device="cuda"))
    for step, pos in enumerate(positions):
        h = torch.empty(d, dtype=torch.float32, device="cuda")
        A.ops.fill_uniform_f32(h, 3, (4 << 56) | (9 << 32) | step, float(np.float32(np.sqrt(3))))
        kc = bf16_f32(att.k_cache[1])
        vc = bf16_f32(att.v_cache[1])
        out = att.decode(h, 1, pos)
        torch.cuda.synchronize()
        ref, xa, kc2, vc2 = N.attention_decode(oatt, 1, h.cpu().numpy(), pos, kc, vc)
        x = bf16_f32(att.xa)
        assert (np.abs(x - xa) <= np.abs(xa) * 2 ** -7 + 1e-30).all()
        # the appended k (after RoPE) and v: within one bf16 ulp
        kn, vn = bf16_f32(att.k_cache[1][:, pos]), bf16_f32(att.v_cache[1][:, pos])
        assert np.all(np.abs(kn - kc2[:, pos]) <= np.abs(kc2[:, pos]) * 2 ** -7 + 1e-6)
        assert np.all(np.abs(vn - vc2[:, pos]) <= np.abs(vc2[:, pos]) * 2 ** -7 + 1e-6)
        close(out.cpu().numpy(), ref, f"pos {pos}")
        # layer 0's cache is untouched
        assert att.k_cache[0].abs().sum().item() == 0


def test_attention_bad_position(P):
    pkg, A = P
    att = A.AttentionStack(1, 1024, 8, 2, max_seq=64, seed=3)
    h = torch.zeros(1024, device="cuda")
    with pytest.raises(pkg.errors.DeviceError):
        att.decode(h, 0, 64)


@pytest.mark.parametrize("d,heads,kv,pos0,T", [
    (1024, 8, 2, 0, 5),          # a fresh prompt inside one tile
    (1024, 8, 2, 70, 130),       # history + a prompt spanning several tiles
    (4096, 32, 8, 0, 64),        # Mixtral-8x7B attention shape
    (4096, 32, 8, 0, 256),       # configs[2]'s 256-token prompt: 4 K/V tiles, 16 token tiles
    (1024, 8, 1, 3, 37),         # MQA-style group 8, ragged token tile
])
def test_attention_prefill_parity(P, d, heads, kv, pos0, T):
    """Batched causal prefill (tcgen05 projections, tensor-core flash
    attention with bf16 q / P operands) vs the oracle run position by
    position, and vs the decode kernels run token by token: outputs within
    the hidden-state bar, cache rows within one bf16 ulp (the GEMM's
    summation order differs)."""
    pkg, A = P
    att = A.AttentionStack(2, d, heads, kv, max_seq=512, seed=5)
    dec = A.AttentionStack(2, d, heads, kv, max_seq=512, seed=5)
    oatt = N.OracleAttention(d, heads, kv, theta=att.theta, seed=5)
    g = torch.Generator(device="cuda").manual_seed(2)
    hist_k = torch.randn(att.k_cache[1].shape, generator=g, device="cuda")
    hist_v = torch.randn(att.v_cache[1].shape, generator=g, device="cuda")
    for a in (att, dec):  # the same history before pos0, nothing after
        a.k_cache[1].copy_(hist_k)
        a.v_cache[1].copy_(hist_v)
        a.k_cache[1][:, pos0:].zero_()
        a.v_cache[1][:, pos0:].zero_()
    h = torch.empty((T, d), dtype=torch.float32, device="cuda")
    A.ops.fill_uniform_f32(h, 5, (4 << 56) | (11 << 32), float(np.float32(np.sqrt(3))))
    kc, vc = bf16_f32(att.k_cache[1]), bf16_f32(att.v_cache[1])
    out = att.prefill(h, 1, pos0)
    ref_dec = torch.stack([dec.decode(h[t], 1, pos0 + t) for t in range(T)])
    torch.cuda.synchronize()
    hn = h.cpu().numpy()
    for t in range(T):
        ref, _, kc, vc = N.attention_decode(oatt, 1, hn[t], pos0 + t, kc, vc)
        close(out[t].cpu().numpy(), ref, f"token {t} vs oracle")
    close(out.cpu().numpy(), ref_dec.cpu().numpy(), "prefill vs decode path")
    span = slice(pos0, pos0 + T)
    for mine, want in ((att.k_cache[1], kc), (att.v_cache[1], vc)):
        m = bf16_f32(mine)[:, span]
        w = want[:, span]
        assert np.all(np.abs(m - w) <= np.abs(w) * 2 ** -7 + 1e-3 * np.abs(w).max())
    assert att.k_cache[0].abs().sum().item() == 0  # layer 0 untouched


def test_attention_prefill_bounds(P):
    pkg, A = P
    att = A.AttentionStack(1, 1024, 8, 2, max_seq=64, seed=3)
    h = torch.zeros((10, 1024), device="cuda")
    with pytest.raises(pkg.ShapeMismatchError):
        att.prefill(h, 0, 60)


@pytest.mark.parametrize("pair", [False, True])  # M <= 768: skinny (default) or forced CTA-pair
@pytest.mark.parametrize("M,K,N,resid", [(1, 512, 256, False), (5, 512, 1024, True),
                                         (256, 4096, 6144, False), (700, 4096, 4096, True),
                                         (1100, 1024, 512, True)])
def test_dense_gemm_parity(P, M, K, N, resid, pair):
    """daop_gemm_bf16_f32 (the prompt attention's projections on the tcgen05
    pipeline: the swap-AB skinny kernel for prompt-sized M, the CTA-pair
    kernel above) vs a float64 numpy product of the same bf16 operands."""
    pkg, A = P
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    a = torch.randn((M, K), generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.rand((N, K), generator=g, device="cuda") - 0.5).to(torch.bfloat16)
    r = torch.randn((M, N), generator=g, device="cuda") if resid else None
    A.ops.set_gemm_mode(1 << 15 if pair else 0)
    try:
        out = A.ops.gemm_bf16_f32(a, w, resid=r)
    finally:
        A.ops.set_gemm_mode(0)
    ref = a.double().cpu().numpy() @ w.double().cpu().numpy().T
    if resid:
        ref = ref + r.double().cpu().numpy()
        # in place: the residual buffer receives the result
        r2 = r.clone()
        A.ops.set_gemm_mode(1 << 15 if pair else 0)
        try:
            A.ops.gemm_bf16_f32(a, w, resid=r2, out=r2)
        finally:
            A.ops.set_gemm_mode(0)
        assert torch.equal(r2, out)
    torch.cuda.synchronize()
    close(out.cpu().numpy(), ref, f"gemm {M}x{K}x{N}")


def test_decode_token_with_attention_l2_prefetch_is_bit_identical(P):
    """The next layer's attention weights prefetched into L2 during the MoE
    kernel (daop_l2_prefetch) is a cache hint: bit-identical results."""
    pkg, A = P
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.model import MoEModel
    L, d = 3, 1024
    m = MoEModel(pkg.ModelShape(L, 8, 2), d, 1024, seed=2)
    outs = []
    for pf in (False, True):
        att = A.AttentionStack(L, d, 8, 2, max_seq=64, seed=2)
        eng = MoEBlockEngine(m)
        eng.attn_prefetch = pf
        h = m.input_hidden(1, stream=3)[0]
        for pos in range(3):
            h = eng.decode_token(h, start=1, attn=att, pos=pos).clone()
        outs.append(h)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("M,K,N,resid", [(256, 4096, 6144, False), (256, 4096, 4096, True),
                                         (100, 1024, 512, True), (37, 4096, 256, False),
                                         (300, 1024, 512, True)])  # > 256 rows: no split
def test_dense_gemm_splitk_parity(P, M, K, N, resid):
    """daop_gemm_bf16_f32_ws (split-K over idle SM pairs + fixed-order
    reduction) vs a float64 product; deterministic, and in place on resid."""
    pkg, A = P
    ops = A.ops
    g = torch.Generator(device="cuda").manual_seed(3 * M + K + N)
    a = torch.randn((M, K), generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.rand((N, K), generator=g, device="cuda") - 0.5).to(torch.bfloat16)
    r = torch.randn((M, N), generator=g, device="cuda") if resid else None
    parts = ops.splitk_parts(M, K, N)
    assert (parts > 1) == (M <= 256 and N // 256 <= 37)
    out = ops.gemm_bf16_f32(a, w, resid=r, ws=True)
    again = ops.gemm_bf16_f32(a, w, resid=r, ws=True)
    assert torch.equal(out, again)
    ref = a.double().cpu().numpy() @ w.double().cpu().numpy().T
    if resid:
        ref = ref + r.double().cpu().numpy()
        r2 = r.clone()
        ops.gemm_bf16_f32(a, w, resid=r2, out=r2, ws=True)
        assert torch.equal(r2, out)
    torch.cuda.synchronize()
    close(out.cpu().numpy(), ref, f"split-K gemm {M}x{K}x{N}")


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("kv,positions", [(8, [0, 5, 511, 1601, 2047]), (4, [63, 64, 900])])
def test_fused_core_oproj_equals_two_launches(P, kv, positions, mode):
    """The attention core + O projection as one cooperative launch (modes 1,
    2; off by default: measured slower) is bit-identical to the two-launch path, including more split tasks than
    SMs (kv 8 at position 1601: 208 tasks) and back-to-back calls (the
    kernel's head / exit counters reset themselves)."""
    pkg, A = P
    from paper_2501_10375_b200 import _lib
    d, heads = 4096, 32
    outs = {}
    for fused in (0, mode):
        _lib.call("daop_set_attn_fused", fused)
        att = A.AttentionStack(1, d, heads, kv, max_seq=2048, seed=5)
        g = torch.Generator(device="cuda").manual_seed(2)
        att.k_cache[0].copy_(torch.randn(att.k_cache[0].shape, generator=g, device="cuda"))
        att.v_cache[0].copy_(torch.randn(att.v_cache[0].shape, generator=g, device="cuda"))
        res = []
        for step, pos in enumerate(positions):
            h = torch.empty(d, dtype=torch.float32, device="cuda")
            A.ops.fill_uniform_f32(h, 5, (4 << 56) | (7 << 32) | step, float(np.float32(np.sqrt(3))))
            res.append(att.decode(h, 0, pos).clone())
        torch.cuda.synchronize()
        outs[fused] = (res, att.k_cache.clone(), att.v_cache.clone())
    _lib.call("daop_set_attn_fused", 0)
    for a, b in zip(outs[0][0], outs[mode][0]):
        assert torch.equal(a, b)
    assert torch.equal(outs[0][1], outs[mode][1]) and torch.equal(outs[0][2], outs[mode][2])


def test_decoder_token_early_plan_launch_is_bit_identical(P):
    """Full decoder layers (attention + MoE, DAOP plans from layer 2): the
    PLAN-mode MoE kernels launched early behind the attention O-proj (weight
    stream started before griddepcontrol.wait, variant bit 8) give the same
    residual and cache as the plain launches, token after token."""
    pkg, A = P
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.model import MoEModel
    L, d, ffn = 4, 1024, 2048
    outs = {}
    for early in (False, True):
        m = MoEModel(pkg.ModelShape(L, 8, 2), d, ffn, seed=4)
        eng = MoEBlockEngine(m)
        eng.decode_early = early
        att = A.AttentionStack(L, d, 8, 2, max_seq=64, seed=4)
        res = []
        for t in range(5):
            h = m.input_hidden(1, stream=11, step=t)[0]
            res.append(eng.decode_token(h, start=2, daop=True, attn=att, pos=t).clone())
        torch.cuda.synchronize()
        outs[early] = (res, att.k_cache.clone())
    for a, b in zip(outs[False][0], outs[True][0]):
        assert torch.equal(a, b)
    assert torch.equal(outs[False][1], outs[True][1])
