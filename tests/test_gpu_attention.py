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
