"""DAOP slow tier (host CPU expert FFN in libdaop_b200.so) vs the oracle.
Runs on CPU in the build container (no GPU involved)."""

import numpy as np

from paper_2501_10375_b200 import _lib
from oracle import numerics as N
from oracle import rng as R


import pytest


@pytest.mark.parametrize("n", [1, 3, 16, 37, 64])
def test_host_expert_ffn_matches_oracle(n):
    """n < 16: AVX-512 BF16 GEMV path; n >= 16: AMX-BF16 tiles when the host
    has them (token blocks of 16, ragged tail zero-padded)."""
    d, ffn = 256, 512
    om = N.OracleModel(2, 4, 2, d, ffn, seed=7)
    w1, w3, w2 = om.w1(1, 2), om.w3(1, 2), om.w2(1, 2)
    to_bits = lambda a: np.ascontiguousarray(R.f32_to_bf16_bits(a))  # noqa: E731
    b1, b3, b2 = to_bits(w1), to_bits(w3), to_bits(w2)
    x = R.round_bf16(np.random.default_rng(0).normal(size=(n, d)).astype(np.float32))
    xb = to_bits(x)
    y = np.empty((n, d), dtype=np.float32)
    _lib.call("daop_host_expert_ffn", xb.ctypes.data, n, b1.ctypes.data, b3.ctypes.data,
              b2.ctypes.data, d, ffn, y.ctypes.data, 0, 4)
    ref = N.expert_ffn(x, w1, w3, w2)
    rms = float(np.sqrt(np.mean(ref ** 2)))
    assert np.abs(y - ref).max() <= 2e-3 * rms + 1e-3 * np.abs(ref).max()
    act = np.zeros((n, ffn), dtype=np.uint16)
    y2 = np.empty((n, d), dtype=np.float32)
    _lib.call("daop_host_expert_ffn", xb.ctypes.data, n, b1.ctypes.data, b3.ctypes.data,
              b2.ctypes.data, d, ffn, y2.ctypes.data, act.ctypes.data, 4)
    assert np.array_equal(y, y2)  # deterministic
    a_ref = N.expert_act(x, w1, w3)
    a = R.bf16_bits_to_f32(act)
    assert np.all(np.abs(a - a_ref) <= np.abs(a_ref) * 2 ** -7 + 1e-3 * np.abs(a_ref).max())


def test_host_caps_reports():
    a = np.zeros(1, dtype=np.int32)
    t = np.zeros(1, dtype=np.int32)
    _lib.call("daop_host_caps", a.ctypes.data, t.ctypes.data)
    assert t[0] >= 1


@pytest.mark.parametrize("n", [1, 5, 16, 40])
@pytest.mark.parametrize("threads", [1, 3, 7])
def test_chunked_schedule_is_bit_identical(n, threads):
    """Rows claimed in chunks (default) vs one contiguous share per worker:
    every output row is computed by one worker in a fixed order either way,
    so the results are bit-identical for any thread count."""
    d, ffn = 256, 1024
    rng = np.random.default_rng(n * 10 + threads)
    mk = lambda *s: np.ascontiguousarray(  # noqa: E731
        R.f32_to_bf16_bits(rng.uniform(-0.06, 0.06, size=s).astype(np.float32)))
    b1, b3, b2, xb = mk(ffn, d), mk(ffn, d), mk(d, ffn), mk(n, d)
    out = []
    for grain in ((0, 0), (32, 16), (3, 5)):
        _lib.call("daop_host_set_grain", *grain)
        y = np.empty((n, d), dtype=np.float32)
        _lib.call("daop_host_expert_ffn", xb.ctypes.data, n, b1.ctypes.data, b3.ctypes.data,
                  b2.ctypes.data, d, ffn, y.ctypes.data, 0, threads)
        out.append(y)
    _lib.call("daop_host_set_grain", 32, 16)
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[0], out[2])


@pytest.mark.parametrize("r0", [0, 128, 384])
def test_host_expert_rows_sum_to_the_expert(r0):
    """daop_host_expert_ffn_rows (the host's share of a slow expert split with
    the GPU, daop.SlowSplit): rows [0, r0) + rows [r0, ffn) == the whole
    expert within the fp32 reassociation of the down sums; rows [0, ffn) vs
    the oracle."""
    d, ffn = 256, 512
    om = N.OracleModel(2, 4, 2, d, ffn, seed=11)
    w1, w3, w2 = om.w1(0, 1), om.w3(0, 1), om.w2(0, 1)
    to_bits = lambda a: np.ascontiguousarray(R.f32_to_bf16_bits(a))  # noqa: E731
    b1, b3, b2 = to_bits(w1), to_bits(w3), to_bits(w2)
    x = R.round_bf16(np.random.default_rng(r0).normal(size=(1, d)).astype(np.float32))
    xb = to_bits(x)
    ref = N.expert_ffn(x, w1, w3, w2)
    tol = 2e-3 * float(np.sqrt(np.mean(ref ** 2))) + 1e-3 * np.abs(ref).max()

    def rows(a, b):
        y = np.empty((1, d), dtype=np.float32)
        _lib.call("daop_host_expert_ffn_rows", xb.ctypes.data, 1, b1.ctypes.data,
                  b3.ctypes.data, b2.ctypes.data, d, ffn, a, b, y.ctypes.data, 3)
        return y

    y = rows(r0, ffn) + (rows(0, r0) if r0 else 0)
    assert np.abs(y - ref).max() <= tol
    with pytest.raises(Exception):
        rows(0, ffn + 1)
