"""The CPU baseline's variants (oracle/baseline.py) agree with the numpy
oracle: the plain-C bf16 expert (oracle/cpu_moe.c) and torch-CPU bf16 give
the same selection and hidden states within the hidden-state tolerance."""

import numpy as np

from oracle import numerics as N
from oracle.baseline import CpuMoELayer


def _close(got, ref, tag):
    rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2)))
    err = np.abs(got.astype(np.float64) - ref)
    assert (err <= 2e-3 * rms + 1e-3 * np.abs(ref)).all(), f"{tag}: {err.max():.3e}"


def test_cpu_variants_match_numpy_oracle():
    layer = CpuMoELayer(2, 8, 2, 512, 1024, seed=4, with_bf16=True)
    h = N.input_hidden(4, 1, 0, 48, 512)
    ref = layer.prefill(h)
    _close(layer.prefill_c(h), ref, "C prefill")
    _close(layer.prefill_bf16(h), ref, "torch bf16 prefill")
    for t in range(3):
        o, s = layer.decode_step(h[t])
        oc, sc = layer.decode_step_c(h[t])
        ob, sb = layer.decode_step_bf16(h[t])
        assert s.tolist() == sc.tolist() == sb.tolist()
        _close(oc, o, "C decode")
        _close(ob, o, "torch bf16 decode")
    assert layer.c_threads() >= 1
