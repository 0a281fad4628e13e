"""Generate golden moesim JSONL trace files with the UNMODIFIED reference.

Build container only (the reference is not on the GPU box):

    python tests/golden/make_trace_golden.py

Imports ``moesim`` from /root/reference/pkg/src (read-only; numba's cache goes
to /tmp, no bytecode written) and writes, with moesim's own ``save_trace``
(moesim/trace.py:332-362), the traces under ``tests/golden/traces/``.  The
tests require our ``save_trace`` to reproduce these files byte for byte and
our ``load_trace`` to read them back to the same arrays.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from moesim import (GeneratorConfig, ModelShape, RoutingTrace, generate_trace,  # noqa: E402
                    save_trace)

OUT = Path(__file__).with_name("traces")


def main():
    OUT.mkdir(exist_ok=True)
    traces = {}
    # full-precision thirds (tests/test_trace.py:163-175)
    third = 1.0 / 3.0
    traces["third"] = RoutingTrace(ModelShape(1, 2, 1), "p", np.array([[[third, 1.0 - third]]]),
                                   np.zeros((0, 1, 2)))
    # exponent formats, denormals, exact 0 / 1, negative zero, a quote in the id
    e = np.array([[[1.0, -0.0, 0.0, 0.0], [1 - 1e-7, 5e-324, 1e-7, 1e-300]],
                  [[0.25, 0.25, 0.25, 0.25], [0.5, 0.125, 0.125, 0.25]]])
    dp = np.array([[[0.1, 0.2, 0.3, 0.4], [0, 0, 0, 0]]])
    traces["edge"] = RoutingTrace(ModelShape(2, 4, 2), 'edge "q"/\\', e, e[:1], decode_predicted=dp,
                                  decode_mask=np.array([[True, False]]))
    # random rows with prefill predictions
    rng = np.random.default_rng(7)
    raw = rng.random((3, 3, 6)) + 1e-3
    pt = raw / raw.sum(axis=2, keepdims=True)
    raw = rng.random((3, 3, 6)) + 1e-3
    pp = raw / raw.sum(axis=2, keepdims=True)
    pp[:, 2] = 0
    pm = np.array([[True, True, False]] * 3)
    traces["random"] = RoutingTrace(ModelShape(3, 6, 2), "r", pt, pt[:2], pp, pm, pp[:2], pm[:2])
    # a generator trace at the Mixtral shape (moesim/generator.py)
    cfg = GeneratorConfig(shape=ModelShape(32, 8, 2), seed=3, num_prefill_tokens=16,
                          num_decode_tokens=4, sequence_id="gen3",
                          prefill_decode_similarity_target=0.6)
    traces["mixtral_gen"] = generate_trace(cfg)
    for name, tr in traces.items():
        save_trace(tr, OUT / f"{name}.jsonl")
    print("wrote", sorted(traces))


if __name__ == "__main__":
    main()
