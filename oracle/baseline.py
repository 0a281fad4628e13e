"""Oracle (TEST / BASELINE INFRASTRUCTURE ONLY): the CPU path timed beside the
GPU in bench.py (`cpu_baseline` and `--impl reference`).

It executes the MoE block exactly as restated in oracle/numerics.py and the
decisions exactly as restated in oracle/decisions.py (the reference's own
algorithm, pinned to its golden vectors) -- numpy, fp32 arithmetic on
bf16-valued weights, all host cores through the BLAS thread pool.  Weights
come from the oracle generator (oracle/rng.py), generated in parallel threads
(numpy releases the GIL), so nothing from the product package is used.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import decisions as D
from . import numerics as N


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:  # pragma: no cover
        pass
    return len(os.sched_getaffinity(0))


class CpuMoELayer:
    """One MoE layer (all experts) on the host, weights as fp32 arrays."""

    def __init__(self, num_layers, num_experts, top_k, d, ffn, seed=0, layer=0, threads=None):
        self.om = N.OracleModel(num_layers, num_experts, top_k, d, ffn, seed)
        self.layer, self.E, self.k = layer, num_experts, top_k
        jobs = [(e, m) for e in range(num_experts) for m in range(3)]
        fns = {0: self.om.w1, 1: self.om.w3, 2: self.om.w2}
        with ThreadPoolExecutor(threads or len(os.sched_getaffinity(0))) as ex:
            mats = list(ex.map(lambda em: fns[em[1]](layer, em[0]), jobs))
        self.w = {(e, m): mats[i] for i, (e, m) in enumerate(jobs)}
        self.gate = self.om.gate(layer)
        self.gate_next = self.om.gate(layer + 1) if layer + 1 < num_layers else None
        self.norm = self.om.norm(layer)

    def decode_step(self, h: np.ndarray):
        """One token (d,) through the layer: router -> top-k -> SwiGLU experts
        -> combine.  Returns (h_out, sel)."""
        x = N.rmsnorm(h[None, :], self.norm)
        p, _ = N.router(x, self.gate, self.gate_next)
        sel = D.topk_rows(p.astype(np.float64), self.k)
        w = N.renorm_weights(p, sel)
        out = h.astype(np.float32).copy()
        for j, e in enumerate(sel[0]):
            y = N.expert_ffn(x, self.w[(e, 0)], self.w[(e, 1)], self.w[(e, 2)])[0]
            out = out + w[0, j] * y
        return out, sel[0]

    def prefill(self, h: np.ndarray):
        x = N.rmsnorm(h, self.norm)
        p, _ = N.router(x, self.gate, self.gate_next)
        sel = D.topk_rows(p.astype(np.float64), self.k)
        w = N.renorm_weights(p, sel)
        off, perm, inv = N.permutation(sel, self.E)
        y = np.zeros((sel.size, h.shape[1]), dtype=np.float32)
        for e in range(self.E):
            a, b = int(off[e]), int(off[e + 1])
            if a < b:
                rows = perm[a:b] // self.k
                y[a:b] = N.expert_ffn(x[rows], self.w[(e, 0)], self.w[(e, 1)], self.w[(e, 2)])
        return N.combine(h, y, inv, w)


def time_steps(fn, inputs, budget_s: float, max_steps: int, warmup: int = 1):
    """min(max_steps, as many as fit in budget_s) timed calls; returns (n, seconds)."""
    for i in range(warmup):
        fn(inputs[i % len(inputs)])
    n, t0 = 0, time.perf_counter()
    while n < max_steps:
        fn(inputs[n % len(inputs)])
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return n, time.perf_counter() - t0
