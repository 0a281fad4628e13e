"""Oracle (TEST / BASELINE INFRASTRUCTURE ONLY): the CPU path timed beside the
GPU in bench.py (`cpu_baseline` and `--impl reference`).

`CpuMoELayer` executes the MoE block exactly as restated in
oracle/numerics.py and the decisions exactly as restated in
oracle/decisions.py (the reference's own algorithm, pinned to its golden
vectors) in three variants, all on every host core: numpy fp32 on the
bf16-valued weights (BLAS thread pool); torch-CPU bf16 (oneDNN, fp32
accumulation); and plain C on the bf16 weights as stored (oracle/cpu_moe.c,
OpenMP, fp32 accumulation -- half the weight bytes of the fp32 port).
bench.py times all three and reports the fastest as the CPU baseline
(BASELINE.md §3 asked for bf16 weights with fp32 accumulation).  Weights come
from the oracle generator (oracle/rng.py), generated in parallel threads
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
    """One MoE layer (all experts) on the host, weights as fp32 arrays (and,
    with_bf16, as torch bf16 tensors for the bf16 variant)."""

    def __init__(self, num_layers, num_experts, top_k, d, ffn, seed=0, layer=0, threads=None,
                 with_bf16=False):
        self.om = N.OracleModel(num_layers, num_experts, top_k, d, ffn, seed)
        self.layer, self.E, self.k, self.d, self.ffn = layer, num_experts, top_k, d, ffn
        self.threads = threads or len(os.sched_getaffinity(0))
        jobs = [(e, m) for e in range(num_experts) for m in range(3)]
        fns = {0: self.om.w1, 1: self.om.w3, 2: self.om.w2}
        with ThreadPoolExecutor(self.threads) as ex:
            mats = list(ex.map(lambda em: fns[em[1]](layer, em[0]), jobs))
        self.w = {(e, m): mats[i] for i, (e, m) in enumerate(jobs)}
        self.gate = self.om.gate(layer)
        self.gate_next = self.om.gate(layer + 1) if layer + 1 < num_layers else None
        self.norm = self.om.norm(layer)
        self.torch = None
        if with_bf16:
            import torch
            torch.set_num_threads(self.threads)
            self.torch = torch
            # the weights are bf16-valued, so the conversion is exact
            self.w13 = [torch.cat([torch.from_numpy(self.w[(e, 0)]),
                                   torch.from_numpy(self.w[(e, 1)])]).to(torch.bfloat16)
                        for e in range(num_experts)]
            self.w2b = [torch.from_numpy(self.w[(e, 2)]).to(torch.bfloat16)
                        for e in range(num_experts)]

    # ---- plain-C bf16 variant (oracle/cpu_moe.c): bf16 weights as stored,
    # fp32 accumulation, OpenMP over every host core
    def _c(self):
        if getattr(self, "_lib", None) is None:
            import ctypes
            from .build import build
            lib = ctypes.CDLL(str(build()))
            lib.oracle_expert_ffn.argtypes = [ctypes.c_void_p, ctypes.c_int] + \
                [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_void_p]
            lib.oracle_threads.restype = ctypes.c_int
            self._lib = lib
            # the weights are bf16-valued fp32: their top 16 bits are the bf16
            self.wb = {key: np.ascontiguousarray((w.view(np.uint32) >> 16).astype(np.uint16))
                       for key, w in self.w.items()}
        return self._lib

    def _expert_c(self, e, x):
        lib = self._c()
        x = np.ascontiguousarray(x, dtype=np.float32)
        n = x.shape[0]
        act = np.empty((n, self.ffn), dtype=np.float32)
        y = np.empty((n, self.d), dtype=np.float32)
        lib.oracle_expert_ffn(x.ctypes.data, n, self.wb[(e, 0)].ctypes.data,
                              self.wb[(e, 1)].ctypes.data, self.wb[(e, 2)].ctypes.data, self.d,
                              self.ffn, act.ctypes.data, y.ctypes.data)
        return y

    def c_threads(self) -> int:
        return int(self._c().oracle_threads())

    def decode_step_c(self, h: np.ndarray):
        """decode_step with the experts in plain C on bf16 weights."""
        x = N.rmsnorm(h[None, :], self.norm)
        p, _ = N.router(x, self.gate, self.gate_next)
        sel = D.topk_rows(p.astype(np.float64), self.k)
        w = N.renorm_weights(p, sel)
        out = h.astype(np.float32).copy()
        for j, e in enumerate(sel[0]):
            out = out + w[0, j] * self._expert_c(int(e), x)[0]
        return out, sel[0]

    def prefill_c(self, h: np.ndarray):
        x = N.rmsnorm(h, self.norm)
        p, _ = N.router(x, self.gate, self.gate_next)
        sel = D.topk_rows(p.astype(np.float64), self.k)
        w = N.renorm_weights(p, sel)
        off, perm, inv = N.permutation(sel, self.E)
        y = np.zeros((sel.size, h.shape[1]), dtype=np.float32)
        for e in range(self.E):
            a, b = int(off[e]), int(off[e + 1])
            if a < b:
                y[a:b] = self._expert_c(e, x[perm[a:b] // self.k])
        return N.combine(h, y, inv, w)

    def _expert_bf16(self, e, x_bf16):
        """torch-CPU bf16: [W1; W3] in one GEMM (oneDNN, fp32 accumulation,
        bf16 outputs), SwiGLU in fp32 -> bf16 act, W2 GEMM -> fp32."""
        F = self.torch.nn.functional
        gu = F.linear(x_bf16, self.w13[e]).float()
        act = (F.silu(gu[:, : self.ffn]) * gu[:, self.ffn:]).to(self.torch.bfloat16)
        return F.linear(act, self.w2b[e]).float()

    def decode_step_bf16(self, h: np.ndarray):
        """decode_step with the experts in torch-CPU bf16."""
        torch = self.torch
        x = N.rmsnorm(h[None, :], self.norm)
        p, _ = N.router(x, self.gate, self.gate_next)
        sel = D.topk_rows(p.astype(np.float64), self.k)
        w = N.renorm_weights(p, sel)
        xb = torch.from_numpy(x).to(torch.bfloat16)
        out = torch.from_numpy(h.astype(np.float32))
        for j, e in enumerate(sel[0]):
            out = out + float(w[0, j]) * self._expert_bf16(int(e), xb)[0]
        return out.numpy(), sel[0]

    def prefill_bf16(self, h: np.ndarray):
        torch = self.torch
        x = N.rmsnorm(h, self.norm)
        p, _ = N.router(x, self.gate, self.gate_next)
        sel = D.topk_rows(p.astype(np.float64), self.k)
        w = N.renorm_weights(p, sel)
        off, perm, inv = N.permutation(sel, self.E)
        y = np.zeros((sel.size, h.shape[1]), dtype=np.float32)
        xb = torch.from_numpy(x).to(torch.bfloat16)
        for e in range(self.E):
            a, b = int(off[e]), int(off[e + 1])
            if a < b:
                rows = torch.from_numpy(perm[a:b] // self.k)
                y[a:b] = self._expert_bf16(e, xb[rows]).numpy()
        return N.combine(h, y, inv, w)

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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    return "unknown"


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
