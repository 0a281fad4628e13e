"""Non-MoE block of a Mixtral-shaped decoder layer.

The reference prices this block as a constant (`t_nonmoe`,
moesim/simulator.py:291); the paper's block is "self-attention, expert
layers, normalization, and residual connections".
`AttentionStack` holds, per layer, the attention RMSNorm weight, the fused
QKV projection [Wq; Wk; Wv] (q + 2 kv, d), the output projection Wo (d, q)
-- bf16, random-init from the counter generator like the experts -- and a
bf16 KV cache (n_kv, max_seq, 128).  `decode(h, layer, pos)` runs one token
through csrc/attention.cu (daop_attn_decode: RMSNorm -> QKV GEMV -> RoPE ->
cache append -> GQA flash-decoding -> O-proj GEMV + residual); `prefill(h,
layer, pos0)` runs a whole prompt causally: RMSNorm rows, the QKV projection
on the tcgen05 GEMM pipeline (daop_gemm_bf16_f32), RoPE + cache append,
FlashAttention-style causal attention on the tensor cores
(daop_attn_prefill), and the O projection with the residual added in the
GEMM epilogue.  Mixtral-8x7B:
d 4096, 32 query heads, 8 KV heads, head dim 128, rope theta 1e6.
"""

from __future__ import annotations

import torch

from . import _lib, ops
from .errors import ShapeMismatchError
from .model import make_tag

KIND_ATTN = 5      # matrix 0 = Wqkv (q + 2 kv, d), 1 = Wo (d, q)
NORM_LAYER_OFFSET = 4096  # attention RMSNorm weights: norm stream of layer + 4096
HEAD_DIM = 128


class AttentionStack:
    def __init__(self, num_layers: int, d_model: int, n_heads: int = 32, n_kv: int = 8,
                 max_seq: int = 4096, theta: float = 1e6, seed: int = 0, device="cuda"):
        self.L, self.d, self.n_heads, self.n_kv = num_layers, d_model, n_heads, n_kv
        self.max_seq, self.theta, self.seed = max_seq, theta, seed
        self.split_k = True  # prompt projections: split-K path (daop_gemm_bf16_f32_ws)
        self.device = torch.device(device)
        self.q_dim, self.kv_dim = n_heads * HEAD_DIM, n_kv * HEAD_DIM
        rows = self.q_dim + 2 * self.kv_dim
        import numpy as np
        s_in = float(np.float32(1.0 / np.sqrt(d_model)))
        s_o = float(np.float32(1.0 / np.sqrt(self.q_dim)))
        dev = self.device
        self.norm = torch.empty((num_layers, d_model), dtype=torch.bfloat16, device=dev)
        self.wqkv = torch.empty((num_layers, rows, d_model), dtype=torch.bfloat16, device=dev)
        self.wo = torch.empty((num_layers, d_model, self.q_dim), dtype=torch.bfloat16, device=dev)
        for l in range(num_layers):
            ops.fill_norm_bf16(self.norm[l], seed, l + NORM_LAYER_OFFSET)
            ops.fill_uniform_bf16(self.wqkv[l], seed, make_tag(KIND_ATTN, l, 0, 0), s_in)
            ops.fill_uniform_bf16(self.wo[l], seed, make_tag(KIND_ATTN, l, 0, 1), s_o)
        self.k_cache = torch.zeros((num_layers, n_kv, max_seq, HEAD_DIM), dtype=torch.bfloat16,
                                   device=dev)
        self.v_cache = torch.zeros_like(self.k_cache)
        nb = torch.zeros(1, dtype=torch.int64)
        _lib.call("daop_attn_workspace", n_heads, n_kv, max_seq, nb.data_ptr())
        self.ws = torch.zeros(int(nb[0]), dtype=torch.uint8, device=dev)
        self.xa = torch.empty(d_model, dtype=torch.bfloat16, device=dev)

    def decode(self, h: torch.Tensor, layer: int, pos: int, out: torch.Tensor | None = None):
        """h (d,) fp32 on the device -> h + Attention(RMSNorm(h)) (d,) fp32;
        appends this token's k, v at `pos` of the layer's cache."""
        ops._dev(h)
        out = torch.empty_like(h) if out is None else out
        _lib.call("daop_attn_decode", h.data_ptr(), self.norm[layer].data_ptr(),
                  self.wqkv[layer].data_ptr(), self.wo[layer].data_ptr(),
                  self.k_cache[layer].data_ptr(), self.v_cache[layer].data_ptr(), self.d,
                  self.n_heads, self.n_kv, self.max_seq, int(pos), float(ops.RMS_EPS),
                  float(self.theta), self.xa.data_ptr(), out.data_ptr(), self.ws.data_ptr(),
                  ops._s())
        return out

    def prefill(self, h: torch.Tensor, layer: int, pos0: int = 0,
                out: torch.Tensor | None = None):
        """h (T, d) fp32 on the device: T prompt tokens at positions pos0 ..
        pos0 + T - 1 -> h + Attention(RMSNorm(h)) (T, d) fp32, causal; appends
        every token's k, v to the layer's cache.  Every step is a library kernel:
        daop_attn_norm_rows, daop_gemm_bf16_f32 (QKV, tcgen05), daop_attn_prefill
        (RoPE + append, tensor-core flash attention), daop_gemm_bf16_f32 (O-proj
        + residual, tcgen05)."""
        ops._dev(h)
        T, d = h.shape
        if pos0 < 0 or pos0 + T > self.max_seq:
            raise ShapeMismatchError(f"prefill positions {pos0}..{pos0 + T - 1} exceed max_seq "
                                     f"{self.max_seq}")
        xa = torch.empty((T, d), dtype=torch.bfloat16, device=h.device)
        _lib.call("daop_attn_norm_rows", h.data_ptr(), T, self.norm[layer].data_ptr(), d,
                  float(ops.RMS_EPS), xa.data_ptr(), ops._s())
        ws = True if self.split_k else None  # split-K over idle SMs for short prompts
        qkv = ops.gemm_bf16_f32(xa, self.wqkv[layer], ws=ws)
        o = torch.empty((T, self.q_dim), dtype=torch.bfloat16, device=h.device)
        _lib.call("daop_attn_prefill", qkv.data_ptr(), T, int(pos0),
                  self.k_cache[layer].data_ptr(), self.v_cache[layer].data_ptr(), self.n_heads,
                  self.n_kv, self.max_seq, float(self.theta), o.data_ptr(), ops._s())
        # O projection with the residual added in the GEMM epilogue
        return ops.gemm_bf16_f32(o, self.wo[layer], resid=h, out=out, ws=ws)

    def prefetch_l2(self, layer: int) -> None:
        """Queue an L2 prefetch of `layer`'s Wqkv and Wo (84 MB at the
        Mixtral-8x7B shape) on the current stream (daop_l2_prefetch): issued
        before the previous layer's MoE decode kernel, it is in L2 when this
        layer's attention GEMVs run."""
        if 0 <= layer < self.L:
            a, b = self.wqkv[layer], self.wo[layer]
            _lib.call("daop_l2_prefetch", a.data_ptr(), a.numel() * 2, b.data_ptr(),
                      b.numel() * 2, ops._s())

    def bytes_per_token_layer(self, ctx: int) -> int:
        """Algorithmic HBM bytes of one decode step of one layer at context
        length ctx: Wqkv + Wo + the k, v rows read (bf16)."""
        w = (self.q_dim + 2 * self.kv_dim) * self.d * 2 + self.d * self.q_dim * 2
        return w + ctx * self.n_kv * HEAD_DIM * 2 * 2
