"""MoE-block execution engine: the numeric hot path the reference only prices.

`MoEBlockEngine` runs one MoE layer of a `MoEModel` on the device:

  decode(h, layer, ...)   one token, one persistent launch (daop_decode_layer):
                          router + DAOP decision + HBM-streaming SwiGLU GEMV +
                          combine.
  prefill(h, layer, ...)  T tokens: fused router (with the per-sequence
                          activation counter) -> stable permutation ->
                          tcgen05 grouped up/down GEMMs -> combine.
  decode_host(h_host)     the end-to-end call a user makes with host memory:
                          H2D of the token, the decode launch, D2H of the
                          result (used for bench.py's `e2e`).

Every buffer is preallocated per engine so the decode step has fixed
addresses (CUDA-graph capturable).  The DAOP sequence-level flow
(calibration init -> prefill counts -> Alg. 1 swaps -> decode plans) is in
daop.py.
"""

from __future__ import annotations

import os
import torch

from . import _lib, ops
from .model import MoEModel


# up to this many permuted rows (T * k) the layer runs the skinny (swap-AB)
# GEMMs of batched decode: below it the prefill GEMM tiles are mostly empty.
# scripts/skinny_crossover.py (8x7B layer, up + down): T 256 0.63 vs 0.96 ms,
# T 384 0.92 vs 1.03, T 512 1.17 vs 1.09 (skinny vs 512-row pair tiles)
SKINNY_MAX_ROWS = 768


class MoEBlockEngine:
    def __init__(self, model: MoEModel, device=None):
        self.model = model
        self.device = model.device if device is None else torch.device(device)
        s = model.shape
        self.d, self.ffn, self.E, self.k = model.d, model.ffn, s.num_experts, s.top_k
        self.bufs = ops.DecodeBuffers(self.d, self.ffn, self.E, self.k, self.device)
        self._h_dev = torch.empty(self.d, dtype=torch.float32, device=self.device)
        self._h_host = None
        self._out_host = None
        self._sel_host = None
        # full decoder layers: prefetch layer l+1's attention weights into L2
        # while layer l's MoE kernel streams its experts.  Measured slower
        # (decoder32 192.7 vs 206.4 tok/s, DESIGN §6 tried and rejected): off
        self.attn_prefetch = False
        # decoder layers: PLAN-mode MoE launches stream before the O-proj ends
        self.decode_early = os.environ.get("DAOP_DECODE_EARLY", "1") != "0"

    # ------------------------------------------------------------ decode
    def decode(self, h: torch.Tensor, layer: int = 0, *, pred_prev=None, mode: int = 0,
               graceful: bool = True, weights_from_pred: bool = False, variant: int = 0,
               h_out=None, sel_out=None):
        """One decode token (h: (d,) fp32 on device) through MoE layer `layer`.
        mode 0 selects by the layer's own gate (true top-k), mode 1 by the DAOP
        plan on `pred_prev` (the prediction carried on layer-1)."""
        m = self.model
        nxt = m.gate[layer + 1] if layer + 1 < m.shape.num_layers else None
        return ops.decode_layer(h, m.norm[layer], m.gate[layer], nxt, m.fast[layer],
                                m.slot_of[layer], m.slab, m.slot_elems, self.d, self.ffn, self.k,
                                self.bufs, pred_prev=pred_prev, mode=mode, graceful=graceful,
                                weights_from_pred=weights_from_pred, variant=variant,
                                h_out=h_out, sel_out=sel_out)

    def decode_host(self, h_host: torch.Tensor, layer: int = 0):
        """End-to-end call from host memory: h (d,) fp32 on the host -> device
        -> decode -> (h_out, selected experts) in pinned host memory.

        The step is one CUDA graph per layer (captured on first use): the H2D
        copy of h from a pinned staging buffer, then the decode launch, which
        writes the residual and the selection straight into pinned host memory
        over the bus (no D2H copy node).  The caller's h is copied into the
        staging buffer, the graph launched and the stream synchronised in one
        native call (daop_graph_step)."""
        c = self._host_graphs.get(layer) if self._out_host is not None else None
        if c is not None and h_host.dtype is torch.float32 and not h_host.is_cuda and \
                h_host.is_contiguous() and h_host.numel() == self.d:
            # fast path: staging copy + launch + wait in one native call
            rc = c[0](c[1], c[2], h_host.data_ptr(), c[3], c[4])
            if rc:
                _lib.check(rc, "daop_graph_step")
            return self._out_host, self._sel_host
        if self._out_host is None:
            self._h_host = torch.empty(self.d, dtype=torch.float32, pin_memory=True)
            self._out_host = torch.empty(self.d, dtype=torch.float32, pin_memory=True)
            self._sel_host = torch.empty(self.k, dtype=torch.int32, pin_memory=True)
            self._host_graphs = {}
        self._h_host.copy_(h_host)
        if layer not in self._host_graphs:
            def step():
                self._h_dev.copy_(self._h_host, non_blocking=True)
                self.decode(self._h_dev, layer, h_out=self._out_host, sel_out=self._sel_host)

            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()  # warm-up outside capture
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            self._graphs_keepalive = getattr(self, "_graphs_keepalive", []) + [g]
            self._host_graphs[layer] = (_lib.LIB.daop_graph_step, g.raw_cuda_graph_exec(),
                                        torch.cuda.current_stream().cuda_stream,
                                        self._h_host.data_ptr(), 4 * self.d)
        c = self._host_graphs[layer]
        _lib.check(c[0](c[1], c[2], c[3], c[3], c[4]), "daop_graph_step")
        return self._out_host, self._sel_host

    def decode_server(self, layer: int = 0, idle_ms: float = 5000.0):
        """Persistent serving mode of `decode_host` (daop_server_*): one
        resident kernel answers every call -- h is read from pinned host
        memory when the host rings, the residual and the selection are written
        back to pinned host memory -- so a call costs no launch and no stream
        synchronisation.  The kernel holds every SM: use it as a context
        manager and run no other GPU work while it is open."""
        return DecodeServer(self, layer, idle_ms)

    @staticmethod
    def host_bytes(d: int, k: int):
        """(h2d, d2h) bytes of one decode_host call: h in; the residual and
        the selection written to host memory by the kernel."""
        return d * 4, d * 4 + k * 4

    # ------------------------------------------------------------ full decode token
    def decode_token(self, h: torch.Tensor, *, start: int = 4, daop: bool = True,
                     weights_from_pred: bool = True, attn=None, pos: int = 0) -> torch.Tensor:
        """One decode token through every layer, all experts HBM-resident:
        layer l < start (or fiddler) selects by its own gate, layer l >= start
        by the DAOP plan on the prediction carried by layer l-1 -- known when
        the launch starts, so its weight stream starts before its router runs.
        With `attn` (an AttentionStack) every layer is a full decoder layer:
        h <- h + Attention(RMSNorm(h)) at position `pos` (KV cache append),
        then the MoE block.  Returns the final residual (a view into a
        ping-pong buffer)."""
        m = self.model
        L = m.shape.num_layers
        if not hasattr(self, "_pp"):
            self._pp = [ops.DecodeBuffers(self.d, self.ffn, self.E, self.k, self.device)
                        for _ in range(2)]
        if attn is not None and not hasattr(self, "_ha"):
            self._ha = torch.empty(self.d, dtype=torch.float32, device=self.device)
        cur = h
        for l in range(L):
            if attn is not None:
                cur = attn.decode(cur, l, pos, out=self._ha)
                if self.attn_prefetch:
                    attn.prefetch_l2(l + 1)  # streams beside this layer's MoE kernel
            b = self._pp[l % 2]
            mode = 1 if (daop and l >= start) else 0
            nxt = m.gate[l + 1] if l + 1 < L else None
            # PLAN layers behind the attention O-proj start streaming their
            # predicted experts before the O-proj completes (variant bit 8)
            early = 0x100 if (attn is not None and mode == 1 and self.decode_early) else 0
            ops.decode_layer(cur, m.norm[l], m.gate[l], nxt, m.fast[l], m.slot_of[l], m.slab,
                             m.slot_elems, self.d, self.ffn, self.k, b,
                             pred_prev=self._pp[(l + 1) % 2].p_pred if mode else None,
                             mode=mode, weights_from_pred=weights_from_pred and mode == 1,
                             variant=early)
            cur = b.h_out
        return cur

    def capture_decode_graph(self, *, start: int = 4, daop: bool = True):
        """Capture decode_token into one CUDA graph (fixed input/output
        buffers): the L persistent launches replay without host involvement.
        Returns (graph, h_in, h_out)."""
        h_in = torch.zeros(self.d, dtype=torch.float32, device=self.device)
        self.decode_token(h_in, start=start, daop=daop)  # allocate + warm
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.decode_token(h_in, start=start, daop=daop)
        return g, h_in, out

    # ------------------------------------------------------------ prefill
    def prefill(self, h: torch.Tensor, layer: int = 0, *, hist=None, tokens_per_seq: int = 0,
                hist_seq_stride: int = 0, group_up: int = 0, group_down: int = 0,
                fused_combine: bool = False):
        """T tokens (h: (T, d) fp32 on device) through MoE layer `layer`.
        Returns dict(out, p, p_pred, topk_idx, topk_w).  `hist` (optional,
        int32 view [seq, E] of this layer) receives the activation counts."""
        m = self.model
        nxt = m.gate[layer + 1] if layer + 1 < m.shape.num_layers else None
        r = ops.router(h, m.norm[layer], m.gate[layer], nxt, self.k, hist=hist,
                       tokens_per_seq=tokens_per_seq, hist_seq_stride=hist_seq_stride)
        pr = ops.permute(r["topk_idx"], self.E, r["x"])
        slot_of = m.slot_of[layer]
        rows = pr["x_perm"].shape[0]
        if rows <= SKINNY_MAX_ROWS and not fused_combine:
            # batched decode: weights are the M side, tokens the N side
            act = ops.expert_gemm_up_skinny(pr["x_perm"], pr["offsets"], slot_of, m.slab,
                                            m.n_slots, m.slot_elems, self.d, self.ffn)
            y = ops.expert_gemm_down_skinny(act, pr["offsets"], slot_of, m.slab, m.n_slots,
                                            m.slot_elems, self.d, self.ffn)
            r["out"] = ops.combine(h, y, pr["inv"], r["topk_w"])
            r["offsets"] = pr["offsets"]
            return r
        act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], slot_of, m.slab, m.n_slots,
                                 m.slot_elems, self.d, self.ffn, group_up)
        if fused_combine:  # combine in the down GEMM's epilogue (measured slower: off)
            out, y = ops.expert_gemm_down_combine(act, pr["offsets"], slot_of, m.slab, m.n_slots,
                                                  m.slot_elems, self.d, self.ffn, pr["perm"],
                                                  pr["inv"], h, r["topk_w"], group_down)
        else:
            y = ops.expert_gemm_down(act, pr["offsets"], slot_of, m.slab, m.n_slots,
                                     m.slot_elems, self.d, self.ffn, group_down)
            out = ops.combine(h, y, pr["inv"], r["topk_w"])
        r["out"] = out
        r["offsets"] = pr["offsets"]
        return r

    @staticmethod
    def prefill_kernels(tokens: int = 1 << 20, k: int = 2) -> int:
        """Kernel launches of one prefill layer of `tokens` tokens: router,
        permute (count, scan, scatter -- one fused kernel when tokens * k fits
        one 4096-row chunk -- then gather), up GEMM, down GEMM, combine."""
        return 6 if tokens * k <= 4096 else 8


class DecodeServer:
    """See MoEBlockEngine.decode_server."""

    def __init__(self, eng: MoEBlockEngine, layer: int, idle_ms: float):
        import ctypes
        m = eng.model
        self.eng = eng
        self.d, self.k = eng.d, eng.k
        self.out = torch.empty(self.d, dtype=torch.float32, pin_memory=True)
        self.sel = torch.empty(self.k, dtype=torch.int32, pin_memory=True)
        self.bufs = ops.DecodeBuffers(eng.d, eng.ffn, eng.E, eng.k, eng.device)
        self.stream = torch.cuda.Stream(eng.device)
        nxt = m.gate[layer + 1] if layer + 1 < m.shape.num_layers else None
        if not bool(m.fast[layer].all()):
            from .errors import ConfigError
            raise ConfigError("decode_server needs every expert of the layer in HBM "
                              "(the slow tier is host work between kernel phases)")
        b = self.bufs
        self._h = ctypes.c_void_p()
        torch.cuda.synchronize(eng.device)  # weights and buffers ready before the kernel starts
        _lib.call("daop_server_start", m.norm[layer].data_ptr(), m.gate[layer].data_ptr(),
                  0 if nxt is None else nxt.data_ptr(), m.fast[layer].data_ptr(),
                  m.slot_of[layer].data_ptr(), m.slab.data_ptr(), m.slot_elems, eng.d, eng.ffn,
                  eng.E, eng.k, float(ops.RMS_EPS), b.x.data_ptr(), b.p.data_ptr(),
                  b.p_pred.data_ptr(), self.sel.data_ptr(), b.w.data_ptr(),
                  b.is_fast.data_ptr(), b.deg.data_ptr(), b.y.data_ptr(), self.out.data_ptr(),
                  b.ws.data_ptr(), float(idle_ms), self.stream.cuda_stream, ctypes.byref(self._h))
        self._step = _lib.LIB.daop_server_step

    def step(self, h_host: torch.Tensor, timeout_ms: float = 5000.0):
        """One decode call: h (d,) fp32 in host memory -> (residual, selection)
        in pinned host memory (valid until the next call)."""
        if self._h is None:
            raise RuntimeError("decode server is closed")
        if h_host.dtype is not torch.float32 or h_host.is_cuda or not h_host.is_contiguous() \
                or h_host.numel() != self.d:
            h_host = h_host.to(device="cpu", dtype=torch.float32).contiguous().view(-1)
        rc = self._step(self._h, h_host.data_ptr(), float(timeout_ms))
        if rc:
            _lib.check(rc, "daop_server_step")
        return self.out, self.sel

    def close(self):
        if self._h is not None:
            h, self._h = self._h, None
            _lib.call("daop_server_stop", h)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
