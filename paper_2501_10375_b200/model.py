"""Mixtral-shaped MoE model state in HBM: router gates, RMSNorm weights and the
expert slot slab.

Layout:
  gate   (L, E, d)   bf16   -- gate of layer l is gate[l]; the fused router
                               reads gate[l] and gate[l+1] from one x read
  norm   (L, d)      bf16
  slab   (S, 3*ffn*d) bf16  -- one slot = [W1 (ffn,d) | W3 (ffn,d) | W2 (d,ffn)],
                               contiguous so a migration is one memcpy and the
                               grouped GEMM addresses any slot with one 3-D TMA
                               descriptor (d, rows, slot)
  slot_of (L, E)     int32  -- HBM slot of (layer, expert) or -1 (host tier)
  fast   (L, E)      uint8  -- residence mask (== slot_of >= 0)

Weights are random-init from the counter-based generator (csrc/rng.cuh ==
oracle/rng.py): W1/W3 ~ U(+-1/sqrt(d)), W2 ~ U(+-1/sqrt(ffn)), gates
U(+-1/sqrt(d)), all rounded to bf16; RMSNorm weight bf16(1 + 0.25 u).  No
checkpoints exist in this environment; BASELINE.json asks for random init.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .trace import ModelShape

KIND_EXPERT, KIND_GATE, KIND_NORM, KIND_INPUT = 1, 2, 3, 4


def make_tag(kind: int, layer: int = 0, expert: int = 0, matrix: int = 0) -> int:
    return (kind << 56) | (layer << 32) | (expert << 16) | matrix


class MoEModel:
    def __init__(self, shape: ModelShape, d_model: int, d_ff: int, seed: int = 0,
                 device="cuda", n_slots: int | None = None, resident_layers=None):
        self.shape = shape
        self.d, self.ffn, self.seed = d_model, d_ff, seed
        self.device = torch.device(device)
        L, E = shape.num_layers, shape.num_experts
        self.scale_in = float(np.float32(1.0 / np.sqrt(d_model)))
        self.scale_ff = float(np.float32(1.0 / np.sqrt(d_ff)))
        self.slot_elems = 3 * d_ff * d_model
        self.gate = torch.empty((L, E, d_model), dtype=torch.bfloat16, device=self.device)
        self.norm = torch.empty((L, d_model), dtype=torch.bfloat16, device=self.device)
        for l in range(L):
            ops.fill_uniform_bf16(self.gate[l], seed, make_tag(KIND_GATE, l), self.scale_in)
            ops.fill_norm_bf16(self.norm[l], seed, l)
        layers = list(range(L)) if resident_layers is None else list(resident_layers)
        if n_slots is None:
            n_slots = len(layers) * E
        self.n_slots = n_slots
        self.slab = torch.empty((n_slots, self.slot_elems), dtype=torch.bfloat16,
                                device=self.device)
        self.slot_of = torch.full((L, E), -1, dtype=torch.int32, device=self.device)
        self.fast = torch.zeros((L, E), dtype=torch.uint8, device=self.device)
        self._slot_host = np.full((L, E), -1, dtype=np.int64)
        self._free = list(range(n_slots))
        for l in layers:
            for e in range(E):
                if self._free:
                    self.load_expert(l, e)

    # -- expert weights ----------------------------------------------------
    def expert_views(self, slot: int):
        d, f = self.d, self.ffn
        s = self.slab[slot]
        return s[: f * d].view(f, d), s[f * d: 2 * f * d].view(f, d), s[2 * f * d:].view(d, f)

    def generate_expert(self, layer: int, expert: int, slot: int) -> None:
        """Materialise W1/W3/W2 of (layer, expert) into a slab slot on device."""
        w1, w3, w2 = self.expert_views(slot)
        ops.fill_uniform_bf16(w1, self.seed, make_tag(KIND_EXPERT, layer, expert, 0), self.scale_in)
        ops.fill_uniform_bf16(w3, self.seed, make_tag(KIND_EXPERT, layer, expert, 1), self.scale_in)
        ops.fill_uniform_bf16(w2, self.seed, make_tag(KIND_EXPERT, layer, expert, 2), self.scale_ff)

    def load_expert(self, layer: int, expert: int, slot: int | None = None) -> int:
        if slot is None:
            slot = self._free.pop(0)
        elif slot in self._free:
            self._free.remove(slot)
        self.generate_expert(layer, expert, slot)
        self._bind(layer, expert, slot)
        return slot

    def _bind(self, layer, expert, slot):
        self._slot_host[layer, expert] = slot
        self.slot_of[layer, expert] = slot
        self.fast[layer, expert] = 1

    def evict(self, layer: int, expert: int) -> int:
        slot = int(self._slot_host[layer, expert])
        self._slot_host[layer, expert] = -1
        self.slot_of[layer, expert] = -1
        self.fast[layer, expert] = 0
        self._free.append(slot)
        return slot

    def resident_mask(self) -> np.ndarray:
        return (self._slot_host >= 0).astype(np.uint8)

    def slot(self, layer: int, expert: int) -> int:
        return int(self._slot_host[layer, expert])

    # -- inputs ------------------------------------------------------------
    def input_hidden(self, t: int, stream: int = 0, step: int = 0) -> torch.Tensor:
        """Synthetic residual-stream input h (t, d) fp32 ~ U(-sqrt3, sqrt3)."""
        h = torch.empty((t, self.d), dtype=torch.float32, device=self.device)
        return ops.fill_uniform_f32(h, self.seed, make_tag(KIND_INPUT, stream, step),
                                    float(np.float32(np.sqrt(3.0))))
