"""Routing data types -- the parity interchange format.

Same public surface as moesim/trace.py (ModelShape :35-53, presets :57-58,
TokenRouting :80-110, RoutingTrace :129-322, SCORE_SUM_TOL :30).  The B200
engine *produces* these from its fused router (true gate of every layer plus
the next-layer prediction), so an engine run can be handed unchanged to the
reference's own analysis functions, and the reference's decisions on it can be
compared with the GPU's with ``==``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .errors import NormalizationError, ShapeMismatchError

SCORE_SUM_TOL = 1e-6
PHASES = ("prefill", "decode")


@dataclass(frozen=True)
class ModelShape:
    """(layers, experts, top-k) of the MoE model."""

    num_layers: int
    num_experts: int
    top_k: int

    def __post_init__(self):
        if self.num_layers < 1:
            raise ShapeMismatchError(f"num_layers must be >= 1, got {self.num_layers}")
        if self.num_experts < 2:
            raise ShapeMismatchError(f"num_experts must be >= 2, got {self.num_experts}")
        if not 1 <= self.top_k <= self.num_experts:
            raise ShapeMismatchError(
                f"top_k must be in [1, {self.num_experts}], got {self.top_k}")


MIXTRAL_SHAPE = ModelShape(num_layers=32, num_experts=8, top_k=2)
PHI_SHAPE = ModelShape(num_layers=32, num_experts=16, top_k=2)


def _frozen(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    a.flags.writeable = False
    return a


def _validate_vector(vec: np.ndarray, name: str) -> None:
    if vec.ndim != 1:
        raise ShapeMismatchError(f"{name} must be a 1-D vector")
    if np.any(vec < 0) or not np.all(np.isfinite(vec)):
        raise NormalizationError(f"{name} has negative or non-finite entries")
    total = float(vec.sum())
    if abs(total - 1.0) > SCORE_SUM_TOL:
        raise NormalizationError(f"{name} sums to {total!r}, expected 1 within 1e-6")


class TokenRouting:
    """One (token, layer) record: true gate probabilities and the optional
    one-layer-ahead prediction (record l forecasts layer l+1)."""

    __slots__ = ("true_scores", "predicted_scores")

    def __init__(self, true_scores, predicted_scores=None):
        t = _frozen(true_scores)
        _validate_vector(t, "true_scores")
        p = None
        if predicted_scores is not None:
            p = _frozen(predicted_scores)
            _validate_vector(p, "predicted_scores")
            if p.shape != t.shape:
                raise ShapeMismatchError("predicted_scores length differs from true_scores")
        object.__setattr__(self, "true_scores", t)
        object.__setattr__(self, "predicted_scores", p)

    def __setattr__(self, name, value):
        raise AttributeError("TokenRouting is immutable")

    def __eq__(self, other):
        if not isinstance(other, TokenRouting):
            return NotImplemented
        if not np.array_equal(self.true_scores, other.true_scores):
            return False
        if (self.predicted_scores is None) != (other.predicted_scores is None):
            return False
        return self.predicted_scores is None or np.array_equal(
            self.predicted_scores, other.predicted_scores)

    def __repr__(self):
        return f"TokenRouting(E={self.true_scores.shape[0]}, pred={self.predicted_scores is not None})"


class RoutingTrace:
    """One sequence's routing for both phases as dense read-only arrays:
    {phase}_true (T, L, E), {phase}_predicted (T, L, E) (zero where absent),
    {phase}_mask (T, L)."""

    def __init__(self, shape: ModelShape, sequence_id: str, prefill_true, decode_true,
                 prefill_predicted=None, prefill_mask=None, decode_predicted=None,
                 decode_mask=None):
        self.shape = shape
        self.sequence_id = str(sequence_id)
        l, e = shape.num_layers, shape.num_experts
        pt = np.asarray(prefill_true, dtype=np.float64)
        dt = np.asarray(decode_true, dtype=np.float64)
        for name, arr in (("prefill_true", pt), ("decode_true", dt)):
            if arr.ndim != 3 or arr.shape[1:] != (l, e):
                raise ShapeMismatchError(f"{name} must be (T, {l}, {e}), got {arr.shape}")
        if pt.shape[0] < 1:
            raise ShapeMismatchError("prefill phase must contain at least one token")

        def prep(pred, mask, n, phase):
            pred = np.zeros((n, l, e)) if pred is None else np.asarray(pred, dtype=np.float64)
            mask = np.zeros((n, l), dtype=bool) if mask is None else np.asarray(mask, dtype=bool)
            if pred.shape != (n, l, e):
                raise ShapeMismatchError(f"{phase} predicted array has wrong shape")
            if mask.shape != (n, l):
                raise ShapeMismatchError(f"{phase} prediction mask has wrong shape")
            return np.where(mask[:, :, None], pred, 0.0), mask

        pp, pm = prep(prefill_predicted, prefill_mask, pt.shape[0], "prefill")
        dp, dm = prep(decode_predicted, decode_mask, dt.shape[0], "decode")
        self.prefill_true, self.decode_true = _frozen(pt), _frozen(dt)
        self.prefill_predicted, self.decode_predicted = _frozen(pp), _frozen(dp)
        pm, dm = pm.copy(), dm.copy()
        pm.flags.writeable = dm.flags.writeable = False
        self.prefill_mask, self.decode_mask = pm, dm
        self._validate()

    @property
    def num_prefill_tokens(self) -> int:
        return self.prefill_true.shape[0]

    @property
    def num_decode_tokens(self) -> int:
        return self.decode_true.shape[0]

    def _validate(self) -> None:
        l = self.shape.num_layers
        for phase in PHASES:
            true = getattr(self, f"{phase}_true")
            pred = getattr(self, f"{phase}_predicted")
            mask = getattr(self, f"{phase}_mask")
            for name, arr, m in (("true", true, None), ("predicted", pred, mask)):
                if np.any(arr < 0) or not np.all(np.isfinite(arr)):
                    raise NormalizationError(
                        f"{phase} {name} scores contain negative/non-finite entries")
                dev = np.abs(arr.sum(axis=2) - 1.0) > SCORE_SUM_TOL
                if m is not None:
                    dev &= m
                if np.any(dev):
                    t, lay = np.argwhere(dev)[0]
                    raise NormalizationError(
                        f"{phase} token {t} layer {lay}: {name} scores do not sum to 1")
            if np.any(mask[:, l - 1]):
                raise ShapeMismatchError(f"{phase}: predicted_scores present on last layer")
        if self.num_decode_tokens and l > 1 and not np.all(self.decode_mask[:, : l - 1]):
            t, lay = np.argwhere(~self.decode_mask[:, : l - 1])[0]
            raise ShapeMismatchError(f"decode token {t} layer {lay}: predicted_scores missing")

    def token_routing(self, phase: str, token: int, layer: int) -> TokenRouting:
        true = getattr(self, f"{phase}_true")[token, layer]
        has = getattr(self, f"{phase}_mask")[token, layer]
        return TokenRouting(true, getattr(self, f"{phase}_predicted")[token, layer] if has else None)

    def token_layers(self, phase: str, token: int) -> tuple:
        return tuple(self.token_routing(phase, token, l) for l in range(self.shape.num_layers))

    def decode_token(self, token: int) -> tuple:
        return self.token_layers("decode", token)

    def prefill_token(self, token: int) -> tuple:
        return self.token_layers("prefill", token)

    def __eq__(self, other):
        if not isinstance(other, RoutingTrace):
            return NotImplemented
        return self.shape == other.shape and self.sequence_id == other.sequence_id and all(
            np.array_equal(getattr(self, a), getattr(other, a))
            for a in ("prefill_true", "decode_true", "prefill_predicted", "decode_predicted",
                      "prefill_mask", "decode_mask"))

    def __repr__(self):
        s = self.shape
        return (f"RoutingTrace({self.sequence_id!r}, L={s.num_layers}, E={s.num_experts}, "
                f"k={s.top_k}, prefill={self.num_prefill_tokens}, "
                f"decode={self.num_decode_tokens})")

    @classmethod
    def from_token_lists(cls, shape: ModelShape, sequence_id: str,
                         prefill: Sequence[Sequence[TokenRouting]],
                         decode: Sequence[Sequence[TokenRouting]] = ()) -> "RoutingTrace":
        l, e = shape.num_layers, shape.num_experts

        def pack(tokens: Iterable, phase: str):
            tokens = list(tokens)
            true = np.zeros((len(tokens), l, e))
            pred = np.zeros_like(true)
            mask = np.zeros((len(tokens), l), dtype=bool)
            for t, layers in enumerate(tokens):
                if len(layers) != l:
                    raise ShapeMismatchError(f"{phase} token {t} has {len(layers)} layers")
                for li, tr in enumerate(layers):
                    if tr.true_scores.shape[0] != e:
                        raise ShapeMismatchError(f"{phase} token {t} layer {li}: length")
                    true[t, li] = tr.true_scores
                    if tr.predicted_scores is not None:
                        pred[t, li] = tr.predicted_scores
                        mask[t, li] = True
            return true, pred, mask

        pt, pp, pm = pack(prefill, "prefill")
        dt, dp, dm = pack(decode, "decode")
        return cls(shape, sequence_id, pt, dt, pp, pm, dp, dm)


def softmax(logits: np.ndarray, axis: int = -1) -> np.ndarray:
    """Stable softmax (trace.py:479-483 semantics) for building test inputs."""
    z = logits - np.max(logits, axis=axis, keepdims=True)
    ez = np.exp(z)
    return ez / ez.sum(axis=axis, keepdims=True)
