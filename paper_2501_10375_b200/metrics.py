"""Activation counter, calibration matrix and prediction reports.

Same surface as the hot-path part of moesim/metrics.py: ActivationMatrix
:25-52, expert_counts :64-71 (the per-sequence activation counter),
activation_matrix :74-82, prediction_accuracy :120-143, routing_fidelity
:177-215, plus experiment.pooled_decode_probabilities :132-142.  Counting and
top-k run on the device operator table (kernels.py); in the engine the
counter is fused into the router kernel's epilogue instead (hist[b, l, e]).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import kernels
from .errors import (ConfigError, EmptyPhaseError, PredictionMissingError,
                     ShapeMismatchError)


@dataclass(frozen=True)
class ActivationMatrix:
    """L x E activation probabilities of one phase (rows sum to k)."""

    values: np.ndarray
    phase: str
    token_count: int

    def __post_init__(self):
        arr = np.ascontiguousarray(self.values, dtype=np.float64)
        if arr.ndim != 2:
            raise ShapeMismatchError("activation matrix must be 2-D")
        if np.any(arr < 0) or not np.all(np.isfinite(arr)):
            raise ShapeMismatchError("activation matrix entries must be >= 0")
        arr.flags.writeable = False
        object.__setattr__(self, "values", arr)

    @property
    def num_layers(self) -> int:
        return self.values.shape[0]

    @property
    def num_experts(self) -> int:
        return self.values.shape[1]


def _phase_topk(trace, phase: str) -> np.ndarray:
    true = getattr(trace, f"{phase}_true")
    s = trace.shape
    return kernels.topk_rows(true.reshape(-1, s.num_experts), s.top_k).reshape(
        true.shape[0], s.num_layers, s.top_k)


def expert_counts(trace, phase: str) -> np.ndarray:
    """(L, E) int64 token counts per expert of the phase's true top-k."""
    if getattr(trace, f"{phase}_true").shape[0] == 0:
        raise EmptyPhaseError(f"trace has no {phase} tokens")
    return kernels.activation_counts(_phase_topk(trace, phase),
                                     trace.shape.num_experts).astype(np.int64)


def activation_matrix(trace, phase: str) -> ActivationMatrix:
    n = getattr(trace, f"{phase}_true").shape[0]
    if n == 0:
        raise EmptyPhaseError(f"trace has no {phase} tokens")
    counts = kernels.activation_counts(_phase_topk(trace, phase), trace.shape.num_experts)
    return ActivationMatrix(counts / n, phase, n)


def prediction_accuracy(trace) -> np.ndarray:
    """Entry l: mean |topk(prediction for l) ∩ topk(true l)| / k; entry 0 NaN."""
    s = trace.shape
    n = trace.num_decode_tokens
    if n == 0:
        raise EmptyPhaseError("trace has no decode tokens")
    out = np.full(s.num_layers, np.nan)
    true_top = _phase_topk(trace, "decode")
    for layer in range(1, s.num_layers):
        if not np.all(trace.decode_mask[:, layer - 1]):
            t = int(np.argwhere(~trace.decode_mask[:, layer - 1])[0][0])
            raise PredictionMissingError(f"decode token {t} lacks a prediction for layer {layer}")
        pred_top = kernels.topk_rows(trace.decode_predicted[:, layer - 1, :], s.top_k)
        out[layer] = kernels.pair_overlap(pred_top, true_top[:, layer, :]).mean() / s.top_k
    return out


def mean_prediction_accuracy(trace) -> float:
    acc = prediction_accuracy(trace)
    vals = acc[~np.isnan(acc)]
    return float(vals.mean()) if vals.size else float("nan")


def routing_fidelity(trace, executed) -> tuple:
    """(set_fidelity, score_mass) of executed expert sets vs the true gates."""
    s = trace.shape
    n = trace.num_decode_tokens
    if len(executed) != n:
        raise ShapeMismatchError(f"executed covers {len(executed)} tokens, trace has {n}")
    true_top = _phase_topk(trace, "decode")
    overlaps, masses = [], []
    for t in range(n):
        if len(executed[t]) != s.num_layers:
            raise ShapeMismatchError(f"token {t}: executed covers {len(executed[t])} layers")
        for l in range(s.num_layers):
            ex = tuple(executed[t][l])
            if len(ex) != s.top_k or len(set(ex)) != s.top_k:
                raise ShapeMismatchError(f"token {t} layer {l}: executed set {ex}")
            tt = set(int(x) for x in true_top[t, l])
            overlaps.append(len(tt.intersection(ex)) / s.top_k)
            scores = trace.decode_true[t, l]
            masses.append(float(scores[list(ex)].sum()) / float(scores[true_top[t, l]].sum()))
    return float(np.mean(overlaps)), float(np.mean(masses))


def pooled_decode_probabilities(traces) -> np.ndarray:
    """Token-pooled decode activation probabilities (experiment.py:132-142)."""
    total, tokens = None, 0
    for tr in traces:
        c = expert_counts(tr, "decode")
        total = c if total is None else total + c
        tokens += tr.num_decode_tokens
    if tokens == 0:
        raise ConfigError("calibration traces contain no decode tokens")
    return total / tokens


def _as_matrix(m) -> np.ndarray:
    if isinstance(m, ActivationMatrix):
        return m.values
    arr = np.asarray(m, dtype=np.float64)
    if arr.ndim != 2:
        raise ShapeMismatchError("similarity expects 2-D matrices")
    return arr


def row_cosines(p, d) -> tuple:
    """Per-layer cosine of two L x E matrices plus the degenerate-row mask
    (moesim/metrics.py:94-111): a zero row on either side scores 0."""
    pv, dv = _as_matrix(p), _as_matrix(d)
    if pv.shape != dv.shape:
        raise ShapeMismatchError(f"matrix dimensions differ: {pv.shape} vs {dv.shape}")
    num = (pv * dv).sum(axis=1)
    n_p, n_d = np.linalg.norm(pv, axis=1), np.linalg.norm(dv, axis=1)
    degenerate = (n_p == 0.0) | (n_d == 0.0)
    cows = np.where(degenerate, 0.0, num / np.where(degenerate, 1.0, n_p * n_d))
    return cows, degenerate


def similarity(p, d) -> float:
    """Eq. 1 of the paper: mean over layers of the row cosines
    (moesim/metrics.py:114-117)."""
    return float(row_cosines(p, d)[0].mean())
