"""Routing data types -- the parity interchange format.

Same public surface as moesim/trace.py (ModelShape :35-53, presets :57-58,
TokenRouting :80-110, RoutingTrace :129-322, SCORE_SUM_TOL :30).  The B200
engine *produces* these from its fused router (true gate of every layer plus
the next-layer prediction), so an engine run can be handed unchanged to the
reference's own analysis functions, and the reference's decisions on it can be
compared with the GPU's with ``==``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .errors import NormalizationError, ShapeMismatchError, TraceParseError

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


_PRESETS = {"mixtral": MIXTRAL_SHAPE, "phi": PHI_SHAPE}


def parse_shape(text: str) -> ModelShape:
    """'mixtral' / 'phi' / 'LxExK' (moesim/trace.py:63-77)."""
    key = text.strip().lower()
    if key in _PRESETS:
        return _PRESETS[key]
    parts = key.split("x")
    if len(parts) != 3:
        raise ShapeMismatchError(f"shape must be 'mixtral', 'phi' or 'LxExK', got {text!r}")
    try:
        l, e, k = (int(p) for p in parts)
    except ValueError:
        raise ShapeMismatchError(f"non-integer component in shape {text!r}") from None
    return ModelShape(l, e, k)


# -- JSON-Lines trace files (moesim/trace.py:325-476) ------------------------
#
# The on-disk boundary to the reference's analysis tools: a trace the B200
# engine exports is byte-identical to what moesim's save_trace would write for
# the same arrays, so `moesim stats / simulate / sweep` read it unchanged, and
# load_trace accepts every file moesim writes with moesim's error semantics.

_HEADER_KEYS = {"format_version", "sequence_id", "L", "E", "k", "num_prefill_tokens",
                "num_decode_tokens"}


def save_trace(trace: RoutingTrace, path) -> None:
    """Write ``trace`` in the canonical JSONL format (moesim/trace.py:332-362).
    Token records are formatted natively (daop_trace_format_phase, "%.17g")."""
    import ctypes

    from . import _lib

    s = trace.shape
    header = {"format_version": 1, "sequence_id": trace.sequence_id, "L": s.num_layers,
              "E": s.num_experts, "k": s.top_k, "num_prefill_tokens": trace.num_prefill_tokens,
              "num_decode_tokens": trace.num_decode_tokens}
    body = []
    for ph, phase in enumerate(PHASES):
        true = np.ascontiguousarray(getattr(trace, f"{phase}_true"), dtype=np.float64)
        pred = np.ascontiguousarray(getattr(trace, f"{phase}_predicted"), dtype=np.float64)
        mask = np.ascontiguousarray(getattr(trace, f"{phase}_mask"), dtype=np.uint8)
        n = ctypes.c_int64(0)
        args = (true.ctypes.data, pred.ctypes.data, mask.ctypes.data, true.shape[0],
                s.num_layers, s.num_experts, ph)
        _lib.call("daop_trace_format_phase", *args, None, 0, ctypes.addressof(n))
        buf = ctypes.create_string_buffer(max(1, n.value))
        _lib.call("daop_trace_format_phase", *args, buf, n.value, ctypes.addressof(n))
        body.append(buf.raw[: n.value])
    with open(path, "wb") as fh:
        fh.write(json.dumps(header, sort_keys=True).encode("utf-8") + b"\n")
        for b in body:
            fh.write(b)


def _check_line_scores(vec, path, line_no, token, layer, name) -> None:
    # moesim/trace.py:465-476
    if np.any(vec < 0) or not np.all(np.isfinite(vec)):
        raise NormalizationError(f"{path}: line {line_no}: token {token} layer {layer}: "
                                 f"{name} has negative or non-finite entries")
    s = float(vec.sum())
    if abs(s - 1.0) > SCORE_SUM_TOL:
        raise NormalizationError(f"{path}: line {line_no}: token {token} layer {layer}: "
                                 f"{name} sum deviates from 1 by {abs(s - 1.0):.3g}")


def _layer_checked(entry, e, path, line_no, idx, li):
    """The per-layer rules of moesim/trace.py:430-456, in their order."""
    ts = entry.get("true_scores") if isinstance(entry, dict) else None
    if not isinstance(ts, list) or len(ts) != e:
        raise ShapeMismatchError(
            f"{path}: line {line_no}: token {idx} layer {li}: true_scores length "
            f"{len(ts) if isinstance(ts, list) else '?'}, expected {e}")
    vec = np.array(ts, dtype=np.float64)
    _check_line_scores(vec, path, line_no, idx, li, "true_scores")
    ps = entry.get("predicted_scores")
    pvec = None
    if ps is not None:
        if not isinstance(ps, list) or len(ps) != e:
            raise ShapeMismatchError(f"{path}: line {line_no}: token {idx} layer {li}: "
                                     f"predicted_scores length mismatch, expected {e}")
        pvec = np.array(ps, dtype=np.float64)
        _check_line_scores(pvec, path, line_no, idx, li, "predicted_scores")
    return vec, pvec


def load_trace(path) -> RoutingTrace:
    """Parse and validate a trace file (moesim/trace.py:376-462): same
    accepted inputs, same error classes and messages.  Each token record is
    validated as one (L, E) block; the per-layer walk runs only to name the
    first offending layer."""
    with open(path, "r", encoding="utf-8") as fh:
        raw = fh.read().splitlines()
    if not raw:
        raise TraceParseError(f"{path}: empty file")

    def parse_line(num, text):
        try:
            return json.loads(text)
        except json.JSONDecodeError as exc:
            raise TraceParseError(f"{path}: line {num}: {exc}") from None

    header = parse_line(1, raw[0])
    if not isinstance(header, dict) or not _HEADER_KEYS.issubset(header):
        raise TraceParseError(f"{path}: line 1: malformed header record")
    if header["format_version"] != 1:
        raise TraceParseError(f"{path}: unsupported format_version {header['format_version']!r}")
    shape = ModelShape(int(header["L"]), int(header["E"]), int(header["k"]))
    n_prefill, n_decode = int(header["num_prefill_tokens"]), int(header["num_decode_tokens"])
    body = [ln for ln in raw[1:] if ln.strip()]
    if len(body) != n_prefill + n_decode:
        raise TraceParseError(
            f"{path}: expected {n_prefill + n_decode} token records, found {len(body)}")
    l, e = shape.num_layers, shape.num_experts
    arrays = {ph: (np.zeros((n, l, e)), np.zeros((n, l, e)), np.zeros((n, l), dtype=bool))
              for ph, n in (("prefill", n_prefill), ("decode", n_decode))}
    counters = {"prefill": 0, "decode": 0}
    for offset, text in enumerate(body):
        line_no = offset + 2
        rec = parse_line(line_no, text)
        if not isinstance(rec, dict) or "phase" not in rec or "layers" not in rec:
            raise TraceParseError(f"{path}: line {line_no}: malformed token record")
        phase = rec["phase"]
        if phase not in PHASES:
            raise TraceParseError(f"{path}: line {line_no}: unknown phase {phase!r}")
        idx = rec.get("token_index")
        if idx != counters[phase]:
            raise TraceParseError(
                f"{path}: line {line_no}: token_index {idx!r} out of order "
                f"(expected {counters[phase]} for phase {phase})")
        layers = rec["layers"]
        if not isinstance(layers, list) or len(layers) != l:
            raise ShapeMismatchError(
                f"{path}: line {line_no}: token {idx} ({phase}) has "
                f"{len(layers) if isinstance(layers, list) else '?'} layers, expected {l}")
        true, pred, mask = arrays[phase]
        ok = False
        try:  # fast path: the whole token as one block
            ts = np.array([ent["true_scores"] for ent in layers], dtype=np.float64)
            pm = np.array([ent["predicted_scores"] is not None for ent in layers])
            ps = np.array([ent["predicted_scores"] if m else [0.0] * e
                           for ent, m in zip(layers, pm)], dtype=np.float64)
            if ts.shape == (l, e) and ps.shape == (l, e):
                good = np.all(ts >= 0) and np.all(np.isfinite(ts)) and np.all(
                    np.abs(ts.sum(axis=1) - 1.0) <= SCORE_SUM_TOL)
                pv = ps[pm]
                good = good and np.all(pv >= 0) and np.all(np.isfinite(pv)) and np.all(
                    np.abs(pv.sum(axis=1) - 1.0) <= SCORE_SUM_TOL)
                ok = bool(good)
        except (TypeError, ValueError, KeyError):
            ok = False
        if ok:
            true[idx], pred[idx], mask[idx] = ts, ps, pm
        else:  # the reference's sequential walk raises the first error
            for li, entry in enumerate(layers):
                vec, pvec = _layer_checked(entry, e, path, line_no, idx, li)
                true[idx, li] = vec
                if pvec is not None:
                    pred[idx, li], mask[idx, li] = pvec, True
        counters[phase] += 1
    pt, pp, pm_ = arrays["prefill"]
    dt, dp, dm = arrays["decode"]
    return RoutingTrace(shape, header["sequence_id"], pt, dt, pp, pm_, dp, dm)
