"""Per-token execution plans for all four engines.

Same surface as moesim/policies.py: ENGINES :32, PREDICTION_START_LAYER_DEFAULT
:34, PolicyConfig :37-47, ExecutedExpert / Degradation / LayerPlan :50-100,
OnDemandPlanner :173-194 / PrefetchPlanner :197-245 (LRU caches :103-140),
FiddlerPlanner :248-261, degrade_selection :264-296, DaopPlanner :299-336,
make_planner :339-348, plan_token_* :359-376, plan_trace_decode :379-387.

The planning executes natively: daop_plan_token_f64 (fiddler / daop; the
identical device routine runs inside the decode launch on the router's
float32 probabilities -- csrc/decide.cuh) and daop_lru_plan_layer (the LRU
baselines, one layer per call, cache state owned by the planner object here
so the GPU engine can drive it layer by layer and move HBM slots with it).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .errors import ConfigError, ShapeMismatchError
from .placement import ExpertPlacement

ENGINES = ("ondemand", "prefetch", "fiddler", "daop")
NATIVE_ENGINES = {"fiddler": 2, "daop": 3}
LRU_ENGINES = {"ondemand": 0, "prefetch": 1}
PREDICTION_START_LAYER_DEFAULT = 4


@dataclass(frozen=True)
class PolicyConfig:
    engine: str
    prediction_start_layer: int = PREDICTION_START_LAYER_DEFAULT
    graceful_degradation: bool = True

    def __post_init__(self):
        if self.engine not in ENGINES:
            raise ConfigError(f"unknown engine {self.engine!r}; pick from {ENGINES}")
        if self.prediction_start_layer < 1:
            raise ConfigError("prediction_start_layer must be >= 1")


@dataclass(frozen=True)
class ExecutedExpert:
    expert: int
    device: str  # fast | slow
    input_source: str  # current | stale
    precalc: bool = False


@dataclass(frozen=True)
class Degradation:
    dropped_expert: int
    dropped_score: float
    substitute_expert: int
    substitute_score: float


@dataclass(frozen=True)
class LayerPlan:
    layer: int
    executed: tuple
    migrations: tuple = ()
    prefetch_issues: tuple = ()
    degraded: tuple = ()

    def executed_experts(self) -> tuple:
        return tuple(x.expert for x in self.executed)

    def to_json_obj(self) -> dict:
        return {
            "layer": self.layer,
            "executed": [{"expert": x.expert, "device": x.device,
                          "input_source": x.input_source, "precalc": x.precalc}
                         for x in self.executed],
            "migrations": list(self.migrations),
            "prefetch_issues": list(self.prefetch_issues),
            "degraded": [{"dropped_expert": d.dropped_expert, "dropped_score": d.dropped_score,
                          "substitute_expert": d.substitute_expert,
                          "substitute_score": d.substitute_score} for d in self.degraded],
        }


def degrade_selection(scores, selection, fast_experts):
    """Swap surplus slow picks for the best cached alternatives (native)."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    e = s.shape[0]
    sel = np.ascontiguousarray(list(selection), dtype=np.int32)
    k = sel.shape[0]
    fast = np.zeros(e, dtype=np.uint8)
    fast[list(fast_experts)] = 1
    drop = np.zeros(max(k, 1), dtype=np.int32)
    sub = np.zeros(max(k, 1), dtype=np.int32)
    nd = np.zeros(1, dtype=np.int32)
    _lib.call("daop_degrade_f64", _lib.ptr(s), e, _lib.ptr(sel), k, _lib.ptr(fast),
              _lib.ptr(drop), _lib.ptr(sub), _lib.ptr(nd))
    deg = tuple(Degradation(int(drop[i]), float(s[drop[i]]), int(sub[i]), float(s[sub[i]]))
                for i in range(int(nd[0])))
    return [int(x) for x in sel], deg


def _token_arrays(token: Sequence, num_experts: int):
    true = np.stack([tr.true_scores for tr in token])
    if true.shape[1] != num_experts:
        raise ShapeMismatchError(
            f"token vectors have length {true.shape[1]}, expected {num_experts}")
    pred = np.zeros_like(true)
    mask = np.zeros(len(token), dtype=np.uint8)
    for l, tr in enumerate(token):
        if tr.predicted_scores is not None:
            pred[l] = tr.predicted_scores
            mask[l] = 1
    return np.ascontiguousarray(true), pred, mask


class _NativePlanner:
    def __init__(self, placement: ExpertPlacement, config: PolicyConfig):
        if config.engine not in NATIVE_ENGINES:
            raise ConfigError(
                f"engine {config.engine!r} is a baseline outside the DAOP hot path "
                "(SURVEY.md §8a a7); only 'daop' and 'fiddler' are built")
        self.placement = placement
        self.config = config
        self.shape = placement.shape
        self._mask = placement.mask()

    def plan_token(self, token: Sequence) -> list:
        s = self.shape
        l, e, k = s.num_layers, s.num_experts, s.top_k
        true, pred, pmask = _token_arrays(token, e)
        if true.shape[0] != l:
            raise ShapeMismatchError(f"token covers {true.shape[0]} layers, expected {l}")
        sel = np.zeros((l, k), dtype=np.int32)
        fast = np.zeros((l, k), dtype=np.uint8)
        drop = np.zeros((l, k), dtype=np.int32)
        sub = np.zeros((l, k), dtype=np.int32)
        nd = np.zeros(l, dtype=np.int32)
        _lib.call("daop_plan_token_f64", _lib.ptr(true), _lib.ptr(pred), _lib.ptr(pmask),
                  _lib.ptr(self._mask), l, e, k, self.config.prediction_start_layer,
                  NATIVE_ENGINES[self.config.engine], int(self.config.graceful_degradation),
                  _lib.ptr(sel), _lib.ptr(fast), _lib.ptr(drop), _lib.ptr(sub), _lib.ptr(nd))
        return plans_from_arrays(sel, fast, drop, sub, nd, pred, self.config)


_EXECUTED = {}  # (expert, kind) -> ExecutedExpert; the values are frozen, so shared


def _executed(e: int, kind: int) -> ExecutedExpert:
    """kind 0: fast / current, 1: slow / stale / precalc, 2: slow / current."""
    x = _EXECUTED.get((e, kind))
    if x is None:
        x = (ExecutedExpert(e, "fast", "current"), ExecutedExpert(e, "slow", "stale", precalc=True),
             ExecutedExpert(e, "slow", "current"))[kind]
        _EXECUTED[(e, kind)] = x
    return x


def plans_from_arrays(sel, fast, drop, sub, nd, pred_scores, config: PolicyConfig) -> list:
    """Build LayerPlans from the native planner's arrays (host or device).

    pred_scores (L, E): predictions carried on each layer (row l-1 scores the
    degradation at layer l).  Runs once per decode token, so the arrays are
    read as Python lists and the (immutable) ExecutedExpert values are shared."""
    daop = config.engine == "daop"
    start = config.prediction_start_layer
    sel_l, fast_l, nd_l = sel.tolist(), fast.tolist(), nd.tolist()
    plans = []
    for l, (row, frow) in enumerate(zip(sel_l, fast_l)):
        slow_kind = 1 if daop and l >= start else 2
        executed = tuple(_executed(e, 0 if f else slow_kind) for e, f in zip(row, frow))
        deg = ()
        if nd_l[l]:
            sc = pred_scores[l - 1]
            deg = tuple(Degradation(int(drop[l, i]), float(sc[drop[l, i]]), int(sub[l, i]),
                                    float(sc[sub[l, i]])) for i in range(nd_l[l]))
        plans.append(LayerPlan(layer=l, executed=executed, degraded=deg))
    return plans


class FiddlerPlanner(_NativePlanner):
    pass


class DaopPlanner(_NativePlanner):
    pass


@dataclass
class LruLayerDecision:
    """One layer of an LRU plan with the slot-level detail the GPU engine
    needs: which expert each migration / prefetch evicted (-1: none)."""
    selection: tuple
    migrations: tuple
    migration_evictions: tuple
    prefetch_issues: tuple
    prefetch_evictions: tuple


class _LruPlanner:
    """Per-layer LRU caches seeded from the placement (policies.py:130-140),
    state persisting across tokens like the reference's planner object."""

    def __init__(self, placement: ExpertPlacement, config: PolicyConfig):
        self.placement = placement
        self.config = config
        self.shape = placement.shape
        s = self.shape
        self.last_use = np.full((s.num_layers, s.num_experts), -1, dtype=np.int64)
        for l, members in enumerate(placement.on_fast):
            for e in members:
                self.last_use[l, e] = 0
        self.capacity = np.array([len(m) for m in placement.on_fast], dtype=np.int32)
        self.step = np.zeros(1, dtype=np.int64)
        k = s.top_k
        self._buf = [np.zeros(k, dtype=np.int32) for _ in range(5)]
        self._n = np.zeros(2, dtype=np.int32)

    def members(self, layer: int) -> tuple:
        return tuple(int(e) for e in np.nonzero(self.last_use[layer] >= 0)[0])

    def plan_layer(self, layer: int, true_row, pred_row=None) -> LruLayerDecision:
        s = self.shape
        tr = np.ascontiguousarray(true_row, dtype=np.float64)
        pr = None if pred_row is None else np.ascontiguousarray(pred_row, dtype=np.float64)
        sel, mig, mev, pf, pev = self._buf
        _lib.call("daop_lru_plan_layer", layer, s.num_layers, s.num_experts, s.top_k,
                  LRU_ENGINES[self.config.engine], self.config.prediction_start_layer,
                  _lib.ptr(tr), 0 if pr is None else _lib.ptr(pr), _lib.ptr(self.last_use),
                  _lib.ptr(self.capacity), _lib.ptr(self.step), _lib.ptr(sel), _lib.ptr(mig),
                  _lib.ptr(mev), self._n.ctypes.data, _lib.ptr(pf), _lib.ptr(pev),
                  self._n.ctypes.data + 4)
        nm, npf = int(self._n[0]), int(self._n[1])
        t = lambda a, n: tuple(int(x) for x in a[:n])  # noqa: E731
        return LruLayerDecision(t(sel, s.top_k), t(mig, nm), t(mev, nm), t(pf, npf), t(pev, npf))

    def plan_token(self, token: Sequence) -> list:
        s = self.shape
        true, pred, pmask = _token_arrays(token, s.num_experts)
        if true.shape[0] != s.num_layers:
            raise ShapeMismatchError(
                f"token covers {true.shape[0]} layers, expected {s.num_layers}")
        plans = []
        for l in range(s.num_layers):
            dec = self.plan_layer(l, true[l], pred[l] if pmask[l] else None)
            plans.append(LayerPlan(
                layer=l, executed=tuple(ExecutedExpert(e, "fast", "current")
                                        for e in dec.selection),
                migrations=dec.migrations, prefetch_issues=dec.prefetch_issues))
        return plans


class OnDemandPlanner(_LruPlanner):
    pass


class PrefetchPlanner(_LruPlanner):
    pass


_PLANNERS = {"ondemand": OnDemandPlanner, "prefetch": PrefetchPlanner,
             "fiddler": FiddlerPlanner, "daop": DaopPlanner}


def make_planner(placement: ExpertPlacement, config: PolicyConfig):
    return _PLANNERS[config.engine](placement, config)


def _single(engine, token, placement, config):
    cfg = config or PolicyConfig(engine=engine)
    if cfg.engine != engine:
        cfg = PolicyConfig(engine, cfg.prediction_start_layer, cfg.graceful_degradation)
    return make_planner(placement, cfg).plan_token(token)


def plan_token_ondemand(token, placement, config=None) -> list:
    """Single-token on-demand plan from a fresh cache snapshot."""
    return _single("ondemand", token, placement, config)


def plan_token_prefetch(token, placement, config=None) -> list:
    return _single("prefetch", token, placement, config)


def plan_token_fiddler(token, placement, config=None) -> list:
    return _single("fiddler", token, placement, config)


def plan_token_daop(token, placement, config=None) -> list:
    return _single("daop", token, placement, config)


def plan_trace_decode(trace, placement: ExpertPlacement, config: PolicyConfig) -> list:
    planner = make_planner(placement, config)
    return [planner.plan_token(trace.decode_token(t)) for t in range(trace.num_decode_tokens)]


def decode_counters(plans_per_token, config: PolicyConfig) -> dict:
    """The simulator's counter semantics (simulator.py:160-167,297-389):
    slow_executions counts current slow picks plus pre-calculated picks
    (dispatched at layer l for layer l+1 when the prediction gate runs),
    stale_inputs the pre-calculated picks, degradations the substitutions,
    migrations the demand migrations, prefetches the early migrations for
    layer l+1 (wasted when l+1 does not execute the expert)."""
    c = {"migrations": 0, "prefetches": 0, "wasted_prefetches": 0,
         "slow_executions": 0, "degradations": 0, "stale_inputs": 0}
    daop = config.engine == "daop"
    start = config.prediction_start_layer
    for plans in plans_per_token:
        n = len(plans)
        for l, p in enumerate(plans):
            c["migrations"] += len(p.migrations)
            for e in p.prefetch_issues:
                c["prefetches"] += 1
                if e not in plans[l + 1].executed_experts():
                    c["wasted_prefetches"] += 1
            c["slow_executions"] += sum(1 for x in p.executed if x.device == "slow" and not x.precalc)
            if daop and l + 1 < n and l + 1 >= start:
                pre = sum(1 for x in plans[l + 1].executed if x.precalc)
                c["slow_executions"] += pre
                c["stale_inputs"] += pre
            c["degradations"] += len(p.degraded)
    return c
