"""`run_single` and its flat run record (moesim/experiment.py:145-211).

Two entry points share the reference's record schema, so `_run_json_obj`,
the CSV writers and any caller reading the record keep working:

* ``run_single(trace, calib_matrix, ecr, engine, cost, ...)`` -- the
  reference's call on a routing trace.  Every DECISION field is computed by
  this package (native placement / Alg. 1 / planners): placements, swaps,
  per-token plans, the simulator's counters, ``set_fidelity``,
  ``score_mass``, ``similarity_prefill_decode``, ``swap_count``.  The
  reference *prices* a timeline with a cost model; this package executes on
  the B200 instead and does not rebuild the pricing, so the
  timing fields of a trace-only call are NaN.  ``cost`` is accepted for
  signature compatibility.
* ``DaopEngine.run_single(h_prompt, decode_inputs, ...)`` (daop.py) -- the
  same flow EXECUTED: the record's timing fields are measured
  (tokens/s, per-token latency, prefill latency, hidden migration time) and
  its decision fields come from the kernels' own decisions, exported as a
  RoutingTrace (``_trace``).

`TimelineResult` mirrors moesim/simulator.py:118-167 (counts, executed,
per-token latency, tokens/s, migration_hidden_ms); ``events`` stays empty (the
engine measures, it does not build an event log).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError
from .metrics import activation_matrix, expert_counts, routing_fidelity, similarity
from .placement import allocate_for_sequence, init_from_calibration
from .policies import ENGINES, PolicyConfig, decode_counters, plan_trace_decode

CSV_SCHEMA_VERSION = 1  # experiment.py:35

COUNT_KEYS = ("migrations", "prefetches", "wasted_prefetches", "slow_executions",
              "degradations", "stale_inputs")  # simulator.py:160-167


@dataclass
class TimelineResult:
    """simulator.py:118-125, filled from measurement (or left NaN)."""

    per_token_latency_ms: list
    counts: dict
    tokens_per_second: float
    executed: list                    # per decode token, per layer, tuple of expert ids
    migration_hidden_ms: float = 0.0
    events: list = field(default_factory=list)
    busy_fraction: dict = field(default_factory=dict)

    def summary_json_obj(self) -> dict:  # simulator.py:143-157
        tps = self.tokens_per_second
        lat = self.per_token_latency_ms
        return {
            "num_tokens": len(lat),
            "total_latency_ms": float(sum(lat)),
            "mean_token_latency_ms": float(np.mean(lat)) if lat else None,
            "tokens_per_second": tps if math.isfinite(tps) else None,
            "counts": dict(self.counts),
            "busy_fraction": dict(self.busy_fraction),
            "migration_hidden_ms": self.migration_hidden_ms,
        }


def _executed(plans_per_token) -> list:
    return [[tuple(int(e) for e in p.executed_experts()) for p in plans]
            for plans in plans_per_token]


def make_record(trace, ecr: float, engine: str, seed: int, placement0, placement, swaps,
                plans_per_token, config: PolicyConfig, *, per_token_latency_ms=None,
                prefill_latency_ms=float("nan"), prefill_hidden_migration_ms=float("nan"),
                busy_fraction=None) -> dict:
    """The flat record of experiment.py:178-210 from decisions (+ timings)."""
    executed = _executed(plans_per_token)
    counts = decode_counters(plans_per_token, config)
    lat = list(per_token_latency_ms) if per_token_latency_ms is not None else []
    tps = 1e3 * len(lat) / sum(lat) if lat and sum(lat) > 0 else float("nan")
    dec = TimelineResult(lat, counts, tps, executed,
                         0.0 if math.isnan(prefill_hidden_migration_ms)
                         else prefill_hidden_migration_ms,
                         busy_fraction=dict(busy_fraction or {}))
    if trace.num_decode_tokens:
        set_f, mass = routing_fidelity(trace, executed)
        sim = similarity(activation_matrix(trace, "prefill"), activation_matrix(trace, "decode"))
    else:
        set_f = mass = sim = float("nan")
    return {
        "schema_version": CSV_SCHEMA_VERSION,
        "trace_id": trace.sequence_id,
        "ecr": ecr,
        "engine": engine,
        "seed": seed,
        "num_prefill_tokens": trace.num_prefill_tokens,
        "num_decode_tokens": trace.num_decode_tokens,
        "tokens_per_second": tps,
        "mean_token_latency_ms": float(np.mean(lat)) if lat else float("nan"),
        "total_latency_ms": float(sum(lat)) if lat else float("nan"),
        **{k: counts[k] for k in COUNT_KEYS},
        "set_fidelity": set_f,
        "score_mass": mass,
        "prefill_latency_ms": prefill_latency_ms,
        "prefill_hidden_migration_ms": prefill_hidden_migration_ms,
        "swap_count": len(swaps),
        "similarity_prefill_decode": sim,
        "_decode_result": dec,
        "_prefill_result": None,
        "_placement_initial": placement0,
        "_placement_final": placement,
        "_swaps": list(swaps),
    }


def run_single(trace, calib_matrix, ecr: float, engine: str, cost=None,
               prediction_start_layer: int = 4, graceful_degradation: bool = True,
               seed: int = 0) -> dict:
    """experiment.py:145-211 on a routing trace: init_from_calibration ->
    (daop only) allocate_for_sequence(expert_counts(prefill)) -> per-token
    plans at the post-swap placement -> counters, fidelity, similarity."""
    if engine not in ENGINES:
        raise ConfigError(f"unknown engine {engine!r}")
    shape = trace.shape
    placement0 = init_from_calibration(calib_matrix, ecr, shape)
    if engine == "daop":
        placement, swaps = allocate_for_sequence(placement0, expert_counts(trace, "prefill"))
    else:
        placement, swaps = placement0, []
    config = PolicyConfig(engine=engine, prediction_start_layer=prediction_start_layer,
                          graceful_degradation=graceful_degradation)
    plans = plan_trace_decode(trace, placement, config) if trace.num_decode_tokens else []
    return make_record(trace, ecr, engine, seed, placement0, placement, swaps, plans, config)
