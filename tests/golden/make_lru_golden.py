"""Golden vectors for the ondemand / prefetch baseline planners (LRU caches),
produced by running the UNMODIFIED reference (build container only):

    python tests/golden/make_lru_golden.py

Records, for random shapes, placements and traces, moesim's own
``plan_trace_decode`` output for engines "ondemand" and "prefetch"
(moesim/policies.py:103-245; cache state replayed across tokens) and the
decode counters of ``simulate_decode`` (simulator.py:297-335: migrations,
prefetches, wasted_prefetches), plus single-token PredictionMissingError cases.
Output: ``tests/golden/lru_plans.json``.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import moesim  # noqa: E402
from moesim import (ExpertPlacement, ModelShape, PolicyConfig, RoutingTrace,  # noqa: E402
                    TokenRouting, plan_trace_decode, simulate_decode)
from moesim.policies import make_planner  # noqa: E402

OUT = Path(__file__).with_name("lru_plans.json")


def f32r(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rand_rows(rng, n, e, tie_frac):
    s = rng.random((n, e)) + 1e-3
    s = s / s.sum(axis=1, keepdims=True)
    m = rng.random((n, e)) < tie_frac
    for i in range(n):
        if m[i].sum() >= 2:
            s[i, m[i]] = s[i, m[i]].mean()
    s = f32r(s)
    return s / s.sum(axis=1, keepdims=True)


def plan_obj(p):
    return {"executed": [[x.expert, x.device, x.input_source, x.precalc] for x in p.executed],
            "migrations": list(p.migrations), "prefetch_issues": list(p.prefetch_issues)}


def main():
    rng = np.random.default_rng(20251017)
    cases = []
    for i in range(40):
        l = int(rng.integers(1, 9))
        e = int(rng.integers(2, 11))
        k = int(rng.integers(1, min(4, e) + 1))
        shape = ModelShape(l, e, k)
        # placement: random per-layer sets, sizes 1..E (capacity = size)
        sets = [frozenset(int(x) for x in rng.choice(e, size=int(rng.integers(1, e + 1)),
                                                      replace=False)) for _ in range(l)]
        budget = sum(len(s) for s in sets)
        placement = ExpertPlacement(shape, sets, budget)
        n_dec = int(rng.integers(1, 9))
        tie = float(rng.choice([0.0, 0.3]))
        pt = rand_rows(rng, 2 * l, e, tie).reshape(2, l, e)
        dt = rand_rows(rng, n_dec * l, e, tie).reshape(n_dec, l, e)
        dp = np.zeros((n_dec, l, e))
        dm = np.zeros((n_dec, l), dtype=bool)
        if l > 1:
            # predictions: often close to the next layer's truth (so prefetch hits)
            nxt = dt[:, 1:, :]
            noise = rand_rows(rng, n_dec * (l - 1), e, 0.0).reshape(n_dec, l - 1, e)
            mix = float(rng.choice([0.0, 0.5, 0.9]))
            pr = f32r(mix * nxt + (1 - mix) * noise)
            dp[:, : l - 1] = pr / pr.sum(axis=2, keepdims=True)
            dm[:, : l - 1] = True
        tr = RoutingTrace(shape, f"c{i}", pt, dt, decode_predicted=dp, decode_mask=dm)
        start = int(rng.integers(1, l + 2))
        obj = {"L": l, "E": e, "k": k, "start": start, "sets": [sorted(s) for s in sets],
               "decode_true": dt.tolist(), "decode_pred": dp.tolist(),
               "decode_mask": dm.tolist(), "prefill_true": pt.tolist()}
        for engine in ("ondemand", "prefetch"):
            cfg = PolicyConfig(engine, prediction_start_layer=start)
            plans = plan_trace_decode(tr, placement, cfg)
            res = simulate_decode(tr, placement, cfg)
            obj[engine] = {"plans": [[plan_obj(p) for p in tok] for tok in plans],
                           "counts": {c: int(res.counts[c]) for c in
                                      ("migrations", "prefetches", "wasted_prefetches",
                                       "slow_executions", "degradations", "stale_inputs")}}
        cases.append(obj)

    # single token, prefetch needs a prediction that is missing
    missing = []
    for i in range(6):
        l, e, k = 4, 6, 2
        shape = ModelShape(l, e, k)
        sets = [frozenset({0, 1, 2})] * l
        placement = ExpertPlacement(shape, sets, 3 * l)
        rows = rand_rows(rng, l, e, 0.0)
        gap = int(rng.integers(0, l - 1))  # layer whose record lacks its prediction
        toks = [TokenRouting(rows[j], None if (j == gap or j == l - 1) else rows[(j + 1) % l])
                for j in range(l)]
        start = int(rng.integers(1, l))
        planner = make_planner(placement, PolicyConfig("prefetch", prediction_start_layer=start))
        try:
            planner.plan_token(toks)
            err = None
        except moesim.MoesimError as exc:
            err = type(exc).__name__
        missing.append({"L": l, "E": e, "k": k, "start": start, "gap": gap,
                        "rows": rows.tolist(), "sets": [sorted(s) for s in sets], "error": err})
    OUT.write_text(json.dumps({"reference": "moesim", "cases": cases, "missing": missing}))
    print("wrote", OUT, len(cases), "cases")


if __name__ == "__main__":
    main()
