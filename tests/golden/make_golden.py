"""Generate golden decision vectors by running the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``moesim`` from /root/reference/pkg/src (read-only; numba's cache
is redirected to /tmp and bytecode writing is disabled so nothing is written
into the reference tree) and records inputs + outputs of every decision
function on the hot path into
``tests/golden/decisions.json``.  The committed JSON is what the CPU and GPU
parity tests compare against; floats are serialised with repr() so they
round-trip exactly.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
import moesim  # noqa: E402
from moesim import _kernels  # noqa: E402
from moesim import (  # noqa: E402
    ExpertPlacement, GeneratorConfig, ModelShape, PolicyConfig, RoutingTrace,
    allocate_for_sequence, default_cost_model, degrade_selection,
    expert_counts, generate_trace, init_from_calibration, make_planner,
    prediction_accuracy,
)
from moesim.experiment import pooled_decode_probabilities, run_single  # noqa: E402

OUT = Path(__file__).with_name("decisions.json")


def f32r(a):
    """Round to float32 and back: what the GPU router exports."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rand_scores(rng, n, e, tie_frac=0.25, fp32=True):
    s = rng.random((n, e)) + 1e-3
    s = s / s.sum(axis=1, keepdims=True)
    if tie_frac:
        m = rng.random((n, e)) < tie_frac
        for i in range(n):
            if m[i].sum() >= 2:
                s[i, m[i]] = s[i, m[i]].mean()
    return f32r(s) if fp32 else s


def plan_to_obj(plan):
    return {
        "layer": plan.layer,
        "executed": [[x.expert, x.device, x.input_source, x.precalc]
                     for x in plan.executed],
        "degraded": [[d.dropped_expert, d.dropped_score, d.substitute_expert,
                      d.substitute_score] for d in plan.degraded],
    }


def main():
    rng = np.random.default_rng(20250117)
    g = {"reference": "moesim " + getattr(moesim, "__version__", "?"),
         "backend": _kernels.BACKEND}

    # a1 topk_rows ------------------------------------------------------
    cases = []
    for _ in range(120):
        n = int(rng.integers(1, 24))
        e = int(rng.integers(2, 17))
        k = int(rng.integers(1, e + 1))
        s = rand_scores(rng, n, e, tie_frac=float(rng.choice([0.0, 0.3, 0.6])))
        if rng.random() < 0.2:
            s = np.round(s, 2)
        cases.append({"scores": s.tolist(), "k": k,
                      "out": _kernels.topk_rows(s, k).tolist()})
    cases.append({"scores": [[0.25, 0.25, 0.25, 0.25]], "k": 2, "out": [[0, 1]]})
    z = np.array([[0.0, -0.0, 0.5, 0.5]])
    cases.append({"scores": z.tolist(), "k": 4, "out": _kernels.topk_rows(z, 4).tolist()})
    g["topk_rows"] = cases

    # a3 activation_counts / expert_counts ---------------------------------
    cases = []
    for _ in range(40):
        t, l, e = int(rng.integers(1, 30)), int(rng.integers(1, 9)), int(rng.integers(2, 11))
        k = int(rng.integers(1, min(4, e) + 1))
        ids = np.stack([np.stack([rng.choice(e, size=k, replace=False) for _ in range(l)])
                        for _ in range(t)])
        cases.append({"topk": ids.tolist(), "E": e,
                      "out": _kernels.activation_counts(ids, e).tolist()})
    ids = np.array([[[0, 2], [1, 1]], [[0, 1], [3, 1]]])
    cases.append({"topk": ids.tolist(), "E": 4,
                  "out": _kernels.activation_counts(ids, 4).tolist()})
    g["activation_counts"] = cases

    cases = []
    for _ in range(30):
        n, e = int(rng.integers(1, 40)), int(rng.integers(2, 12))
        ka, kb = int(rng.integers(1, e + 1)), int(rng.integers(1, e + 1))
        a = np.stack([rng.choice(e, size=ka, replace=False) for _ in range(n)])
        b = np.stack([rng.choice(e, size=kb, replace=False) for _ in range(n)])
        cases.append({"a": a.tolist(), "b": b.tolist(),
                      "out": _kernels.pair_overlap(a, b).tolist()})
    g["pair_overlap"] = cases

    cases = []
    for _ in range(30):
        l, e = int(rng.integers(1, 9)), int(rng.integers(2, 11))
        k = int(rng.integers(1, min(4, e) + 1))
        shape = ModelShape(l, e, k)
        t = int(rng.integers(1, 40))
        pt = rand_scores(rng, t * l, e).reshape(t, l, e)
        pt = pt / pt.sum(axis=2, keepdims=True)
        tr = RoutingTrace(shape, "c", pt, np.zeros((0, l, e)))
        cases.append({"L": l, "E": e, "k": k, "prefill_true": pt.tolist(),
                      "out": expert_counts(tr, "prefill").tolist()})
    g["expert_counts"] = cases

    # a5 init_from_calibration -----------------------------------------
    cases = []
    for _ in range(80):
        l, e = int(rng.integers(1, 9)), int(rng.integers(2, 11))
        calib = rng.random((l, e))
        if rng.random() < 0.4:  # count-derived calibration with ties
            calib = rng.integers(0, 5, size=(l, e)) / 7.0
        ecr = float(rng.uniform(0.05, 1.0))
        obj = {"calib": calib.tolist(), "ecr": ecr, "L": l, "E": e}
        try:
            p = init_from_calibration(calib, ecr, ModelShape(l, e, min(2, e)))
            obj["on_fast"] = [sorted(s) for s in p.on_fast]
            obj["budget"] = p.slot_budget
        except moesim.MoesimError as exc:
            obj["error"] = type(exc).__name__
        cases.append(obj)
    calib = np.random.default_rng(0).random((32, 8))
    for ecr in (0.25, 0.469, 0.5, 0.75, 1.0, 0.0, 1.5):
        obj = {"calib": calib.tolist(), "ecr": ecr, "L": 32, "E": 8}
        try:
            p = init_from_calibration(calib, ecr, ModelShape(32, 8, 2))
            obj["on_fast"] = [sorted(s) for s in p.on_fast]
            obj["budget"] = p.slot_budget
        except moesim.MoesimError as exc:
            obj["error"] = type(exc).__name__
        cases.append(obj)
    obj = {"calib": [[0.9, 0.7, 0.3, 0.1], [0.6, 0.5, 0.4, 0.65]], "ecr": 0.625,
           "L": 2, "E": 4}
    p = init_from_calibration(np.array(obj["calib"]), 0.625, ModelShape(2, 4, 2))
    obj["on_fast"] = [sorted(s) for s in p.on_fast]
    obj["budget"] = p.slot_budget
    cases.append(obj)
    g["init_from_calibration"] = cases

    # a6 allocate_for_sequence -----------------------------------------
    cases = []
    for i in range(300):
        l, e = int(rng.integers(1, 6)), int(rng.integers(2, 11))
        sets = [sorted(rng.choice(e, size=int(rng.integers(1, e + 1)), replace=False).tolist())
                for _ in range(l)]
        counts = rng.integers(0, 65, size=(l, e))
        thr = float(rng.choice([1.05, 1.05, 1.0, 1.5, 0.9, 2.0]))
        pl = ExpertPlacement(ModelShape(l, e, 1), sets, sum(len(s) for s in sets))
        new, ev = allocate_for_sequence(pl, counts, thr)
        cases.append({"on_fast": sets, "counts": counts.tolist(), "swap_in_out": thr,
                      "new": [sorted(s) for s in new.on_fast],
                      "events": [[x.layer, x.swapped_in, x.swapped_out, x.hot_tokens,
                                  x.cold_tokens] for x in ev]})
    for sets, counts in (([[0]], [[20, 21]]), ([[0]], [[20, 20]]),
                         ([[0, 1]], [[5, 9, 30, 0]]), ([[0, 1]], [[50, 40, 3, 2]]),
                         ([[0, 1]], [[0, 0, 64, 32]])):
        e = len(counts[0])
        pl = ExpertPlacement(ModelShape(1, e, 1), sets, len(sets[0]))
        new, ev = allocate_for_sequence(pl, np.array(counts))
        cases.append({"on_fast": sets, "counts": counts, "swap_in_out": 1.05,
                      "new": [sorted(s) for s in new.on_fast],
                      "events": [[x.layer, x.swapped_in, x.swapped_out, x.hot_tokens,
                                  x.cold_tokens] for x in ev]})
    g["allocate_for_sequence"] = cases

    # a8 degrade_selection ---------------------------------------------
    cases = []
    for _ in range(300):
        e = int(rng.integers(3, 11))
        k = int(rng.integers(2, min(4, e) + 1))
        s = rand_scores(rng, 1, e)[0]
        fast = sorted(rng.choice(e, size=int(rng.integers(0, e + 1)), replace=False).tolist())
        sel = _kernels.topk_rows(s[None, :], k)[0].tolist()
        new, deg = degrade_selection(s, sel, set(fast))
        cases.append({"scores": s.tolist(), "selection": sel, "fast": fast,
                      "new": [int(x) for x in new],
                      "degraded": [[d.dropped_expert, d.dropped_score,
                                    d.substitute_expert, d.substitute_score] for d in deg]})
    g["degrade_selection"] = cases

    # a7 plan_token (daop + fiddler) -----------------------------------
    cases = []
    for _ in range(150):
        l, e = int(rng.integers(2, 9)), int(rng.integers(3, 11))
        k = int(rng.integers(1, min(4, e) + 1))
        start = int(rng.integers(1, l + 1))
        engine = str(rng.choice(["daop", "daop", "fiddler"]))
        degr = bool(rng.random() < 0.85)
        shape = ModelShape(l, e, k)
        sets = [sorted(rng.choice(e, size=int(rng.integers(0, e + 1)), replace=False).tolist())
                for _ in range(l)]
        pl = ExpertPlacement(shape, sets, sum(len(s) for s in sets))
        true = rand_scores(rng, l, e)
        pred = np.zeros((l, e))
        pred[: l - 1] = rand_scores(rng, l - 1, e)
        from moesim import TokenRouting
        token = [TokenRouting(true[i] / true[i].sum() if False else true[i],
                              pred[i] if i < l - 1 else None) for i in range(l)]
        cfg = PolicyConfig(engine=engine, prediction_start_layer=start,
                           graceful_degradation=degr)
        plans = make_planner(pl, cfg).plan_token(token)
        cases.append({"L": l, "E": e, "k": k, "start": start, "engine": engine,
                      "degrade": degr, "on_fast": sets, "true": true.tolist(),
                      "pred": pred.tolist(), "plans": [plan_to_obj(p) for p in plans]})
    g["plan_token"] = cases

    # a9 prediction accuracy ------------------------------------------
    cases = []
    for _ in range(15):
        l, e = int(rng.integers(2, 7)), int(rng.integers(3, 9))
        k = int(rng.integers(1, min(3, e) + 1))
        n = int(rng.integers(1, 20))
        dt = rand_scores(rng, n * l, e).reshape(n, l, e)
        dp = np.zeros((n, l, e))
        dm = np.zeros((n, l), dtype=bool)
        dp[:, : l - 1] = rand_scores(rng, n * (l - 1), e).reshape(n, l - 1, e)
        dm[:, : l - 1] = True
        tr = RoutingTrace(ModelShape(l, e, k), "a", dt[:1], dt, decode_predicted=dp,
                          decode_mask=dm)
        acc = prediction_accuracy(tr)
        cases.append({"L": l, "E": e, "k": k, "decode_true": dt.tolist(),
                      "decode_pred": dp.tolist(),
                      "out": [None if np.isnan(a) else float(a) for a in acc]})
    g["prediction_accuracy"] = cases

    # a13 run_single decision flow on reference-generated traces -------
    traces, cases = [], []
    cost = default_cost_model()
    for shape, npre, ndec in ((ModelShape(8, 8, 2), 64, 64), (ModelShape(32, 8, 2), 64, 32)):
        calib_traces = [generate_trace(GeneratorConfig(shape=shape, seed=100 + i,
                                                        num_prefill_tokens=npre,
                                                        num_decode_tokens=ndec))
                        for i in range(4)]
        calib = pooled_decode_probabilities(calib_traces)
        trace = generate_trace(GeneratorConfig(shape=shape, seed=7,
                                               num_prefill_tokens=npre,
                                               num_decode_tokens=ndec))
        traces.append({
            "shape": [shape.num_layers, shape.num_experts, shape.top_k],
            "calib": calib.tolist(),
            "prefill_true": trace.prefill_true.tolist(),
            "decode_true": trace.decode_true.tolist(),
            "decode_pred": trace.decode_predicted.tolist(),
        })
        for ecr in (0.25, 0.5, 0.75):
            for engine in ("daop", "fiddler"):
                rec = run_single(trace, calib, ecr, engine, cost)
                dec = rec["_decode_result"]
                cases.append({
                    "trace": len(traces) - 1, "ecr": ecr, "engine": engine,
                    "placement_initial": [sorted(s) for s in rec["_placement_initial"].on_fast],
                    "placement_final": [sorted(s) for s in rec["_placement_final"].on_fast],
                    "swaps": [[s.layer, s.swapped_in, s.swapped_out, s.hot_tokens,
                               s.cold_tokens] for s in rec["_swaps"]],
                    "counts": {k2: int(v) for k2, v in dec.counts.items()},
                    "executed": [[list(map(int, ex)) for ex in tok] for tok in dec.executed],
                    "set_fidelity": rec["set_fidelity"],
                    # the rest of the flat record's decision fields (experiment.py:178-210)
                    "record": {key: rec[key] for key in (
                        "schema_version", "trace_id", "ecr", "engine", "seed",
                        "num_prefill_tokens", "num_decode_tokens", "migrations", "prefetches",
                        "wasted_prefetches", "slow_executions", "degradations", "stale_inputs",
                        "set_fidelity", "score_mass", "swap_count",
                        "similarity_prefill_decode")},
                })
        if shape.num_layers == 8:
            # calibration + fidelity metrics (experiment.py:132-142,
            # metrics.py:74-82,114-117,177-215) on the same traces
            from moesim import activation_matrix, routing_fidelity, similarity
            rng = np.random.default_rng(5)
            execs = []
            for _ in range(3):  # random executed sets (k distinct experts per layer)
                execs.append([[sorted(rng.choice(shape.num_experts, shape.top_k,
                                                 replace=False).tolist())
                               for _ in range(shape.num_layers)]
                              for _ in range(trace.num_decode_tokens)])
            g["metrics"] = {
                "shape": [shape.num_layers, shape.num_experts, shape.top_k],
                "calib_decode_true": [t.decode_true.tolist() for t in calib_traces],
                "calib_prefill_true": [t.prefill_true.tolist() for t in calib_traces],
                "pooled_decode_probabilities": calib.tolist(),
                "trace": len(traces) - 1,
                "activation_prefill": activation_matrix(trace, "prefill").values.tolist(),
                "activation_decode": activation_matrix(trace, "decode").values.tolist(),
                "similarity": similarity(activation_matrix(trace, "prefill"),
                                         activation_matrix(trace, "decode")),
                "executed": execs,
                "routing_fidelity": [list(routing_fidelity(trace, ex)) for ex in execs],
            }
    g["run_single"] = {"traces": traces, "cases": cases}

    OUT.write_text(json.dumps(g, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
