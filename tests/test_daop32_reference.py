"""BASELINE configs[2] at scale (32 Mixtral-8x7B layers, 256-token prompt,
16 decode tokens, ECR 0.75 / 0.5 / 0.25): every decision the B200 engine made
equals what the UNMODIFIED reference decides on the engine's own exported
trace with the engine's own calibration (moesim/experiment.py:145-211
run_single; golden written by tests/golden/make_daop32_golden.py from the
committed GPU export of scripts/daop32.py --export-dir).

Checked exactly: initial placement (init_from_calibration), the Alg. 1 swaps
and the post-swap placement (allocate_for_sequence on the device activation
counter's counts), the per-token executed expert sets of the DAOP planner
(prediction from layer 4, graceful degradation), the simulator's counters
(slow_executions, degradations, stale_inputs, migrations) -- plus the device
counter against the counts the trace implies."""

import gzip
import json
import tempfile
from pathlib import Path

import numpy as np
import pytest

import paper_2501_10375_b200 as P
from oracle import decisions as D

DIR = Path(__file__).parent / "golden" / "daop32"
ECRS = sorted(json.loads(p.read_text())["ecr"] for p in DIR.glob("engine_ecr*.json")) \
    if DIR.exists() else []


def _load(ecr):
    eng = json.loads((DIR / f"engine_ecr{ecr}.json").read_text())
    ref = json.loads((DIR / f"reference_ecr{ecr}.json").read_text())
    raw = gzip.decompress((DIR / f"trace_ecr{ecr}.jsonl.gz").read_bytes())
    with tempfile.NamedTemporaryFile(suffix=".jsonl") as f:
        f.write(raw)
        f.flush()
        trace = P.load_trace(f.name)
    return eng, ref, trace


@pytest.mark.skipif(not ECRS, reason="no exported 32-layer run")
@pytest.mark.parametrize("ecr", ECRS)
def test_engine_decisions_equal_reference_run_single(ecr):
    eng, ref, trace = _load(ecr)
    assert trace.shape == P.ModelShape(32, 8, 2)
    assert trace.num_prefill_tokens == 256 and trace.num_decode_tokens == 16
    for key in ("placement_initial", "placement_final", "swaps", "executed"):
        assert eng[key] == ref[key], key
    assert eng["counts"] == ref["counts"]
    assert len(eng["swaps"]) == ref["swap_count"]
    # the device activation counter == the counts of the exported true gates
    counts = D.expert_counts(trace.prefill_true, 2)
    assert np.array_equal(np.array(eng["device_counts"]), counts)


@pytest.mark.skipif(not ECRS, reason="no exported 32-layer run")
@pytest.mark.parametrize("ecr", ECRS)
def test_native_host_decisions_reproduce_the_run(ecr):
    """The package's own host decision path (native placement / Alg. 1 /
    planner) on the exported trace reproduces the engine's run too."""
    eng, ref, trace = _load(ecr)
    calib = np.array(json.loads((DIR / "calib.json").read_text())["calib"])
    pl0 = P.init_from_calibration(calib, ecr, trace.shape)
    assert [sorted(s) for s in pl0.on_fast] == ref["placement_initial"]
    pl, swaps = P.allocate_for_sequence(pl0, D.expert_counts(trace.prefill_true, 2))
    assert [sorted(s) for s in pl.on_fast] == ref["placement_final"]
    cfg = P.PolicyConfig("daop")
    plans = P.plan_trace_decode(trace, pl, cfg)
    assert [[list(p.executed_experts()) for p in tok] for tok in plans] == ref["executed"]
    assert P.decode_counters(plans, cfg) == ref["counts"]
