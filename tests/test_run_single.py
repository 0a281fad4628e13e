"""`run_single` drop-in (moesim/experiment.py:145-211) and the calibration /
fidelity metrics, against golden vectors written by the unmodified reference
(tests/golden/make_golden.py -> decisions.json "run_single" / "metrics"), and
the error classes' identity with moesim's when the reference is installed.

run_single and the metrics count activations through the operator table
(kernels.py: top-k / histogram on the device), so those tests are GPU tests;
the golden JSON travels to the GPU box with the repo."""

import json
import math
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2501_10375_b200 as P

GOLD = Path(__file__).parent / "golden" / "decisions.json"
ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def golden():
    return json.loads(GOLD.read_text())


def _trace(shape, tid, pre, dt, dp=None):
    l = shape.num_layers
    dt = np.array(dt)
    dp = dt if dp is None else np.array(dp)
    dm = np.zeros(dt.shape[:2], dtype=bool)
    dm[:, : l - 1] = True
    return P.RoutingTrace(shape, tid, np.array(pre), dt, decode_predicted=dp, decode_mask=dm)


def _same(a, b):
    if isinstance(b, float) and math.isnan(b):
        return isinstance(a, float) and math.isnan(a)
    return a == b


@pytest.mark.gpu
def test_run_single_record_matches_reference(golden):
    rs = golden["run_single"]
    for c in rs["cases"]:
        tr = rs["traces"][c["trace"]]
        shape = P.ModelShape(*tr["shape"])
        trace = _trace(shape, c["record"]["trace_id"], tr["prefill_true"], tr["decode_true"],
                       tr["decode_pred"])
        rec = P.run_single(trace, np.array(tr["calib"]), c["ecr"], c["engine"], None)
        for key, want in c["record"].items():
            assert _same(rec[key], want), (c["ecr"], c["engine"], key, rec[key], want)
        assert [sorted(s) for s in rec["_placement_initial"].on_fast] == c["placement_initial"]
        assert [sorted(s) for s in rec["_placement_final"].on_fast] == c["placement_final"]
        assert [[s.layer, s.swapped_in, s.swapped_out, s.hot_tokens, s.cold_tokens]
                for s in rec["_swaps"]] == c["swaps"]
        dec = rec["_decode_result"]
        assert isinstance(dec, P.TimelineResult)
        assert dec.counts == c["counts"]
        assert [[list(ex) for ex in tok] for tok in dec.executed] == c["executed"]
        # timings are measured by DaopEngine.run_single; a trace-only call has none
        assert math.isnan(rec["tokens_per_second"])


@pytest.mark.gpu
def test_run_single_rejects_unknown_engine(golden):
    tr = golden["run_single"]["traces"][0]
    shape = P.ModelShape(*tr["shape"])
    trace = _trace(shape, "t", tr["prefill_true"], tr["decode_true"], tr["decode_pred"])
    with pytest.raises(P.ConfigError):
        P.run_single(trace, np.array(tr["calib"]), 0.5, "magic", None)
    with pytest.raises(P.BudgetError):
        P.run_single(trace, np.array(tr["calib"]), 0.0, "daop", None)


@pytest.mark.gpu
def test_calibration_and_fidelity_metrics_match_reference(golden):
    g = golden["metrics"]
    shape = P.ModelShape(*g["shape"])
    calib = [_trace(shape, f"c{i}", pre, dt) for i, (pre, dt) in
             enumerate(zip(g["calib_prefill_true"], g["calib_decode_true"]))]
    assert np.array_equal(P.pooled_decode_probabilities(calib),
                          np.array(g["pooled_decode_probabilities"]))
    tr = golden["run_single"]["traces"][g["trace"]]
    trace = _trace(shape, "t", tr["prefill_true"], tr["decode_true"], tr["decode_pred"])
    ap, ad = P.activation_matrix(trace, "prefill"), P.activation_matrix(trace, "decode")
    assert np.array_equal(ap.values, np.array(g["activation_prefill"]))
    assert np.array_equal(ad.values, np.array(g["activation_decode"]))
    assert ap.token_count == trace.num_prefill_tokens and ap.phase == "prefill"
    assert P.similarity(ap, ad) == g["similarity"]
    for ex, want in zip(g["executed"], g["routing_fidelity"]):
        assert list(P.routing_fidelity(trace, ex)) == want


@pytest.mark.skipif(not Path("/root/reference/pkg/src/moesim").exists(),
                    reason="the reference is only present in the build container")
def test_errors_are_moesim_classes_when_installed(tmp_path):
    code = (
        "import numpy as np, moesim, paper_2501_10375_b200 as P\n"
        "assert P.errors.REFERENCE_CLASSES\n"
        "for n in ('MoesimError','BudgetError','ShapeMismatchError','ConfigError',"
        "'PredictionMissingError','NormalizationError','EmptyPhaseError','TraceParseError'):\n"
        "    assert getattr(P, n) is getattr(moesim, n), n\n"
        "try:\n"
        "    P.init_from_calibration(np.ones((2, 4)) / 2, 0.0, P.ModelShape(2, 4, 2))\n"
        "except moesim.BudgetError:\n"
        "    print('caught')\n")
    env = dict(os.environ, PYTHONPATH=f"{ROOT}:/root/reference/pkg/src",
               NUMBA_CACHE_DIR=str(tmp_path / "numba"), PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=tmp_path, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "caught" in r.stdout


def test_errors_standalone_without_reference():
    assert issubclass(P.BudgetError, P.MoesimError)
    assert issubclass(P.DeviceError, RuntimeError)
