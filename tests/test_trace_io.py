"""moesim JSONL trace files: the on-disk boundary to the
reference's analysis tools.  Golden files were written by the reference's own
save_trace (tests/golden/make_trace_golden.py); ours must reproduce them byte
for byte and read them back exactly, with moesim's error semantics
(moesim/trace.py:325-476, tests/test_trace.py:52-175)."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2501_10375_b200 as P

GOLD = Path(__file__).parent / "golden" / "traces"
NAMES = ["third", "edge", "random", "mixtral_gen"]


def test_golden_edge_trace_byte_identical(tmp_path):
    # the in-memory trace of make_trace_golden.py "edge": exponent formats,
    # denormals, exact 0 / 1, negative zero, JSON escapes in the id
    e = np.array([[[1.0, -0.0, 0.0, 0.0], [1 - 1e-7, 5e-324, 1e-7, 1e-300]],
                  [[0.25, 0.25, 0.25, 0.25], [0.5, 0.125, 0.125, 0.25]]])
    dp = np.array([[[0.1, 0.2, 0.3, 0.4], [0, 0, 0, 0]]])
    tr = P.RoutingTrace(P.ModelShape(2, 4, 2), 'edge "q"/\\', e, e[:1], decode_predicted=dp,
                        decode_mask=np.array([[True, False]]))
    out = tmp_path / "o.jsonl"
    P.save_trace(tr, out)
    assert out.read_bytes() == (GOLD / "edge.jsonl").read_bytes()
    # json reads "-0" as the integer 0, in moesim's loader and in ours alike
    back = P.load_trace(out)
    assert back.prefill_true[0, 0, 1] == 0.0 and back.prefill_true[1, 1, 1] == 0.125


@pytest.mark.parametrize("name", ["third", "random", "mixtral_gen"])
def test_golden_files_roundtrip_byte_identical(name, tmp_path):
    src = GOLD / f"{name}.jsonl"
    tr = P.load_trace(src)
    out = tmp_path / "o.jsonl"
    P.save_trace(tr, out)
    assert out.read_bytes() == src.read_bytes()
    assert P.load_trace(out) == tr


@pytest.mark.parametrize("name", NAMES)
def test_golden_values_exact(name):
    lines = (GOLD / f"{name}.jsonl").read_text().splitlines()
    hdr = json.loads(lines[0])
    tr = P.load_trace(GOLD / f"{name}.jsonl")
    assert tr.shape == P.ModelShape(hdr["L"], hdr["E"], hdr["k"])
    assert tr.sequence_id == hdr["sequence_id"]
    for ln in lines[1:]:
        rec = json.loads(ln)
        ph, t = rec["phase"], rec["token_index"]
        for l, ent in enumerate(rec["layers"]):
            assert getattr(tr, f"{ph}_true")[t, l].tolist() == ent["true_scores"]
            has = ent["predicted_scores"] is not None
            assert bool(getattr(tr, f"{ph}_mask")[t, l]) == has
            if has:
                assert getattr(tr, f"{ph}_predicted")[t, l].tolist() == ent["predicted_scores"]


def test_full_precision_third(tmp_path):
    third = 1.0 / 3.0
    tr = P.RoutingTrace(P.ModelShape(1, 2, 1), "p", np.array([[[third, 1 - third]]]),
                        np.zeros((0, 1, 2)))
    path = tmp_path / "p.jsonl"
    P.save_trace(tr, path)
    assert P.load_trace(path).prefill_true[0, 0, 0] == third
    assert "0.33333333333333331" in path.read_text().splitlines()[1]


def _random_trace(rng, shape, n_prefill, n_decode, sid, prefill_predictions):
    l, e = shape.num_layers, shape.num_experts

    def rows(n):
        raw = rng.random((n, e)) + 1e-3
        return raw / raw.sum(axis=1, keepdims=True)

    pt = rows(n_prefill * l).reshape(n_prefill, l, e)
    dt = rows(max(n_decode, 1) * l).reshape(-1, l, e)[:n_decode]
    dp, dm = np.zeros((n_decode, l, e)), np.zeros((n_decode, l), dtype=bool)
    if n_decode and l > 1:
        dp[:, : l - 1] = rows(n_decode * (l - 1)).reshape(n_decode, l - 1, e)
        dm[:, : l - 1] = True
    pp, pm = np.zeros((n_prefill, l, e)), np.zeros((n_prefill, l), dtype=bool)
    if prefill_predictions and l > 1:
        pp[:, : l - 1] = rows(n_prefill * (l - 1)).reshape(n_prefill, l - 1, e)
        pm[:, : l - 1] = True
    return P.RoutingTrace(shape, sid, pt, dt, pp, pm, dp, dm)


def test_roundtrip_randomized(tmp_path):
    # tests/test_trace.py:139-160, plus fp32-rounded engine-style scores
    rng = np.random.default_rng(123)
    for i in range(50):
        shape = P.ModelShape(int(rng.integers(1, 5)), int(rng.integers(2, 7)), 1)
        tr = _random_trace(rng, shape, int(rng.integers(1, 4)), int(rng.integers(0, 4)),
                           f"r{i}", bool(rng.integers(0, 2)))
        path = tmp_path / f"{i}.jsonl"
        P.save_trace(tr, path)
        assert P.load_trace(path) == tr


def test_large_trace_parallel_formatting(tmp_path):
    # many tokens -> the native writer splits across threads; order and bytes
    # must not depend on the split
    rng = np.random.default_rng(5)
    tr = _random_trace(rng, P.ModelShape(8, 8, 2), 700, 300, "big", True)
    path = tmp_path / "big.jsonl"
    P.save_trace(tr, path)
    lines = path.read_text().splitlines()
    assert len(lines) == 1001
    assert [json.loads(x)["token_index"] for x in lines[1:4]] == [0, 1, 2]
    assert json.loads(lines[701])["phase"] == "decode"
    # every line equals the straightforward per-token formatting
    for t in (0, 349, 699):
        ent = json.loads(lines[1 + t])["layers"]
        exp = ",".join(format(float(v), ".17g") for v in tr.prefill_true[t, 3])
        assert f'"true_scores":[{exp}]' in lines[1 + t]
        assert len(ent) == 8
    assert P.load_trace(path) == tr


HDR = {"format_version": 1, "sequence_id": "b", "L": 1, "E": 2, "k": 1,
       "num_prefill_tokens": 1, "num_decode_tokens": 0}


def _write(path, header, *tokens):
    path.write_text("\n".join([json.dumps(header)] + [json.dumps(t) for t in tokens]) + "\n")


def test_shape_mismatch_names_token_and_layer(tmp_path):
    path = tmp_path / "bad.jsonl"
    _write(path, HDR, {"phase": "prefill", "token_index": 0,
                       "layers": [{"true_scores": [0.2, 0.3, 0.5], "predicted_scores": None}]})
    with pytest.raises(P.ShapeMismatchError) as exc:
        P.load_trace(path)
    assert "token 0" in str(exc.value) and "layer 0" in str(exc.value)


def test_parse_error_names_line(tmp_path):
    path = tmp_path / "bad.jsonl"
    path.write_text(json.dumps(HDR) + "\n{not json}\n")
    with pytest.raises(P.TraceParseError) as exc:
        P.load_trace(path)
    assert "line 2" in str(exc.value)


def test_normalization_error_on_bad_sum(tmp_path):
    path = tmp_path / "bad.jsonl"
    _write(path, HDR, {"phase": "prefill", "token_index": 0,
                       "layers": [{"true_scores": [0.6, 0.6], "predicted_scores": None}]})
    with pytest.raises(P.NormalizationError) as exc:
        P.load_trace(path)
    assert "deviates" in str(exc.value)


def test_first_bad_layer_is_named(tmp_path):
    hdr = dict(HDR, L=3)
    good = {"true_scores": [0.5, 0.5], "predicted_scores": None}
    path = tmp_path / "bad.jsonl"
    _write(path, hdr, {"phase": "prefill", "token_index": 0,
                       "layers": [good, {"true_scores": [-0.5, 1.5], "predicted_scores": None},
                                  {"true_scores": [0.9, 0.9], "predicted_scores": None}]})
    with pytest.raises(P.NormalizationError) as exc:
        P.load_trace(path)
    assert "layer 1" in str(exc.value) and "negative" in str(exc.value)
    _write(path, hdr, {"phase": "prefill", "token_index": 0,
                       "layers": [good, good, {"true_scores": [0.5, 0.5],
                                               "predicted_scores": [0.5]}]})
    with pytest.raises(P.ShapeMismatchError) as exc:
        P.load_trace(path)
    assert "layer 2" in str(exc.value) and "predicted_scores length" in str(exc.value)


@pytest.mark.parametrize("body,err,frag", [
    ("", P.TraceParseError, "empty file"),
    ('[1,2]\n', P.TraceParseError, "malformed header"),
    (json.dumps(dict(HDR, format_version=2)) + "\n", P.TraceParseError, "format_version"),
    (json.dumps(HDR) + "\n", P.TraceParseError, "expected 1 token records, found 0"),
    (json.dumps(HDR) + '\n{"phase":"x","token_index":0,"layers":[]}\n', P.TraceParseError,
     "unknown phase"),
    (json.dumps(HDR) + '\n{"phase":"prefill","token_index":3,"layers":[]}\n', P.TraceParseError,
     "out of order"),
    (json.dumps(HDR) + '\n{"phase":"prefill","token_index":0,"layers":[]}\n',
     P.ShapeMismatchError, "has 0 layers"),
    (json.dumps(HDR) + '\n{"token_index":0}\n', P.TraceParseError, "malformed token record"),
])
def test_file_errors(tmp_path, body, err, frag):
    path = tmp_path / "e.jsonl"
    path.write_text(body)
    with pytest.raises(err) as exc:
        P.load_trace(path)
    assert frag in str(exc.value)


def test_decode_predictions_required(tmp_path):
    hdr = dict(HDR, L=2, num_decode_tokens=1)
    t = {"true_scores": [0.5, 0.5], "predicted_scores": None}
    path = tmp_path / "d.jsonl"
    _write(path, hdr, {"phase": "prefill", "token_index": 0, "layers": [t, t]},
           {"phase": "decode", "token_index": 0, "layers": [t, t]})
    with pytest.raises(P.ShapeMismatchError):
        P.load_trace(path)


def test_parse_shape():
    assert P.parse_shape("mixtral") == P.MIXTRAL_SHAPE
    assert P.parse_shape(" PHI ").num_experts == 16
    assert P.parse_shape("4x6x2") == P.ModelShape(4, 6, 2)
    for bad in ("4x6", "axbxc"):
        with pytest.raises(P.ShapeMismatchError):
            P.parse_shape(bad)
