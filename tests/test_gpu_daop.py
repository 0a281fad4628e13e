"""End-to-end DAOP sequence on the GPU vs the oracle (reference decisions).

The engine runs calibration placement -> prefill (device activation counter,
Alg. 1 per layer, pinned-memory migrations, slow experts on the host tier)
-> decode (device DAOP plans, degradation, stale pre-calculation on the host
tier).  Then the REFERENCE decision flow (oracle/decisions.py, pinned to
moesim's golden vectors) is run on the trace the engine exported and every
decision must agree bit-for-bit; hidden states are checked teacher-forced.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import decisions as D  # noqa: E402
from oracle import numerics as N  # noqa: E402


def _calib(L, E, k, seed):
    rng = np.random.default_rng(seed)
    c = rng.dirichlet(np.ones(E) * 0.7, size=L) * k
    return c


@pytest.mark.parametrize("engine,ecr,start,attention,E,k", [
    ("daop", 0.5, 4, False, 8, 2), ("daop", 0.25, 2, False, 8, 2),
    ("fiddler", 0.5, 4, False, 8, 2), ("daop", 1.0, 4, False, 8, 2),
    ("ondemand", 0.5, 4, False, 8, 2), ("prefetch", 0.25, 2, False, 8, 2),
    # full decoder layers: attention with a KV cache before every MoE block
    ("daop", 0.5, 4, True, 8, 2), ("ondemand", 0.5, 4, True, 8, 2),
    # the widest shape the decode kernel takes (E <= 16), top-4
    ("daop", 0.5, 3, False, 16, 4)])
def test_daop_sequence_matches_reference_decisions(engine, ecr, start, attention, E, k):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.daop import DaopEngine

    L, d, ffn = 8, 256, 512
    shape = P.ModelShape(L, E, k)
    calib = _calib(L, E, k, 5)
    cfg = P.PolicyConfig(engine, prediction_start_layer=start)
    eng = DaopEngine(shape, d, ffn, calib, ecr, cfg, seed=0, device="cuda",
                     attention=attention, max_seq=128)
    prompt = eng.model.input_hidden(64, stream=11)
    toks = [eng.model.input_hidden(1, stream=12, step=i)[0] for i in range(10)]
    rec = eng.run_sequence(prompt, toks, "s0")
    tr = rec.trace

    # (a5) calibration placement
    sets0, budget = D.init_from_calibration(calib, ecr)
    assert [set(s) for s in rec.prefill.placement_initial.on_fast] == sets0
    assert rec.prefill.placement_initial.slot_budget == budget
    # (a3) device activation counter == reference expert_counts on the exported trace
    counts = D.expert_counts(tr.prefill_true, k)
    assert np.array_equal(rec.prefill.counts, counts)
    # (a6) Alg. 1 swaps (only daop reallocates; moesim/experiment.py:158-163)
    if engine == "daop":
        sets, evs = D.allocate_for_sequence(sets0, counts)
    else:
        sets, evs = [set(s) for s in sets0], []
    assert [(s.layer, s.swapped_in, s.swapped_out, s.hot_tokens, s.cold_tokens)
            for s in rec.prefill.swaps] == evs
    assert [set(s) for s in rec.prefill.placement.on_fast] == sets
    # (a11) swap copies overlap the resident experts' GEMMs; the hidden part is
    # measured like simulator.py:495-502 prices it
    pf = rec.prefill
    if evs:
        assert pf.migration_ms > 0 and 0.0 <= pf.migration_hidden_ms <= pf.migration_ms
    else:
        assert pf.migration_ms == 0.0 and pf.migration_hidden_ms == 0.0
    # the HBM slot table follows the placement (LRU engines move it during decode)
    if engine in ("daop", "fiddler"):
        assert np.array_equal(eng.model.resident_mask(), rec.prefill.placement.mask())
    # (a7/a8/a9) per-token plans on the exported trace
    mask = np.array([l < L - 1 for l in range(L)])
    if engine in ("ondemand", "prefetch"):
        caches = D.LruCaches(sets)
        oplans = [D.plan_token_lru(tr.decode_true[t], tr.decode_predicted[t], mask, caches, k,
                                   engine, start) for t in range(tr.num_decode_tokens)]
        # the HBM residence ends equal to the replayed LRU caches
        assert [set(np.nonzero(r)[0].tolist()) for r in eng.model.resident_mask()] \
            == [set(c) for c in caches.last_use]
    else:
        oplans = [D.plan_token(tr.decode_true[t], tr.decode_predicted[t], mask, sets, k, engine,
                               start=start) for t in range(tr.num_decode_tokens)]
    for t, (got, exp) in enumerate(zip([r.plans for r in rec.decode], oplans)):
        for l in range(L):
            assert [(x.expert, x.device, x.input_source, x.precalc) for x in got[l].executed] \
                == [tuple(x) for x in exp[l]["executed"]], (t, l)
            assert [(g.dropped_expert, g.substitute_expert) for g in got[l].degraded] \
                == [(a, c) for a, _, c, _ in exp[l]["degraded"]], (t, l)
            assert list(got[l].migrations) == list(exp[l].get("migrations", []))
            assert list(got[l].prefetch_issues) == list(exp[l].get("prefetch_issues", []))
    # (a10) simulator counters
    assert rec.counts == D.decode_counters(oplans, engine, start)
    # trace is reference-valid: sums to 1 within SCORE_SUM_TOL (checked at construction)
    assert tr.num_decode_tokens == 10 and tr.num_prefill_tokens == 64
    # ... and survives the moesim JSONL file boundary exactly
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        P.save_trace(tr, f"{td}/t.jsonl")
        assert P.load_trace(f"{td}/t.jsonl") == tr

    # numerics, teacher-forced with the engine's decisions
    om = N.OracleModel(L, E, k, d, ffn, seed=0)
    h = prompt.cpu().numpy()
    ptop = D.topk_rows(tr.prefill_true.reshape(-1, E), k).reshape(64, L, k)
    if attention:
        oatt = N.OracleAttention(d, d // 128, max(1, d // 512), theta=eng.attn.theta, seed=0)
        caches = {}
    for l in range(L):
        if attention:  # causal attention over the prompt (the oracle keeps its own cache)
            kc = np.zeros((oatt.n_kv, 128, 128), dtype=np.float32)
            vc = np.zeros_like(kc)
            for t in range(64):
                h[t], _, kc, vc = N.attention_decode(oatt, l, h[t], t, kc, vc)
            caches[l] = [kc, vc]
        p = tr.prefill_true[:, l, :].astype(np.float32)
        sel = ptop[:, l, :]
        h = N.moe_layer(om, l, h, sel=sel, w=N.renorm_weights(p, sel))["out"]
    ref = h
    got = rec.prefill.out.cpu().numpy()
    rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2)))
    assert np.abs(got - ref).max() <= 5e-3 * rms + 2e-3 * np.abs(ref).max()
    for t in range(3):
        plans = rec.decode[t].plans
        sel = [([x.expert for x in p.executed], [x.device == "slow" for x in p.executed])
               for p in plans]
        pre = None
        if attention:
            def pre(hv, l, pos=64 + t):
                out, _, caches[l][0], caches[l][1] = N.attention_decode(
                    oatt, l, hv, pos, caches[l][0], caches[l][1])
                return out
        ref = N.daop_decode_token(om, toks[t].cpu().numpy(), sel, start, True,
                                  engine if engine in ("daop", "fiddler") else "fiddler", pre=pre)
        got = rec.decode[t].out.cpu().numpy()
        rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2)))
        assert np.abs(got - ref).max() <= 5e-3 * rms + 2e-3 * np.abs(ref).max(), t


def test_full_decode_token_and_graph_match_engine():
    """MoEBlockEngine.decode_token (all layers HBM-resident, DAOP plans from
    layer `start`) and its CUDA-graph replay == DaopEngine at ECR 1.0, bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.daop import DaopEngine
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.model import MoEModel

    L, E, k, d, ffn = 6, 8, 2, 256, 512
    shape = P.ModelShape(L, E, k)
    m = MoEModel(shape, d, ffn, seed=3)
    eng = MoEBlockEngine(m)
    de = DaopEngine(shape, d, ffn, np.full((L, E), k / E), 1.0,
                    P.PolicyConfig("daop", prediction_start_layer=2), seed=3)
    g, g_in, g_out = eng.capture_decode_graph(start=2)
    for t in range(4):
        h = m.input_hidden(1, stream=21, step=t)[0]
        a = eng.decode_token(h, start=2).clone()
        b = de.decode(h).out
        g_in.copy_(h)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(a, b), t
        assert torch.equal(g_out, a), t


def test_decode_host_graph_matches_device_decode():
    """The end-to-end host API (graph: H2D, decode launch, D2H) returns the
    same residual and selection as the device call, for any host tensor."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.model import MoEModel

    L, E, k, d, ffn = 2, 8, 2, 256, 512
    m = MoEModel(P.ModelShape(L, E, k), d, ffn, seed=4)
    eng = MoEBlockEngine(m)
    for t in range(4):
        for layer in (0, 1):
            h = m.input_hidden(1, stream=31, step=t)[0]
            h_host = h.cpu()  # pageable on purpose: staged into the pinned buffer
            out, sel = eng.decode_host(h_host, layer)
            out, sel = out.clone(), sel.clone()
            eng.decode(h, layer)
            torch.cuda.synchronize()
            assert torch.equal(out, eng.bufs.h_out.cpu()), (t, layer)
            assert torch.equal(sel, eng.bufs.sel.cpu()), (t, layer)


def test_host_pool_device_fill_matches_host_fill():
    """HostExpertPool generated on the GPU (bench / daop32 fast path) is bit-
    identical to the host generator's pool."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.daop import HostExpertPool
    shape = P.ModelShape(2, 4, 2)
    a = HostExpertPool(shape, 256, 512, seed=9)
    b = HostExpertPool(shape, 256, 512, seed=9, device="cuda")
    assert torch.equal(a.buf.view(torch.int16), b.buf.view(torch.int16))
    # registered with the driver: copies from it are true async DMAs
    assert b.pinned and b.buf.is_pinned()


@pytest.mark.parametrize("attention", [False, True])
def test_resident_prefill_graph_equals_eager(attention):
    """A fully resident model's prefill replays as one CUDA graph per prompt
    length: bit-identical output, counts and exported scores to the eager
    per-layer loop, also when the graph is replayed for a second prompt."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.daop import DaopEngine, HostExpertPool
    L, E, k, d, ffn = 4, 8, 2, 256, 512
    shape = P.ModelShape(L, E, k)
    pool = HostExpertPool(shape, d, ffn, seed=3)
    res = {}
    for graphs in (False, True):
        eng = DaopEngine(shape, d, ffn, np.full((L, E), 0.25), 1.0, P.PolicyConfig("daop"),
                         seed=3, host_pool=pool, attention=attention, max_seq=128)
        eng.prefill_graphs = graphs  # the switch, both ways
        outs = []
        for s_ in (0, 1):
            pre = eng.prefill(eng.model.input_hidden(40, stream=500 + s_))
            outs.append((pre.out.clone(), pre.counts.copy(), pre.true_scores.copy(),
                         pre.pred_scores.copy()))
        res[graphs] = outs
        assert len(eng._pf_graphs) == (1 if graphs else 0)
    for a, b in zip(res[False], res[True]):
        assert torch.equal(a[0], b[0])
        for x, y in zip(a[1:], b[1:]):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("rows", [128, 256])
def test_slow_split_equals_host_expert(rows):
    """A slow expert split between the GPU (rows [0, R) pulled from the pinned
    pool over PCIe, skinny tcgen05 GEMMs) and the host tier (rows [R, ffn))
    equals the host tier's whole expert within the fp32 reassociation of the
    down sums (tried: off by default)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.daop import HostExpertPool, SlowSplit, host_expert_ffn
    shape = P.ModelShape(2, 4, 2)
    d, ffn = 256, 512
    pool = HostExpertPool(shape, d, ffn, seed=5, device="cuda")
    sp = SlowSplit(pool, rows, "cuda", threads=4)
    from oracle import rng as R
    xb = R.f32_to_bf16_bits(np.random.default_rng(rows).normal(size=(1, d)).astype(np.float32))
    for layer, e in ((0, 1), (1, 3)):
        ref = host_expert_ffn(pool, layer, e, xb, 4)
        y = sp.run(layer, e, xb)
        tol = 2e-3 * float(np.sqrt(np.mean(ref ** 2))) + 1e-3 * np.abs(ref).max()
        assert np.abs(y - ref).max() <= tol
