"""BASELINE configs[2]: Mixtral-8x7B-shaped 32-layer decode under DAOP at
expert-cache ratios 0.75 / 0.5 / 0.25, slow experts on the host tier.

    python scripts/daop32.py [--layers 32] [--prompt 256] [--decode 16] [--out file]

Flow per ECR (moesim/experiment.py:145-211 run_single, executed):
  calibration  : one sequence at ECR 1.0 -> pooled decode activation matrix
  init         : init_from_calibration(calib, ecr)    (slot budget in HBM)
  prefill      : prompt tokens, device activation counter, Alg. 1 swaps with
                 pinned-host -> HBM migrations, slow experts on the host tier
  decode       : tokens/s with DAOP plans, stale pre-calculation on the host
Also reports the reference's counters (slow_executions, degradations,
stale_inputs, migrations) and prediction accuracy on the exported trace.
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.daop import DaopEngine, HostExpertPool  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--prompt", type=int, default=256)
    ap.add_argument("--decode", type=int, default=16)
    ap.add_argument("--ecr", type=float, nargs="+", default=[0.75, 0.5, 0.25])
    ap.add_argument("--out", default="")
    ap.add_argument("--trace-dir", default="", help="save each run's routing trace (moesim JSONL)")
    ap.add_argument("--attention", action="store_true",
                    help="full decoder layers: attention with a KV cache before each MoE block")
    ap.add_argument("--export-dir", default="",
                    help="write the calibration, each run's trace (gzipped moesim JSONL) and the "
                         "engine's decisions for the reference parity test "
                         "(tests/golden/make_daop32_golden.py)")
    ap.add_argument("--host-fill", action="store_true",
                    help="generate the pinned pool with the host generator (default: on the GPU)")
    a = ap.parse_args()
    shape = P.ModelShape(a.layers, 8, 2)
    t0 = time.perf_counter()
    pool = HostExpertPool(shape, a.d, a.ffn, seed=0,
                          device=None if a.host_fill else torch.device("cuda"))
    res = {"config": {"layers": a.layers, "d": a.d, "ffn": a.ffn, "experts": 8, "top_k": 2,
                      "prompt_tokens": a.prompt, "decode_tokens": a.decode,
                      "attention": a.attention},
           "host_pool_gb": pool.buf.numel() * 2 / 1e9,
           "host_pool_setup_s": time.perf_counter() - t0}
    caps = np.zeros(2, dtype=np.int32)
    from paper_2501_10375_b200 import _lib
    _lib.call("daop_host_caps", caps.ctypes.data, caps.ctypes.data + 4)
    res["host"] = {"avx512_bf16": bool(caps[0]), "threads": int(caps[1])}

    # calibration sequence at ECR 1.0 (everything in HBM)
    cal = DaopEngine(shape, a.d, a.ffn, np.full((a.layers, 8), 0.25), 1.0,
                     P.PolicyConfig("daop"), seed=0, host_pool=pool)
    crec = cal.run_sequence(cal.model.input_hidden(64, stream=300),
                            [cal.model.input_hidden(1, stream=301, step=i)[0] for i in range(16)],
                            "calib")
    calib = P.pooled_decode_probabilities([crec.trace])
    exp = Path(a.export_dir) if a.export_dir else None
    if exp:
        exp.mkdir(parents=True, exist_ok=True)
        (exp / "calib.json").write_text(json.dumps({"calib": calib.tolist()}))
    res["calibration_prediction_accuracy"] = P.mean_prediction_accuracy(crec.trace)
    del cal, crec
    torch.cuda.empty_cache()

    runs = []
    for ecr in a.ecr:
        eng = DaopEngine(shape, a.d, a.ffn, calib, ecr, P.PolicyConfig("daop"), seed=0,
                         host_pool=pool, attention=a.attention,
                         max_seq=a.prompt + a.decode + 64)
        prompt = eng.model.input_hidden(a.prompt, stream=400)
        toks = [eng.model.input_hidden(1, stream=401, step=i)[0] for i in range(a.decode)]
        torch.cuda.synchronize()
        rec = eng.run_sequence(prompt, toks, f"ecr{ecr}")
        tr = rec.trace
        if a.trace_dir:
            Path(a.trace_dir).mkdir(parents=True, exist_ok=True)
            P.save_trace(tr, Path(a.trace_dir) / f"daop_ecr{ecr}.jsonl")
        n = tr.num_decode_tokens
        if exp:
            import gzip
            import tempfile
            with tempfile.NamedTemporaryFile(suffix=".jsonl") as f:
                P.save_trace(tr, f.name)
                (exp / f"trace_ecr{ecr}.jsonl.gz").write_bytes(gzip.compress(Path(f.name).read_bytes()))
            pre = rec.prefill
            (exp / f"engine_ecr{ecr}.json").write_text(json.dumps({
                "ecr": ecr, "engine": "daop", "prediction_start_layer": 4,
                "placement_initial": [sorted(x) for x in pre.placement_initial.on_fast],
                "placement_final": [sorted(x) for x in pre.placement.on_fast],
                "swaps": [[e.layer, e.swapped_in, e.swapped_out, e.hot_tokens, e.cold_tokens]
                          for e in pre.swaps],
                "device_counts": pre.counts.tolist(),
                "executed": [[[int(x) for x in p.executed_experts()] for p in r.plans]
                             for r in rec.decode],
                "devices": [[[x.device for x in p.executed] for p in r.plans] for r in rec.decode],
                "degraded": [[[[dg.dropped_expert, dg.substitute_expert] for dg in p.degraded]
                               for p in r.plans]
                             for r in rec.decode],
                "counts": rec.counts}))
        runs.append({
            "ecr": ecr,
            "slot_budget": eng.placement0.slot_budget,
            "hbm_expert_gb": eng.placement0.slot_budget * 3 * a.d * a.ffn * 2 / 1e9,
            "decode_tokens_per_s": rec.tokens_per_second,
            "decode_ms_per_token": [round(r.ms, 2) for r in rec.decode],
            "decode_host_tier_ms_per_token": eng.host_ms / n,
            "prefill_host_tier_ms": eng.prefill_host_ms,
            "prefill_ms": rec.prefill.ms,
            "prefill_tokens_per_s": a.prompt / (rec.prefill.ms / 1e3),
            "swaps": len(rec.prefill.swaps),
            "prefill_migration_ms": rec.prefill.migration_ms,
            "prefill_migration_hidden_ms": rec.prefill.migration_hidden_ms,
            "prefill_slow_expert_batches": rec.prefill.slow_executions,
            "counts": rec.counts,
            "slow_executions_per_token": rec.counts["slow_executions"] / n,
            "degradations_per_token": rec.counts["degradations"] / n,
            "prediction_accuracy": P.mean_prediction_accuracy(tr),
            "set_fidelity": P.routing_fidelity(
                tr, [[p.executed_experts() for p in r.plans] for r in rec.decode])[0],
        })
        print(json.dumps(runs[-1]), flush=True)
        del eng
        torch.cuda.empty_cache()
    res["runs"] = runs
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        Path(a.out).write_text(s)


if __name__ == "__main__":
    main()
