"""Run the reference simulator (moesim simulate, cli.py:180-192) on routing
traces exported by scripts/daop32.py, once with its default (A100-era)
CostModel and once with the one fitted on the B200 (scripts/fit_cost_model.py),
and set the predictions beside the tokens/s the engine measured.

Container-only analysis (imports the reference from /root/reference):
    python scripts/sim_compare.py --traces gpurun_out/traces \
        --cost gpurun_out/cost_model_b200.json --measured gpurun_out/daop32_trace.json \
        --out profiles/r01/cost_model/sim_compare.json
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

REF = "/root/reference/pkg/src"


def simulate(trace, calib, ecr, cost, out):
    env = dict(os.environ, PYTHONPATH=REF, PYTHONDONTWRITEBYTECODE="1",
               MOESIM_DISABLE_NUMBA="1", NUMBA_CACHE_DIR=tempfile.gettempdir() + "/nb")
    cmd = [sys.executable, "-c", "import sys; from moesim.cli import main; sys.exit(main(sys.argv[1:]))",
           "simulate", "--trace", str(trace), "--calib-trace", str(calib), "--ecr", str(ecr),
           "--engine", "daop", "--out", str(out)]
    if cost:
        cmd += ["--cost-model", str(cost)]
    subprocess.run(cmd, check=True, env=env, cwd=tempfile.gettempdir(), capture_output=True)
    (f,) = Path(out).glob("*.json")
    return json.loads(f.read_text())["decode"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", required=True)
    ap.add_argument("--cost", required=True)
    ap.add_argument("--measured", required=True)
    ap.add_argument("--calib-ecr", default="1.0")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    measured = {r["ecr"]: r for r in json.loads(Path(a.measured).read_text())["runs"]}
    calib = (Path(a.traces) / f"daop_ecr{a.calib_ecr}.jsonl").resolve()
    rows = []
    with tempfile.TemporaryDirectory() as tmp:
        for ecr, m in sorted(measured.items()):
            trace = (Path(a.traces) / f"daop_ecr{ecr}.jsonl").resolve()
            d = simulate(trace, calib, ecr, None, Path(tmp) / f"d{ecr}")
            b = simulate(trace, calib, ecr, Path(a.cost).resolve(), Path(tmp) / f"b{ecr}")
            n = b["num_tokens"]
            rows.append({"ecr": ecr, "measured_tok_s": m["decode_tokens_per_s"],
                         "sim_b200_cost_tok_s": b["tokens_per_second"],
                         "sim_default_cost_tok_s": d["tokens_per_second"],
                         "measured_over_sim_b200": m["decode_tokens_per_s"] / b["tokens_per_second"],
                         "sim_slow_executions_per_token": b["counts"]["slow_executions"] / n,
                         "measured_slow_executions_per_token": m["slow_executions_per_token"],
                         "sim_degradations_per_token": b["counts"]["degradations"] / n,
                         "measured_degradations_per_token": m["degradations_per_token"]})
    res = {"cost_model_b200": json.loads(Path(a.cost).read_text()),
           "note": "simulator calibrated on the ECR %s trace's decode phase; the engine on its own "
                   "calibration sequence, so placements (and slow counts) can differ" % a.calib_ecr,
           "runs": rows}
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
