"""BASELINE configs[2] decisions at scale: the UNMODIFIED reference's
run_single on the engine's own 32-layer traces, with the engine's own
calibration (VERDICT r01 "next round" #2).

Input (committed, from a GPU run of `scripts/daop32.py --export-dir`):
  tests/golden/daop32/calib.json              pooled decode probabilities of
                                              the engine's calibration sequence
  tests/golden/daop32/trace_ecr{E}.jsonl.gz   the exported RoutingTrace (true
                                              gates + next-layer predictions,
                                              fp32 widened to float64)
  tests/golden/daop32/engine_ecr{E}.json      what the B200 engine decided
Output:
  tests/golden/daop32/reference_ecr{E}.json   moesim.run_single's placements,
                                              swaps, per-token executed sets,
                                              counters and fidelity

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_daop32_golden.py
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from moesim import default_cost_model, load_trace  # noqa: E402
from moesim.experiment import run_single  # noqa: E402

DIR = Path(__file__).with_name("daop32")


def main():
    calib = np.array(json.loads((DIR / "calib.json").read_text())["calib"])
    cost = default_cost_model()
    for eng_file in sorted(DIR.glob("engine_ecr*.json")):
        eng = json.loads(eng_file.read_text())
        ecr = eng["ecr"]
        raw = gzip.decompress((DIR / f"trace_ecr{ecr}.jsonl.gz").read_bytes())
        with tempfile.NamedTemporaryFile(suffix=".jsonl") as f:
            f.write(raw)
            f.flush()
            trace = load_trace(f.name)
        rec = run_single(trace, calib, ecr, "daop", cost,
                         prediction_start_layer=eng["prediction_start_layer"])
        dec = rec["_decode_result"]
        out = {
            "ecr": ecr,
            "placement_initial": [sorted(s) for s in rec["_placement_initial"].on_fast],
            "placement_final": [sorted(s) for s in rec["_placement_final"].on_fast],
            "swaps": [[s.layer, s.swapped_in, s.swapped_out, s.hot_tokens, s.cold_tokens]
                      for s in rec["_swaps"]],
            "executed": [[list(map(int, ex)) for ex in tok] for tok in dec.executed],
            "counts": {k: int(v) for k, v in dec.counts.items()},
            "set_fidelity": rec["set_fidelity"],
            "score_mass": rec["score_mass"],
            "similarity_prefill_decode": rec["similarity_prefill_decode"],
            "swap_count": rec["swap_count"],
        }
        path = DIR / f"reference_ecr{ecr}.json"
        path.write_text(json.dumps(out))
        print(f"wrote {path}")


if __name__ == "__main__":
    main()
