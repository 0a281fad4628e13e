"""Fit moesim's CostModel from kernels timed on this B200.

    python scripts/fit_cost_model.py [--out cost_model_b200.json] [--ctx 512]

Writes the `moesim simulate --cost-model` JSON (the reference's seven fields
only) and, beside it, `<out>.detail.json` with the shape and raw timings.
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2501_10375_b200 import costmodel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/cost_model_b200.json")
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    res = costmodel.measure(d=a.d, ffn=a.ffn, ctx=a.ctx, reps=a.reps)
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    costmodel.save(res, out)
    out.with_suffix(".detail.json").write_text(json.dumps(res, indent=2, sort_keys=True) + "\n")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
