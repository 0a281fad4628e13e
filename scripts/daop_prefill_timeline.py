"""DAOP prefill at ECR < 1 (32 layers, host tier, 256-token prompt): per-layer
wall-clock timeline -- waiting for the GPU (histogram / offsets syncs), the
host tier, swaps -- to see what the prefill's critical path is (development
aid, GPU box)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.daop import DaopEngine, HostExpertPool  # noqa: E402

L, E, K, D, FFN = 32, 8, 2, 4096, 14336
ecr = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
shape = P.ModelShape(L, E, K)
pool = HostExpertPool(shape, D, FFN, seed=0, device=torch.device("cuda"))
cal = DaopEngine(shape, D, FFN, np.full((L, E), K / E), 1.0, P.PolicyConfig("daop"), seed=0,
                 host_pool=pool)
crec = cal.run_sequence(cal.model.input_hidden(64, stream=300),
                        [cal.model.input_hidden(1, stream=301, step=i)[0] for i in range(16)],
                        "calib")
calib = P.pooled_decode_probabilities([crec.trace])
del cal, crec
torch.cuda.empty_cache()
for rep in range(4):
    eng = DaopEngine(shape, D, FFN, calib, ecr, P.PolicyConfig("daop"), seed=0, host_pool=pool)
    eng.prefill_serial_migrations = rep % 2 == 0  # A/B on the same box
    eng.prefill_trace = []
    eng.prefill_host_ms = 0.0
    prompt = eng.model.input_hidden(256, stream=400)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pre = eng.prefill(prompt)
    wall = 1e3 * (time.perf_counter() - t0)
    tr = eng.prefill_trace
    tot = {"gpu_wait_hist": 0.0, "gpu_wait_offsets": 0.0, "host": 0.0, "rest": 0.0}
    for t in tr:
        a = t["t0"]
        hs = t.get("hist_synced", a)
        os_ = t.get("offsets_synced", hs)
        h0, h1 = t.get("host_start", os_), t.get("host_end", os_)
        tot["gpu_wait_hist"] += hs - a
        tot["gpu_wait_offsets"] += os_ - hs
        tot["host"] += h1 - h0
        tot["rest"] += (t["t1"] - a) - (hs - a) - (os_ - hs) - (h1 - h0)
    print(f"rep {rep} {'serial ' if eng.prefill_serial_migrations else 'overlap'} ECR {ecr}: prefill {wall:.1f} ms, host tier {eng.prefill_host_ms:.1f} ms, "
          f"migrations {pre.migration_ms:.1f} ms (hidden {pre.migration_hidden_ms:.1f}), "
          f"swaps {len(pre.swaps)}, slow execs {pre.slow_executions}", flush=True)
    print("   wall-clock components (ms):", {k: round(1e3 * v, 1) for k, v in tot.items()})
    keys = ["t0", "hist_synced", "alg1_done", "swaps_queued", "offsets_synced", "xs_queued",
            "gemms_queued", "host_start", "host_end", "t1"]
    seg = {}
    for t in tr:
        prev = t["t0"]
        for k_ in keys[1:]:
            if k_ in t:
                seg[k_] = seg.get(k_, 0.0) + 1e3 * (t[k_] - prev)
                prev = t[k_]
    print("   per-segment totals (ms, ending at):", {k_: round(v, 1) for k_, v in seg.items()})
    if rep == 3:
        for t in tr:
            a = t["t0"]
            print(f"   L{t['layer']:2d} {1e3 * (t['t1'] - a):6.1f} ms  wait-hist "
                  f"{1e3 * (t.get('hist_synced', a) - a):5.1f}  wait-off "
                  f"{1e3 * (t.get('offsets_synced', a) - t.get('hist_synced', a)):5.1f}  host "
                  f"{1e3 * (t.get('host_end', a) - t.get('host_start', a)):5.1f}  swaps {t['swaps']} "
                  f"slow {t['slow']} rows {t['slow_rows']}")
