"""DAOP decode at ECR 0.5 (32 layers, host tier): where the token time goes.
Runs the bench's configs[2] flow once (calibration, init, prefill), then
decodes with several host-tier thread counts and reports tokens/s, the host
tier's busy time per token and its per-expert time in situ (development aid,
GPU box; bench.py `daop` is the measurement)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200.daop import DaopEngine, HostExpertPool, host_expert_ffn  # noqa: E402

L, E, K, D, FFN = 32, 8, 2, 4096, 14336
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
eng = DaopEngine(shape, D, FFN, calib, 0.5, P.PolicyConfig("daop"), seed=0, host_pool=pool)
prompt = eng.model.input_hidden(256, stream=400)
eng.prefill(prompt)
toks = [eng.model.input_hidden(1, stream=401, step=i)[0] for i in range(24)]
xs = np.random.default_rng(0).standard_normal((1, D)).astype(np.float32)
ncpu = len(os.sched_getaffinity(0))
configs = [(0, 0), (0, 4096), (0, 3072), (0, 5120), (0, 0), (0, 4096)]
if len(sys.argv) > 1 and sys.argv[1] == "threads":
    configs = [(0, 0), (ncpu - 1, 0), (ncpu, 0), (2 * ncpu, 0), (0, 0)]
for th, split in configs:
    # standalone per-expert time at this thread count
    t0 = time.perf_counter()
    for e in range(8):
        host_expert_ffn(pool, 5, e, xs, th)
    solo = (time.perf_counter() - t0) / 8 * 1e3
    eng.host_threads = th
    eng.slow_split_rows = split
    eng.host_ms = 0.0
    for t in toks[:4]:
        eng.decode(t)
    eng.host_ms = 0.0
    slow = 0
    t0 = time.perf_counter()
    n = 12
    for t in toks[4:4 + n]:
        r = eng.decode(t)
        slow += sum(1 for lp in r.plans for ex in lp.executed if ex.device == "slow")
    dt = (time.perf_counter() - t0) / n * 1e3
    print(f"host_threads {th or ncpu:3d} gpu split rows {split:5d}: {1e3 / dt:6.2f} tok/s, "
          f"{dt:6.1f} ms/token, host tier busy {eng.host_ms / n:6.1f} ms/token, {slow / n:5.1f} "
          f"slow/token -> {eng.host_ms / max(slow, 1):5.2f} ms/expert in situ (host alone, solo "
          f"{solo:5.2f})", flush=True)
