"""Prompt-sized dense projections (256-token QKV / O-proj shapes) on the
skinny tcgen05 kernel: cold (L2 flushed) and warm times (development aid)."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2501_10375_b200 import ops

T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
WS = len(sys.argv) > 2 and sys.argv[2] == "ws"  # split-K CTA-pair path instead
import os
if os.environ.get("GEMM_MODE"):  # tuning / diagnostic bits (ops.set_gemm_mode)
    ops.set_gemm_mode(int(os.environ["GEMM_MODE"], 0))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
for name, n, k in (("qkv", 6144, 4096), ("oproj", 4096, 4096)):
    a = (torch.randn(T, k, device="cuda", generator=g) * 0.1).bfloat16()
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.02).bfloat16()
    out = torch.empty(T, n, device="cuda")
    ws = torch.empty(8 * T * n, device="cuda") if WS else None
    for cold in (True, False):
        ts = []
        for _ in range(30):
            if cold:
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.gemm_bf16_f32(a, w, out=out, ws=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = statistics.median(ts[5:])
        print(f"{name} T={T} {'splitK' if WS else 'skinny'} {'cold' if cold else 'warm'} {us:.1f} us  "
              f"{n * k * 2 / us / 1e3:.0f} GB/s weights  {2 * T * n * k / us / 1e6:.0f} TF/s")
    ref = a.float() @ w.float().t()
    print(name, "max|err|", (out - ref).abs().max().item())
