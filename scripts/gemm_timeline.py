"""Per-CTA timeline of one CTA-pair GEMM launch (daop_gemm_timeline):
entry, setup done, last MMA commit, last epilogue warp -- relative to the
first CTA's entry (development aid).  argv: T [N K]."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2501_10375_b200 import _lib, ops

T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
k = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
a = (torch.randn(T, k, device="cuda") * 0.1).bfloat16()
w = (torch.randn(n, k, device="cuda") * 0.02).bfloat16()
out = torch.empty(T, n, device="cuda")
ws = torch.empty(8 * T * n, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    ops.gemm_bf16_f32(a, w, out=out, ws=ws)
torch.cuda.synchronize()
tl = np.zeros((512, 6), dtype=np.uint64)
for cold in (True, False):
    if cold:
        flush.fill_(1)
    torch.cuda.synchronize()
    _lib.call("daop_gemm_timeline", 1, 0)
    ops.gemm_bf16_f32(a, w, out=out, ws=ws)
    torch.cuda.synchronize()
    _lib.call("daop_gemm_timeline", 0, tl.ctypes.data)
    used = tl[:, 0] > 0
    t = tl[used].astype(np.int64)
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    print(f"T={T} N={n} K={k} {'cold' if cold else 'warm'}: {used.sum()} CTAs")
    for i, name in enumerate(("entry", "setup", "mma_done", "epi_done", "acc_ready", "first_ld")):
        col = r[:, i][t[:, i] > 0]
        if len(col):
            print(f"  {name:9s} min {col.min():6.2f} med {np.median(col):6.2f} max {col.max():6.2f} us")
