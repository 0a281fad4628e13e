"""Measured B200 cost model for the reference simulator.

`moesim` prices a decode token with `CostModel` (moesim/simulator.py:38-96):
seven per-token durations / parallelism fields, read by `moesim simulate
--cost-model file.json` through `CostModel.from_json_obj` (`:88-92`, unknown
fields are a ConfigError, `__post_init__` rejects negatives and
slow_parallelism < 1, `:64-76`).  Its defaults are A100-era figures.  This
module fills the same fields from kernels timed on this GPU, so the
reference's analysis tools run on numbers the B200 path actually achieves:

  t_nonmoe_fast      attention block (RMSNorm + QKV + attention over `ctx`
                     cached positions + O-proj + residual), one token-layer
  t_expert_fast      one expert of one token on the GPU: (decode layer with
                     k picks - router alone) / k  -- the decode kernel fuses
                     the gate, so the router is priced separately
  t_expert_slow      one expert of one token on the host tier (AVX-512 BF16 /
                     AMX GEMV over pinned memory, all host threads)
  t_gate             the router for one token (RMSNorm, own + next gate)
  t_migrate_expert   one expert [W1|W3|W2] pinned host -> HBM slot
  t_activation_xfer  one direction of a d-vector (bf16) host <-> device
  slow_parallelism   host experts in flight at once (the host tier runs one
                     expert at a time over every core -> 1)

GPU durations are CUDA-event means over a CUDA-graph replay of `reps` calls
(kernel time, not Python launch time) after warm-up;
host durations are perf_counter medians.  All in milliseconds.
"""

from __future__ import annotations

import json
import os
import statistics
import time

import numpy as np
import torch

from . import ops
from .errors import ConfigError

# moesim/simulator.py:78-86 (CostModel._SCALAR_FIELDS), same order
FIELDS = ("t_nonmoe_fast", "t_expert_fast", "t_expert_slow", "t_gate", "t_migrate_expert",
          "t_activation_xfer", "slow_parallelism")
_NONNEG = FIELDS[:-1]


def validate(obj: dict) -> dict:
    """The checks `CostModel.from_json_obj` + `__post_init__` apply
    (moesim/simulator.py:64-76,88-92), so a file we write loads there.
    Stricter on two points the reference lets through: NaN durations and a
    non-integer slow_parallelism are rejected too."""
    unknown = set(obj) - set(FIELDS)
    if unknown:
        raise ConfigError(f"unknown cost model fields: {sorted(unknown)}")
    for name in _NONNEG:
        if name in obj and not obj[name] >= 0:
            raise ConfigError(f"{name} must be >= 0")
    if "slow_parallelism" in obj:
        sp = obj["slow_parallelism"]
        if not isinstance(sp, int) or isinstance(sp, bool) or sp < 1:
            raise ConfigError("slow_parallelism must be >= 1")
    return obj


def save(obj: dict, path) -> None:
    """Write the `--cost-model` JSON (only the reference's fields)."""
    obj = validate({k: v for k, v in obj.items() if k != "_detail"})
    with open(path, "w") as fh:
        json.dump(obj, fh, indent=2, sort_keys=True)
        fh.write("\n")


def load(path) -> dict:
    with open(path) as fh:
        return validate(json.load(fh))


def _gpu_ms(fn, reps: int, warmup: int = 3, graph: bool = True) -> float:
    """Device time of one fn() call.  The calls are captured into one CUDA
    graph and the replay is timed, so host-side launch cost (allocation,
    ctypes) is not mistaken for kernel time."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    run = fn
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                fn()
        run = g.replay
        g.replay()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    if graph:
        run()
    else:
        for _ in range(reps):
            run()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / reps


def _host_ms(fn, reps: int, warmup: int = 2) -> float:
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


def measure(d: int = 4096, ffn: int = 14336, k: int = 2, num_experts: int = 8, ctx: int = 512,
            n_heads: int = 32, n_kv: int = 8, seed: int = 0, reps: int = 50,
            host_reps: int = 5, host_threads: int = 0, device="cuda") -> dict:
    """Time every CostModel field on the current GPU / host at the given
    model shape.  Returns {field: value, ..., "_detail": {...}}; `save`
    drops `_detail`."""
    from .attention import AttentionStack
    from .daop import HostExpertPool, host_expert_ffn
    from .engine import MoEBlockEngine
    from .model import MoEModel
    from .trace import ModelShape

    dev = torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    torch.cuda.set_device(dev)
    shape = ModelShape(2, num_experts, k)
    # layer 0 resident (k picks stream from HBM), layer 1 only for the next gate
    model = MoEModel(shape, d, ffn, seed=seed, device=dev, resident_layers=[0])
    eng = MoEBlockEngine(model)
    h = model.input_hidden(1, stream=7)[0].contiguous()
    h2 = h.view(1, d)
    t_layer = _gpu_ms(lambda: eng.decode(h, 0), reps)
    t_gate = _gpu_ms(lambda: ops.router(h2, model.norm[0], model.gate[0], model.gate[1], k),
                     reps)
    t_fast = max(t_layer - t_gate, 0.0) / k

    attn = AttentionStack(1, d, n_heads, n_kv, max_seq=max(ctx + 1, 64), seed=seed, device=dev)
    out = torch.empty_like(h)
    t_nonmoe = _gpu_ms(lambda: attn.decode(h, 0, ctx, out), reps)
    del attn

    # one expert's bytes, pinned host -> a free slot (HostExpertPool layout)
    pool = HostExpertPool(ModelShape(1, 2, 1), d, ffn, seed=seed, threads=host_threads or None)
    src = pool.slot(0, 0)
    dst = torch.empty_like(src, device=dev)
    t_mig = _gpu_ms(lambda: dst.copy_(src, non_blocking=True), max(3, reps // 10), warmup=2,
                    graph=False)
    del dst

    xh = torch.zeros(d, dtype=torch.bfloat16, pin_memory=True)
    xd = torch.empty(d, dtype=torch.bfloat16, device=dev)

    def xfer():  # what the engine pays per direction: copy + wait for it
        xd.copy_(xh, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    t_x = _host_ms(xfer, reps)

    x1 = np.asarray(model.input_hidden(1, stream=8).to(torch.bfloat16).view(torch.int16).cpu()
                    ).view(np.uint16)
    t_slow = _host_ms(lambda: host_expert_ffn(pool, 0, 0, x1, host_threads), host_reps)
    res = {"t_nonmoe_fast": t_nonmoe, "t_expert_fast": t_fast, "t_expert_slow": t_slow,
           "t_gate": t_gate, "t_migrate_expert": t_mig, "t_activation_xfer": t_x,
           "slow_parallelism": 1}
    res["_detail"] = {
        "gpu": torch.cuda.get_device_name(dev), "d": d, "ffn": ffn, "top_k": k,
        "num_experts": num_experts, "attention_ctx": ctx, "n_heads": n_heads, "n_kv": n_kv,
        "decode_layer_ms": t_layer, "expert_bytes": int(src.numel() * 2),
        "migrate_gb_s": src.numel() * 2 / t_mig / 1e6,
        "host_threads": host_threads or len(os.sched_getaffinity(0)),
        "reps": reps, "host_reps": host_reps}
    return res
