#!/usr/bin/env python
"""Benchmark of the B200-native DAOP MoE-block hot path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload (BASELINE.json configs[1]): ONE Mixtral-8x7B-shaped MoE
layer (d=4096, ffn=14336, E=8, top-2), bf16 weights, decode batch 1 on one
B200, all 8 experts resident in HBM.  A step = one decode token through the
layer = one persistent kernel launch (fused router + selection + SwiGLU
expert GEMV streaming both picked experts' 704.8 MB + combine).  Every step
takes a fresh token, so the picked experts change step to step; the 2.8 GB
of expert weights exceed the 126 MB L2, so no L2 flush is needed.

  value  tokens/s with the token already in HBM (device clock, max over ranks)
  e2e    tokens/s through the public host API with host buffers every step:
         MoEBlockEngine.decode_server().step (persistent kernel: h pulled from
         pinned memory on a doorbell, residual + picks written back to pinned
         memory) -- e2e_launch is the launch-per-call MoEBlockEngine.decode_host
  roofline  HBM: algorithmic bytes per launch / CUDA-event launch duration,
            against MEASURED_PEAKS.json hbm_gbs (driver-measured copy peak)
  prefill   BASELINE configs[3]: 8 sequences x 4096 tokens through the same
            layer (router, permutation, tcgen05 grouped GEMMs, combine),
            tensor roofline against the measured bf16 peak
  cpu_baseline  the oracle CPU path (oracle/baseline.py) on this host's cores
            for a bounded sample of the same workload

--impl reference times that CPU path alone as the reference arm (the
reference package itself executes no numerics -- SPEC.md:347,356 -- so its
own algorithm restated in oracle/ is the arm).
With N > 1 (torchrun) the headline is expert parallelism (run_b200_ep,
BASELINE configs[4], strong scaling): a Mixtral-8x22B-shaped layer, the
prompt's tokens and the experts sharded over the ranks, dispatch / return
over NVLink peer memory (`--ep-headline` runs that path on one GPU).

  ep        BASELINE configs[4]: a Mixtral-8x22B-shaped layer, prefill of
            8 x 4096 tokens sharded over the N ranks, experts sharded E/N per
            rank, expert-parallel with NCCL over NVLink (strong scaling; at
            N = 1 the same path without a collective)
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE decode tokens/s & prefill tokens/s (Mixtral-8x7B shape), % HBM/tensor roofline"
D, FFN, E, K = 4096, 14336, 8, 2
DECODE_BYTES = 2 * 3 * D * FFN * 2 + 2 * E * D * 2          # 704,774,144 B per token-layer
PREFILL_SEQS, PREFILL_LEN = 8, 4096


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int, period_s: float = 0.01):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        import statistics
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def ncu_traffic():
    """dram bytes per launch of the decode kernel from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_decode_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


# ------------------------------------------------------------------ reference arm


def cpu_decode_layer():
    from oracle.baseline import CpuMoELayer
    return CpuMoELayer(2, E, K, D, FFN, seed=0, layer=0, with_bf16=True)


def cpu_inputs(n, rank=0):
    from oracle import numerics as N
    return [N.input_hidden(0, 100 + rank, i, 1, D)[0] for i in range(n)]


def cpu_arm(layer, xs, steps, warmup, budget_s, fns=None, tokens_per_step=1,
            what="decode tokens through one Mixtral-8x7B layer"):
    """Time the CPU path: the faster of the oracle's numpy fp32 restatement and
    the torch-CPU bf16 (oneDNN, fp32 accumulation) deployment of the same
    block, each on all host cores (decided on 2 calibration steps); both
    numbers are reported."""
    from oracle.baseline import blas_threads, cpu_model, time_steps
    cand = fns or {"numpy_f32": layer.decode_step, "torch_bf16": layer.decode_step_bf16,
                   "c_bf16": layer.decode_step_c}
    probe = {}
    for name, fn in cand.items():
        n, sec = time_steps(fn, xs, budget_s=5.0, max_steps=2, warmup=1)
        probe[name] = tokens_per_step * n / sec
    best = max(probe, key=probe.get)
    n, sec = time_steps(cand[best], xs, budget_s=budget_s, max_steps=steps, warmup=warmup)
    desc = {"numpy_f32": "oracle numpy fp32 on bf16-valued weights",
            "torch_bf16": "torch-CPU bf16 weights/activations, oneDNN fp32 accumulation",
            "c_bf16": "oracle C (oracle/cpu_moe.c) on bf16 weights, fp32 accumulation, "
                      "OpenMP"}[best]
    cores = layer.c_threads() if best == "c_bf16" else blas_threads()
    return {"value": tokens_per_step * n / sec, "unit": "tokens/s", "cores": cores,
            "kind": "port", "cpu_model": cpu_model(), "variant": best,
            "variants_tok_s": {k: round(v, 2) for k, v in probe.items()},
            "sample": f"{n} steps of {tokens_per_step} x {what} ({desc}, {sec:.1f} s)",
            "steps": n, "seconds": sec}


def workload_config(world):
    """The config dict both arms print (same workload, same keys)."""
    if world > 1:
        return {"workload": f"Mixtral-8x22B-shaped MoE layer (d={EP_D}, ffn={EP_FFN}, E={E}, "
                            f"top-{K}), prefill {EP_TOKENS} tokens sharded over {world} GPUs, "
                            f"expert-parallel (BASELINE configs[4])",
                "d_model": EP_D, "d_ff": EP_FFN, "experts": E, "top_k": K,
                "global_batch": EP_TOKENS, "parallelism": f"ep{world}",
                "l2": "inputs larger than L2 (4.8 GB of experts per layer)"}
    return {"workload": "decode b=1, one Mixtral-8x7B MoE layer (BASELINE configs[1])",
            "d_model": D, "d_ff": FFN, "experts": E, "top_k": K, "global_batch": 1,
            "parallelism": "single",
            "l2": "inputs larger than L2 (2.8 GB of experts, 704.8 MB streamed per step)"}


def run_reference(args, world, rank):
    if rank != 0:
        return None
    if world > 1:
        # our arm's N > 1 workload: the Mixtral-8x22B layer's prefill; the CPU
        # runs a bounded sample of it (64 prompt tokens per step)
        from oracle.baseline import CpuMoELayer
        from oracle import numerics as N
        layer = CpuMoELayer(2, E, K, EP_D, EP_FFN, seed=0, layer=0, with_bf16=True)
        xs = [N.input_hidden(0, 300, i, 64, EP_D) for i in range(2)]
        cb = cpu_arm(layer, xs, steps=args.steps, warmup=args.warmup, budget_s=90.0,
                     fns={"numpy_f32": layer.prefill, "torch_bf16": layer.prefill_bf16,
                          "c_bf16": layer.prefill_c},
                     tokens_per_step=64, what="64 prompt tokens through one Mixtral-8x22B layer")
    else:
        layer = cpu_decode_layer()
        xs = cpu_inputs(16)
        cb = cpu_arm(layer, xs, steps=args.steps, warmup=args.warmup, budget_s=60.0)
    v = cb["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
        "n_gpus": world, "steps": cb["steps"], "warmup": args.warmup,
        "ms_per_step": 1e3 * cb["seconds"] / cb["steps"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if cb["variant"] == "numpy_f32" else "bf16",
        "data": "synthetic (counter-RNG random-init weights and tokens)",
        "config": workload_config(world),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "cpu_model",
                                              "variant", "variants_tok_s", "sample")},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if world > 1:
        line["scaling"] = "strong"
        line["note"] = "rank 0 alone runs the host CPU path; the other ranks exit without work"
    return line


# ------------------------------------------------------------------ B200 arm


def run_b200(args, world, rank, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.model import MoEModel

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    hbm_peak, tf_peak, tf_sus, peak_kind = peaks()
    # the full 32-layer Mixtral-8x7B expert set (90.2 GB) is resident in HBM;
    # the headline and prefill use layer 0, decode32 runs every layer
    n_layers = 2 if args.no_decode32 else 32
    model = MoEModel(P.ModelShape(n_layers, E, K), D, FFN, seed=0, device=dev)
    eng = MoEBlockEngine(model)
    n_in = 64
    hs = [model.input_hidden(1, stream=100 + rank, step=i)[0] for i in range(n_in)]
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # decisions of the first tokens, for the free-running routing agreement
    # the cpu_baseline leg reports (untimed)
    dec_sel = []
    for i in range(n_in):
        dec_sel.append(eng.decode(hs[i]).sel.clone())
    dec_sel = torch.stack(dec_sel).cpu().numpy()

    # -------- device-resident timed loop (value)
    for i in range(args.warmup):
        eng.decode(hs[i % n_in])
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            eng.decode(hs[i % n_in])
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * args.steps / (ms_max / 1e3)

    # -------- per-launch kernel duration for the roofline (events around each launch)
    nl = min(args.steps, 200)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(nl)]
    torch.cuda.synchronize()
    for i in range(nl):
        evs[i][0].record(stream)
        eng.decode(hs[i % n_in])
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    launch_ms = sorted(a.elapsed_time(b) for a, b in evs)
    launch_ms_mean = float(np.mean(launch_ms))
    # achieved over the timed region (one launch per step, back to back); the
    # event-bracketed single launches above add their own gaps and are
    # reported beside it
    achieved = DECODE_BYTES / (ms_max / args.steps / 1e3) / 1e9

    # -------- prefill (BASELINE configs[3]: 8 x 4096 tokens)
    prefill = None
    pf_sample = None
    if not args.no_prefill:
        T = PREFILL_SEQS * PREFILL_LEN
        hp = model.input_hidden(T, stream=200 + rank)
        hist = torch.zeros((PREFILL_SEQS, n_layers, E), dtype=torch.int32, device=dev)
        for _ in range(2):
            rp = eng.prefill(hp, 0, hist=hist[:, 0], tokens_per_seq=PREFILL_LEN,
                             hist_seq_stride=n_layers * E)
        # one sequence's routing, for the free-running agreement (untimed)
        pf_sample = {"h": hp[:PREFILL_LEN].cpu().numpy(),
                     "sel": rp["topk_idx"][:PREFILL_LEN].cpu().numpy(),
                     "x": rp["x"][:PREFILL_LEN].float().cpu().numpy()}
        del rp
        barrier()
        torch.cuda.synchronize()
        # 10 back-to-back layers (~170 ms): the power-capped regime the
        # sustained bf16 peak is measured in, whatever --steps is
        kp = 10
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local_rank) as pclk:
            p0.record(stream)
            for _ in range(kp):
                eng.prefill(hp, 0, hist=hist[:, 0], tokens_per_seq=PREFILL_LEN,
                            hist_seq_stride=n_layers * E)
            p1.record(stream)
            torch.cuda.synchronize()
        pms = p0.elapsed_time(p1) / kp
        tp = torch.tensor([pms], device=dev)
        if world > 1:
            dist.all_reduce(tp, op=dist.ReduceOp.MAX)
        pms = float(tp.item())
        flops = 2.0 * K * T * 3 * D * FFN
        prefill = {
            "workload": f"prefill {PREFILL_SEQS} x {PREFILL_LEN} tokens, one layer (BASELINE configs[3])",
            "value": world * T / (pms / 1e3), "unit": "tokens/s", "ms_per_layer": pms,
            # a prefill step is a long back-to-back run of tensor-core GEMMs
            # (power-capped like cuBLAS's sustained run): the sustained
            # measured peak is the denominator, the burst fraction is beside it
            "roofline": {"bound": "tensor", "achieved": flops / (pms / 1e3) / 1e12,
                         "peak": tf_sus, "unit": "TFLOP/s",
                         "frac": flops / (pms / 1e3) / 1e12 / tf_sus,
                         "peak_kind": f"{peak_kind} sustained",
                         "frac_of_burst": flops / (pms / 1e3) / 1e12 / tf_peak,
                         "flops_per_layer": flops},
            "gpu_launches": kp * MoEBlockEngine.prefill_kernels(),
            "layers_timed": kp, "clocks": pclk.summary(),
        }
        del hp

    # -------- batched decode: 64 sequences' next tokens through the same layer
    # (router -> permutation -> skinny tcgen05 GEMMs -> combine)
    decode_b64 = None
    try:
        B = 64
        hb = model.input_hidden(B, stream=500 + rank)
        for _ in range(3):
            rb = eng.prefill(hb, 0)
        torch.cuda.synchronize()
        active = int((rb["offsets"][1:] - rb["offsets"][:-1] > 0).sum())
        # one CUDA graph per step (router, permutation, GEMMs, combine), replayed
        # like a serving loop would: the step's kernels without Python in between
        gb = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            eng.prefill(hb, 0)
            with torch.cuda.graph(gb):
                eng.prefill(hb, 0)
        stream.wait_stream(side)
        gb.replay()
        torch.cuda.synchronize()
        nb_ = 50
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(nb_):
            gb.replay()
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / nb_
        tb_ = torch.tensor([bms], device=dev)
        if world > 1:
            dist.all_reduce(tb_, op=dist.ReduceOp.MAX)
        bms = float(tb_.item())
        wbytes = active * 3 * D * FFN * 2 + 2 * E * D * 2
        decode_b64 = {
            "workload": "decode step of 64 sequences (b=64) through one Mixtral-8x7B MoE layer: "
                        "router, permutation, skinny tcgen05 grouped GEMMs (weights as the M "
                        "side), combine; one CUDA graph per step",
            "value": world * B / (bms / 1e3), "unit": "tokens/s", "ms_per_step": bms,
            "active_experts": active,
            "roofline": {"bound": "hbm", "achieved": wbytes / (bms / 1e3) / 1e9,
                         "peak": hbm_peak, "unit": "GB/s",
                         "frac": wbytes / (bms / 1e3) / 1e9 / hbm_peak,
                         "bytes_per_step": wbytes},
            "gpu_launches_per_step": MoEBlockEngine.prefill_kernels(B),
        }
        del hb, rb, gb
    except Exception as exc:
        decode_b64 = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # -------- end-to-end through the host API (value measured with host buffers)
    hh = [torch.empty(D, dtype=torch.float32, pin_memory=True) for _ in range(8)]
    for i, h in enumerate(hh):
        h.copy_(hs[i].cpu())
    h2d, d2h = MoEBlockEngine.host_bytes(D, K)
    ne = min(args.steps, 1000)
    for i in range(min(args.warmup, 20)):
        eng.decode_host(hh[i % 8])
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(ne):
        eng.decode_host(hh[i % 8])
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    te = torch.tensor([max(e0.elapsed_time(e1) / 1e3, wall)], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = world * ne / float(te.item())

    # -------- the same calls through the persistent decode server (no launch,
    # no stream synchronisation per call; MoEBlockEngine.decode_server)
    e2e_server = None
    try:
        if args.no_server:
            raise RuntimeError("skipped (--no-server)")
        with eng.decode_server() as srv:
            for i in range(min(args.warmup, 20)):
                srv.step(hh[i % 8])
            t0 = time.perf_counter()
            for i in range(ne):
                srv.step(hh[i % 8])
            wall_s = time.perf_counter() - t0
        ts = torch.tensor([wall_s], device=dev)
        if world > 1:
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        e2e_server = {"value": world * ne / float(ts.item()), "unit": "tokens/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "api": "MoEBlockEngine.decode_server().step (persistent kernel, "
                             "host doorbell, result in pinned host memory)"}
    except Exception as exc:
        e2e_server = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    torch.cuda.synchronize()

    # -------- 32-layer decode token (BASELINE configs[2], ECR 1.0: all experts in HBM)
    decode32 = None
    if not args.no_decode32:
        start = 4
        g, g_in, g_out = eng.capture_decode_graph(start=start, daop=True)
        for i in range(3):
            g_in.copy_(hs[i])
            g.replay()
        barrier()
        torch.cuda.synchronize()
        nt = max(10, min(100, args.steps // 20))
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for i in range(nt):
            g_in.copy_(hs[i % n_in])
            g.replay()
        d1.record(stream)
        torch.cuda.synchronize()
        tok_ms = d0.elapsed_time(d1) / nt
        td = torch.tensor([tok_ms], device=dev)
        if world > 1:
            dist.all_reduce(td, op=dist.ReduceOp.MAX)
        tok_ms = float(td.item())
        bytes_tok = 32 * DECODE_BYTES - 2 * E * D  # no next-layer gate after the last layer
        decode32 = {
            "workload": "decode b=1 through 32 Mixtral-8x7B MoE layers (BASELINE configs[2]), "
                        "ECR 1.0, DAOP plans from layer 4 (prediction-driven selection, "
                        "graceful degradation), one CUDA graph per token",
            "value": world * 1e3 / tok_ms, "unit": "tokens/s", "ms_per_token": tok_ms,
            "roofline": {"bound": "hbm", "achieved": bytes_tok / (tok_ms / 1e3) / 1e9,
                         "peak": hbm_peak, "unit": "GB/s",
                         "frac": bytes_tok / (tok_ms / 1e3) / 1e9 / hbm_peak,
                         "bytes_per_token": bytes_tok},
            "gpu_launches": nt * 32,
        }

    # -------- full decoder layers: attention with a KV cache + MoE (32 layers)
    decoder32 = None
    if not args.no_decode32:
        try:
            decoder32 = run_decoder32(args, world, dev, eng, model, hs, hbm_peak, barrier)
        except Exception as exc:
            decoder32 = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # -------- expert parallelism (BASELINE configs[4]: Mixtral-8x22B shape)
    ep = None
    if not args.no_ep:
        del eng, model
        torch.cuda.empty_cache()
        # decode first: the short HBM-bound run is not measured on a GPU left
        # hot by the prefill GEMMs
        try:
            ep_dec = run_ep_decode(args, world, rank, dev, hbm_peak, barrier)
        except Exception as exc:
            ep_dec = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            ep = run_ep(args, world, rank, dev, tf_sus, barrier, impl="peer")
        except Exception as exc:  # keep the headline line if this section fails
            ep = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            ep_nccl = run_ep(args, world, rank, dev, tf_sus, barrier, impl="nccl")
        except Exception as exc:
            ep_nccl = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        if isinstance(ep, dict):
            ep["nccl_baseline"] = ep_nccl
        if isinstance(ep, dict):
            ep["decode"] = ep_dec
        try:
            ep_b64 = run_ep(args, world, rank, dev, tf_sus, barrier, impl="peer", tokens=64,
                            hbm_peak=hbm_peak)
        except Exception as exc:
            ep_b64 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        if isinstance(ep, dict):
            ep["decode_b64"] = ep_b64

    # -------- DAOP at ECR < 1 (BASELINE configs[2]): 32 layers, slow tier on the host
    daop = None
    if not args.no_daop:
        try:
            daop = run_daop(args, dev, rank)
        except Exception as exc:
            daop = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()

    # -------- CPU baseline (rank 0, N = 1 only) + free-running routing agreement
    cpu = None
    agreement = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        layer = cpu_decode_layer()
        xs = cpu_inputs(16)
        cpu = cpu_arm(layer, xs, steps=200, warmup=1, budget_s=20.0)
        for key in ("steps", "seconds"):
            cpu.pop(key)
        agreement = routing_agreement(layer, [h.cpu().numpy() for h in hs], dec_sel, pf_sample)
        del layer

    if rank != 0:
        return None
    e2e_launch = {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                  "d2h_bytes_per_step": d2h,
                  "api": "MoEBlockEngine.decode_host (one CUDA graph launch + sync per call)"}
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-RNG random-init weights and tokens)",
        "config": workload_config(1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": ncu_traffic(),
                     "peak_kind": peak_kind, "bytes_per_launch": DECODE_BYTES,
                     "launch_us_mean": launch_ms_mean * 1e3,
                     "launch_us_p50": launch_ms[len(launch_ms) // 2] * 1e3,
                     "frac_of_8tbs": achieved / 8000.0},
        "cpu_baseline": cpu,
        # headline end-to-end: the serving call (persistent kernel), when it ran;
        # the launch-per-call host API beside it
        "e2e": (dict(e2e_server) if e2e_server and "value" in e2e_server else e2e_launch),
        "e2e_launch": e2e_launch,
        "e2e_server": e2e_server,
        "gpu_launches": args.steps,
        "clocks": clocks,
        "prefill": prefill,
        "decode_b64": decode_b64,
        "decode32": decode32,
        "decoder32": decoder32,
        "ep": ep,
        "daop": daop,
        "routing_agreement": agreement,
    }
    line["summary"] = summarize(line)  # last key: survives a truncated stdout tail
    return line


def _g(d, *path):
    for p in path:
        if not isinstance(d, dict) or p not in d:
            return None
        d = d[p]
    return round(d, 4) if isinstance(d, float) else d


def summarize(line):
    """Compact copy of every section's headline number."""
    dr = _g(line, "daop", "runs") or []
    return {
        "decode_tok_s": _g(line, "value"), "decode_frac": _g(line, "roofline", "frac"),
        "e2e_tok_s": _g(line, "e2e", "value"), "cpu_tok_s": _g(line, "cpu_baseline", "value"),
        "prefill_ms_layer": _g(line, "prefill", "ms_per_layer"),
        "prefill_frac_sustained": _g(line, "prefill", "roofline", "frac"),
        "prefill_frac_burst": _g(line, "prefill", "roofline", "frac_of_burst"),
        "decode_b64_ms": _g(line, "decode_b64", "ms_per_step"),
        "decode_b64_frac": _g(line, "decode_b64", "roofline", "frac"),
        "decode32_tok_s": _g(line, "decode32", "value"),
        "decode32_frac": _g(line, "decode32", "roofline", "frac"),
        "decoder32_tok_s": _g(line, "decoder32", "value"),
        "decoder32_frac": _g(line, "decoder32", "roofline", "frac"),
        "ep_prefill_ms": _g(line, "ep", "ms_per_layer"),
        "ep_prefill_frac": _g(line, "ep", "roofline", "frac"),
        "ep_decode_b64_ms": _g(line, "ep", "decode_b64", "ms_per_step"),
        "ep_decode_b1_ms": _g(line, "ep", "decode", "ms_per_step"),
        "daop": [{"ecr": r.get("ecr"), "tok_s": _g(r, "tokens_per_second"),
                  "slow_per_tok": _g(r, "slow_executions_per_token"),
                  "prefill_ms": _g(r, "prefill_latency_ms")} for r in dr],
        "routing_agreement": {k: _g(line, "routing_agreement", k, "agree_frac")
                              for k in ("decode", "prefill")},
    }


def routing_agreement(layer, hs, dec_sel, pf_sample):
    """Free-running routing of the GPU vs the CPU oracle on the same h
    (moesim/_kernels.py:63-79 tie rule): the oracle computes x = RMSNorm(h),
    p and top-k from h alone.  Disagreeing rows are reported, split into
    near ties (oracle top-(k+1) gap < 1e-5) and the rest (should be 0)."""
    import numpy as np
    from oracle import decisions as Dd
    from oracle import numerics as N

    def rows(h, sel_gpu, x_gpu=None):
        x = N.rmsnorm(h, layer.norm)
        p, _ = N.router(x, layer.gate, layer.gate_next)
        sel = Dd.topk_rows(p.astype(np.float64), K)
        srt = -np.sort(-p.astype(np.float64), axis=1)[:, : K + 1]
        gap = np.min(srt[:, :-1] - srt[:, 1:], axis=1)
        diff = np.any(sel != sel_gpu, axis=1)
        out = {"rows": int(len(diff)), "agree_frac": float(1.0 - diff.mean()),
               "near_tie_exempt": int((diff & (gap < 1e-5)).sum()),
               "mismatch_non_tie": int((diff & (gap >= 1e-5)).sum())}
        if x_gpu is not None:
            out["x_bits_equal_frac"] = float((x_gpu == x).mean())
        return out

    res = {"decode": rows(np.stack(hs), dec_sel.astype(np.int64))}
    if pf_sample is not None:
        res["prefill"] = rows(pf_sample["h"], pf_sample["sel"].astype(np.int64), pf_sample["x"])
    return res


def run_daop(args, dev, rank):
    """BASELINE configs[2]: Mixtral-8x7B-shaped 32-layer DAOP sequence at ECR
    < 1 (default 0.5): calibration sequence at ECR 1.0 -> init_from_calibration
    -> 256-token prefill (device activation counter, Alg. 1 swaps as pinned-host
    -> HBM copies on a side stream, slow experts on the host tier) -> decode
    tokens with DAOP plans, graceful degradation and the stale-input
    pre-calculation on the host tier.  Returned as the reference's run_single
    record (moesim/experiment.py:178-210), timings measured."""
    import numpy as np
    import torch

    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.daop import DaopEngine, HostExpertPool

    if rank != 0 and not args.daop_all_ranks:
        return None
    L, n_pre, n_dec = 32, 256, args.daop_tokens
    shape = P.ModelShape(L, E, K)
    t0 = time.perf_counter()
    pool = HostExpertPool(shape, D, FFN, seed=0, device=dev)
    setup_s = time.perf_counter() - t0
    cal = DaopEngine(shape, D, FFN, np.full((L, E), K / E), 1.0, P.PolicyConfig("daop"), seed=0,
                     host_pool=pool)
    crec = cal.run_sequence(cal.model.input_hidden(64, stream=300),
                            [cal.model.input_hidden(1, stream=301, step=i)[0] for i in range(16)],
                            "calib")
    calib = P.pooled_decode_probabilities([crec.trace])
    del cal, crec
    torch.cuda.empty_cache()
    runs = []
    for ecr in args.daop_ecr:
        # the calibration run above already loaded every kernel in this process
        eng_run = DaopEngine(shape, D, FFN, calib, ecr, P.PolicyConfig("daop"), seed=0,
                             host_pool=pool)
        prompt = eng_run.model.input_hidden(n_pre, stream=400)
        toks = [eng_run.model.input_hidden(1, stream=401, step=i)[0] for i in range(n_dec)]
        torch.cuda.synchronize()
        rec = eng_run.run_single(prompt, toks, f"daop_ecr{ecr}")
        n = rec["num_decode_tokens"]
        runs.append({
            "ecr": ecr, "slot_budget": eng_run.placement0.slot_budget,
            "tokens_per_second": rec["tokens_per_second"],
            "mean_token_latency_ms": rec["mean_token_latency_ms"],
            "prefill_latency_ms": rec["prefill_latency_ms"],
            "prefill_hidden_migration_ms": rec["prefill_hidden_migration_ms"],
            "swap_count": rec["swap_count"],
            "slow_executions_per_token": rec["slow_executions"] / n,
            "degradations_per_token": rec["degradations"] / n,
            "stale_inputs_per_token": rec["stale_inputs"] / n,
            "host_tier_ms_per_token": eng_run.host_ms / n,
            "set_fidelity": rec["set_fidelity"], "score_mass": rec["score_mass"],
            "similarity_prefill_decode": rec["similarity_prefill_decode"],
            "prediction_accuracy": P.mean_prediction_accuracy(rec["_trace"]),
        })
        del eng_run, rec
        torch.cuda.empty_cache()
    del pool
    return {"workload": f"32 Mixtral-8x7B MoE layers, {n_pre}-token prompt + {n_dec} decode "
                        f"tokens per ECR, DAOP (prediction from layer 4, graceful degradation), "
                        f"slow experts on the host tier (BASELINE configs[2]); the reference's "
                        f"run_single record, timings measured",
            "host_pool_gb": L * E * 3 * D * FFN * 2 / 1e9, "host_pool_setup_s": setup_s,
            "runs": runs}


DEC_CTX = 512  # context position of the decoder32 measurement


def run_decoder32(args, world, dev, eng, model, hs, hbm_peak, barrier):
    """BASELINE configs[2] with the non-MoE block executed: 32 Mixtral-8x7B
    decoder layers per token = attention with a KV cache (RMSNorm, QKV GEMV,
    RoPE, GQA flash-decoding over DEC_CTX cached positions, O-proj + residual)
    then the MoE block (DAOP plans from layer 4, all experts in HBM)."""
    import torch
    import torch.distributed as dist

    from paper_2501_10375_b200.attention import AttentionStack

    L = model.shape.num_layers
    att = AttentionStack(L, D, 32, 8, max_seq=DEC_CTX + 256, seed=0, device=dev)
    # a filled history: the cache rows before DEC_CTX are random bf16 values
    g = torch.Generator(device=dev).manual_seed(7)
    att.k_cache[:, :, :DEC_CTX].copy_(torch.randn(att.k_cache[:, :, :DEC_CTX].shape,
                                                  generator=g, device=dev))
    att.v_cache[:, :, :DEC_CTX].copy_(torch.randn(att.v_cache[:, :, :DEC_CTX].shape,
                                                  generator=g, device=dev))
    h_in = torch.empty(D, dtype=torch.float32, device=dev)
    for i in range(3):
        h_in.copy_(hs[i])
        eng.decode_token(h_in, start=4, daop=True, attn=att, pos=DEC_CTX + i)
    barrier()
    torch.cuda.synchronize()
    nt = max(10, min(100, args.steps // 20))
    stream = torch.cuda.current_stream()

    def run(prefetch):
        eng.attn_prefetch = prefetch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(nt):
            h_in.copy_(hs[i % len(hs)])
            eng.decode_token(h_in, start=4, daop=True, attn=att, pos=DEC_CTX + 3 + i % 200)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / nt

    pf_ms = run(True)      # next layer's attention weights prefetched into L2 (measured slower)
    tok_ms = run(False)    # default: the attention GEMVs stream their weights
    eng.attn_prefetch = False
    t = torch.tensor([tok_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tok_ms = float(t.item())
    ctx = DEC_CTX + 3 + nt // 2
    bytes_tok = 32 * DECODE_BYTES - 2 * E * D + L * att.bytes_per_token_layer(ctx)
    del att
    torch.cuda.empty_cache()
    return {
        "workload": f"decode b=1 through 32 full Mixtral-8x7B decoder layers (attention with a "
                    f"KV cache at context ~{DEC_CTX}, 32 q / 8 kv heads, then the MoE block; "
                    f"DAOP plans from layer 4, all experts in HBM)",
        "value": world * 1e3 / tok_ms, "unit": "tokens/s", "ms_per_token": tok_ms,
        "roofline": {"bound": "hbm", "achieved": bytes_tok / (tok_ms / 1e3) / 1e9,
                     "peak": hbm_peak, "unit": "GB/s",
                     "frac": bytes_tok / (tok_ms / 1e3) / 1e9 / hbm_peak,
                     "bytes_per_token": bytes_tok},
        "with_attn_l2_prefetch": {"tokens_per_s": 1e3 / pf_ms, "ms_per_token": pf_ms},
        "gpu_launches": nt * L * 5,
    }

EP_D, EP_FFN, EP_TOKENS = 6144, 16384, 8 * 4096


def run_ep(args, world, rank, dev, tf_sus, barrier, impl="peer", tokens=None, hbm_peak=None,
           steps=None, warmup=2, e2e=False):
    """Mixtral-8x22B-shaped MoE layer (d=6144, ffn=16384, E=8, top-2),
    prefill 8 x 4096 tokens sharded T/G per rank, experts sharded E/G per
    rank, expert-parallel over the ranks.  Total work is fixed as G grows
    (strong scaling).

    impl "peer" (the product, ep.PeerEP): router + permutation, dispatch
      kernel storing x rows straight into the owners' receive buffers over
      NVLink, tcgen05 grouped GEMMs, down-GEMM epilogue storing outputs
      straight into the sources' buffers, combine -- no host sync.
    impl "nccl" (baseline, ep.gpu_ep_layer): the same kernels around NCCL
      count all_to_all + grouped send/recv, with host syncs for the splits."""
    import torch
    import torch.distributed as dist

    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.ep import PeerEP, ep_model, gpu_ep_layer

    if world > 1 and not dist.is_initialized():
        return None
    total = tokens or EP_TOKENS
    t_local = total // world
    m = ep_model(P.ModelShape(2, E, K), EP_D, EP_FFN, rank, world, seed=0, device=dev)
    h = m.input_hidden(t_local, stream=300 + rank)
    phases = []
    if impl == "peer":
        ctx = PeerEP(m, 0, t_local, rank, world)

        def step(record=False):
            return ctx.layer(h)
    else:
        def step(record=False):
            return gpu_ep_layer(m, 0, h, timings=phases if record else None)[:3]
    if tokens is not None:
        # batched decode right after the power-capped prefill GEMMs: let the
        # clocks recover, then a longer warm-up and window (HBM-bound steps
        # of ~1 ms are sensitive to the state the previous section left)
        time.sleep(1.0)
        warmup = max(warmup, 20)
    for _ in range(warmup):
        step()
    barrier()
    torch.cuda.synchronize()
    kp = steps or (5 if tokens is None else 200)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        e0.record(stream)
        for i in range(kp):
            step(record=i == kp - 1)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    e2e_res = None
    if e2e and impl == "peer":
        # the same layer through the public call with HOST buffers: this rank's
        # tokens copied in from pinned memory and the output copied back, every step
        h_host = torch.empty(h.shape, dtype=h.dtype, pin_memory=True)
        h_host.copy_(h)
        o_host = torch.empty(h.shape, dtype=torch.float32, pin_memory=True)
        h_dev = torch.empty_like(h)
        for _ in range(warmup):
            h_dev.copy_(h_host, non_blocking=True)
            o_host.copy_(ctx.layer(h_dev)[0], non_blocking=True)
        torch.cuda.synchronize()
        barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        q0.record(stream)
        for _ in range(kp):
            h_dev.copy_(h_host, non_blocking=True)
            o_host.copy_(ctx.layer(h_dev)[0], non_blocking=True)
        q1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        te = torch.tensor([max(q0.elapsed_time(q1) / 1e3, wall)], device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_res = {"value": total * kp / float(te.item()), "unit": "tokens/s",
                   "h2d_bytes_per_step": int(h.numel() * 4), "d2h_bytes_per_step": int(h.numel() * 4),
                   "api": "PeerEP.layer with this rank's tokens from pinned host memory, output "
                          "copied back every step"}
        barrier()
    if impl == "peer":
        ctx.check()
        off = ctx._cur["offsets"].tolist()
        sent = off[-1] - sum(off[e + 1] - off[e] for e in range(E) if e * world // E == rank)
    ms = e0.elapsed_time(e1) / kp
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    split = {}
    for (_, a), (name, b) in zip(phases, phases[1:]):
        split[name] = a.elapsed_time(b)
    flops = 2.0 * K * EP_TOKENS * 3 * EP_D * EP_FFN
    if impl == "peer":
        ctx.close()
        desc = ("peer-memory kernels over NVLink (dispatch = permutation gather with remote "
                "stores; return fused into the down GEMM epilogue; epoch flags)"
                if world > 1 else "none (G=1)")
        # router, permute (count, scan, scatter), publish, dispatch, recv, up,
        # fused-return down, wait, combine
        launches = 11
    else:
        desc = ("nccl all_to_all (counts) + grouped send/recv (payload, outputs)"
                if world > 1 else "none (G=1)")
        launches = 9  # router, permute (4), up, down, combine + NCCL
    if tokens is not None:  # batched decode: HBM-bound on the active experts' weights
        wbytes = E * 3 * EP_D * EP_FFN * 2
        out = {
            "workload": f"Mixtral-8x22B-shaped layer, decode step of {total} sequences sharded "
                        f"{t_local}/rank, experts {E // world}/GPU over {world} GPU(s), skinny "
                        f"GEMMs (BASELINE configs[4], b={total})",
            "impl": impl, "value": total / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
            "scaling": "strong",
            "roofline": {"bound": "hbm", "achieved": wbytes / (ms / 1e3) / 1e9,
                         "peak": hbm_peak * world, "unit": "GB/s",
                         "frac": wbytes / (ms / 1e3) / 1e9 / (hbm_peak * world),
                         "bytes_per_step": wbytes, "note": "all 8 experts active at b=64"},
            "clocks": clk.summary(),
        }
        if impl == "peer":
            ctx.close()
        del m
        torch.cuda.empty_cache()
        return out
    out = {
        "workload": f"Mixtral-8x22B-shaped layer (d={EP_D}, ffn={EP_FFN}, E={E}, top-{K}), "
                    f"prefill {EP_TOKENS} tokens sharded {t_local}/rank, expert-parallel "
                    f"over {world} GPU(s) (BASELINE configs[4])",
        "impl": impl,
        "value": EP_TOKENS / (ms / 1e3), "unit": "tokens/s", "ms_per_layer": ms,
        "scaling": "strong", "experts_per_gpu": E // world,
        "collective": desc,
        "roofline": {"bound": "tensor", "achieved_per_gpu": flops / world / (ms / 1e3) / 1e12,
                     "peak": tf_sus, "unit": "TFLOP/s",
                     "frac": flops / world / (ms / 1e3) / 1e12 / tf_sus,
                     "flops_per_layer": flops},
    }
    out["steps"] = kp
    out["clocks"] = clk.summary()
    if e2e_res:
        out["e2e"] = e2e_res
    if split:
        out["rank0_phase_ms"] = split
    if impl == "peer":
        out["rank0_payload_bytes_sent"] = int(sent) * EP_D * 2
    out["gpu_launches_per_layer"] = launches
    del m
    torch.cuda.empty_cache()
    return out


def run_b200_ep(args, world, rank, local_rank):
    """--gpus N > 1: the headline is expert parallelism (BASELINE configs[4]):
    one Mixtral-8x22B-shaped layer, a prefill of 8 x 4096 tokens sharded
    T/N per rank, experts sharded E/N per rank, the product peer-memory path
    (ep.PeerEP: dispatch = permutation gather with NVLink stores, return fused
    into the down-GEMM epilogue).  value = whole-job tokens/s over the max
    rank time of exactly K steps; e2e = the same call with host buffers.
    The NCCL-collective path and the EP decode steps are reported beside it."""
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    hbm_peak, tf_peak, tf_sus, peak_kind = peaks()

    def barrier():
        if world > 1:
            dist.barrier()

    head = run_ep(args, world, rank, dev, tf_sus, barrier, impl="peer", steps=args.steps,
                  warmup=args.warmup, e2e=True)
    try:
        nccl = run_ep(args, world, rank, dev, tf_sus, barrier, impl="nccl")
    except Exception as exc:
        nccl = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    try:
        dec = run_ep_decode(args, world, rank, dev, hbm_peak, barrier)
    except Exception as exc:
        dec = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    try:
        b64 = run_ep(args, world, rank, dev, tf_sus, barrier, impl="peer", tokens=64,
                     hbm_peak=hbm_peak)
    except Exception as exc:
        b64 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if rank != 0:
        return None
    ms = head["ms_per_layer"]
    line = {
        "metric": METRIC, "value": head["value"], "unit": "tokens/s", "n_gpus": world,
        "steps": head["steps"], "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-RNG random-init weights and tokens)",
        "config": workload_config(world),
        "roofline": {"bound": "tensor", "achieved": head["roofline"]["achieved_per_gpu"],
                     "peak": tf_sus, "unit": "TFLOP/s", "frac": head["roofline"]["frac"],
                     "peak_kind": f"{peak_kind} sustained", "traffic": None,
                     "flops_per_launch": head["roofline"]["flops_per_layer"] / world},
        "cpu_baseline": None,
        "e2e": head.get("e2e"),
        "gpu_launches": head["gpu_launches_per_layer"] * head["steps"],
        "clocks": head.get("clocks"),
        "ep": {"peer": head, "nccl_baseline": nccl, "decode": dec, "decode_b64": b64},
    }
    line["summary"] = {"ep_prefill_tok_s": _g(head, "value"), "ep_prefill_ms": _g(head, "ms_per_layer"),
                       "ep_prefill_frac": _g(head, "roofline", "frac"),
                       "nccl_prefill_ms": _g(nccl, "ms_per_layer"),
                       "ep_decode_b1_ms": _g(dec, "ms_per_step"),
                       "ep_decode_b64_ms": _g(b64, "ms_per_step"),
                       "e2e_tok_s": _g(head, "e2e", "value")}
    return line


def run_ep_decode(args, world, rank, dev, hbm_peak, barrier):
    """Mixtral-8x22B-shaped layer, decode b=1, experts sharded E/G per rank
    (ep.PeerEPDecode): the residual is replicated, every rank runs the fused
    decode kernel on its own experts, so the token's 2 experts (2 x 604 MB)
    are streamed by up to 2 GPUs in parallel; outputs are shared through
    peer memory and combined in fixed order on every rank."""
    import torch
    import torch.distributed as dist

    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.ep import PeerEPDecode, ep_model

    if world > 1 and not dist.is_initialized():
        return None
    m = ep_model(P.ModelShape(2, E, K), EP_D, EP_FFN, rank, world, seed=0, device=dev)
    dec = PeerEPDecode(m, rank, world)
    hs = [m.input_hidden(1, stream=400, step=i)[0] for i in range(32)]
    for i in range(8):
        dec.layer(hs[i % 32])
    barrier()
    torch.cuda.synchronize()
    steps = max(50, min(args.steps, 1000))
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        dec.layer(hs[i % 32])
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    dec.check()
    ms = e0.elapsed_time(e1) / steps
    # NCCL baseline of the same step (decode kernel + all_reduce of the picks' outputs)
    from paper_2501_10375_b200 import ops as _ops
    from paper_2501_10375_b200.ep import nccl_ep_decode_layer
    nb = _ops.DecodeBuffers(EP_D, EP_FFN, E, K, dev)
    y_sum = torch.empty((K, EP_D), dtype=torch.float32, device=dev)
    o_n = torch.empty(EP_D, dtype=torch.float32, device=dev)
    for i in range(8):
        nccl_ep_decode_layer(m, 0, hs[i % 32], nb, y_sum, o_n)
    barrier()
    torch.cuda.synchronize()
    n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0.record(stream)
    for i in range(steps):
        nccl_ep_decode_layer(m, 0, hs[i % 32], nb, y_sum, o_n)
    n1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_n = n0.elapsed_time(n1) / steps
    tn = torch.tensor([ms_n], device=dev)
    if world > 1:
        dist.all_reduce(tn, op=dist.ReduceOp.MAX)
    ms_n = float(tn.item())
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    step_bytes = 2 * 3 * EP_D * EP_FFN * 2 + 2 * E * EP_D * 2  # 2 experts + 2 gates
    active = min(world, K)  # b = 1: at most k GPUs hold a pick
    dec.close()
    del dec, m
    torch.cuda.empty_cache()
    return {
        "workload": f"Mixtral-8x22B-shaped layer, decode b=1, experts sharded {E // world}/GPU "
                    f"over {world} GPU(s) (BASELINE configs[4])",
        "value": 1e3 / ms, "unit": "tokens/s", "ms_per_step": ms, "steps": steps,
        "scaling": "strong",
        "collective": ("peer-memory share of the picks' outputs (NVLink stores + epoch flags)"
                       if world > 1 else "none (G=1)"),
        "roofline": {"bound": "hbm", "achieved": step_bytes / (ms / 1e3) / 1e9,
                     "peak": hbm_peak * active if world > 1 else hbm_peak, "unit": "GB/s",
                     "frac": step_bytes / (ms / 1e3) / 1e9 / (hbm_peak * (active if world > 1 else 1)),
                     "bytes_per_step": step_bytes,
                     "note": "b=1 touches 2 experts: at most 2 GPUs stream; peak = that many x HBM"},
        "gpu_launches_per_step": 2,
        "nccl_baseline": {"value": 1e3 / ms_n, "unit": "tokens/s", "ms_per_step": ms_n,
                          "collective": "nccl all_reduce of the k x d pick outputs"
                                        if world > 1 else "none (G=1)"},
    }

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference", "ours"])
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-decode32", action="store_true")
    ap.add_argument("--no-ep", action="store_true")
    ap.add_argument("--no-server", action="store_true")
    ap.add_argument("--no-daop", action="store_true")
    ap.add_argument("--daop-ecr", type=float, nargs="+", default=[0.5])
    ap.add_argument("--daop-tokens", type=int, default=16)
    ap.add_argument("--daop-all-ranks", action="store_true")
    ap.add_argument("--ep-headline", action="store_true",
                    help="N = 1: run the N > 1 expert-parallel headline path (exercises it on one GPU)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, world, rank)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        ep_head = world > 1 or args.ep_headline
        line = (run_b200_ep if ep_head else run_b200)(args, world, rank, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
