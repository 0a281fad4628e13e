"""DAOP sequence engine: the reference's `run_single` flow, executed.

moesim/experiment.py:145-211 (`run_single`) *prices* a sequence under DAOP:

  placement0 = init_from_calibration(calib, ecr)              placement.py:128
  placement, swaps = allocate_for_sequence(placement0,
                         expert_counts(trace, "prefill"))     placement.py:188
  simulate_prefill(trace, placement0, swaps)                  simulator.py:408
  simulate_decode(trace, placement, PolicyConfig("daop"))     simulator.py:259

`DaopEngine` *executes* the same order on the B200 with real numerics:

  * init: placement0 from the calibration matrix (native, bit-exact); the HBM
    slab holds exactly `slot_budget` expert slots, every expert also lives in
    a pinned host pool (the slow tier and the migration source).
  * prefill: per layer, the fused router produces the layer's activation
    counts on device (`hist`), Alg. 1 runs for that layer right after its gate
    (swaps are issued after the gate, simulator.py:446-456), each swap is a
    pinned-host -> HBM `cudaMemcpyAsync` on a side stream, and the layer's
    experts run at the post-swap residence (resident ones on tcgen05 grouped
    GEMMs, waiting on the migration event; the rest on the host tier).
  * decode: per token and layer, one decode launch; below the prediction
    start layer the selection is the layer's own top-k (Fiddler rule), from
    it on the DAOP plan on the prediction carried by layer l-1 with graceful
    degradation -- computed on device inside the launch.  Slow picks run on
    the host tier on the current input (l < start) or the stale x_{l-1}
    (pre-calculation, l >= start), and are combined with the resident picks
    in fixed pick order.
  * everything the reference consumes is exported: the `RoutingTrace` (true
    gate of every layer + next-layer predictions, fp32 probabilities widened
    to float64), placements, `SwapEvent`s, per-token `LayerPlan`s and the
    simulator's counters (`migrations`, `slow_executions`, `degradations`,
    `stale_inputs`), so the reference's own decision functions can be run on
    the exported trace and compared with `==`.

This first version synchronises with the host once per layer (to hand the
slow tier its inputs); the decision path is fully on device.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, ops
from .errors import ConfigError, ShapeMismatchError
from .engine import SKINNY_MAX_ROWS
from .model import KIND_EXPERT, MoEModel, make_tag
from .nvtx import nvtx_pop, nvtx_push, nvtx_range
from .placement import (SWAP_IN_OUT_DEFAULT, ExpertPlacement, SwapEvent,
                        allocate_for_sequence, init_from_calibration)
from .policies import (ExecutedExpert, LayerPlan, PolicyConfig, decode_counters, make_planner,
                       plans_from_arrays)
from .trace import ModelShape, RoutingTrace


class HostExpertPool:
    """Every expert's [W1 | W3 | W2] in pinned host memory (bf16), generated
    with the same counter-based generator as the device (bit-identical)."""

    def __init__(self, shape: ModelShape, d: int, ffn: int, seed: int = 0, threads=None,
                 device=None):
        self.shape, self.d, self.ffn, self.seed = shape, d, ffn, seed
        L, E = shape.num_layers, shape.num_experts
        self.slot_elems = 3 * ffn * d
        # pinned by the library: mmap + huge pages + parallel first touch +
        # cudaHostRegister (~5x faster than cudaHostAlloc for 90 GB)
        self._nbytes = L * E * self.slot_elems * 2
        ptr, reg = ctypes.c_void_p(), ctypes.c_int32(0)
        _lib.call("daop_host_pool_alloc", self._nbytes, 0, ctypes.addressof(ptr),
                  ctypes.addressof(reg))
        self._ptr, self.pinned = ptr.value, bool(reg.value)
        arr = np.ctypeslib.as_array((ctypes.c_int16 * (self._nbytes // 2)).from_address(self._ptr))
        self.buf = torch.from_numpy(arr).view(torch.bfloat16).view(L * E, self.slot_elems)
        sc_in = float(np.float32(1.0 / np.sqrt(d)))
        sc_ff = float(np.float32(1.0 / np.sqrt(ffn)))
        mats = ((0, ffn * d, sc_in), (ffn * d, ffn * d, sc_in), (2 * ffn * d, d * ffn, sc_ff))
        if device is not None:
            # generate each slot on the GPU (the device generator is bit-identical
            # to the host one) and copy it down: ~PCIe speed instead of the
            # host generator's ~1.5 GB/s (90 GB of Mixtral-8x7B experts)
            scratch = [torch.empty(self.slot_elems, dtype=torch.bfloat16, device=device)
                       for _ in range(2)]
            for i in range(L * E):
                l, e = divmod(i, E)
                buf = scratch[i % 2]
                for mtx, (off, n, sc) in enumerate(mats):
                    ops.fill_uniform_bf16(buf[off: off + n], seed, make_tag(KIND_EXPERT, l, e, mtx),
                                          sc)
                self.buf[i].copy_(buf, non_blocking=True)
            torch.cuda.synchronize(device)
            return
        th = threads or len(os.sched_getaffinity(0))
        for l in range(L):
            for e in range(E):
                base = self.buf[l * E + e].data_ptr()
                for mtx, (off, n, sc) in enumerate(mats):
                    _lib.call("daop_fill_uniform_bf16_host", base + off * 2, n, seed,
                              make_tag(KIND_EXPERT, l, e, mtx), sc, 0, th)

    def close(self):
        if getattr(self, "_ptr", None):
            self.buf = None
            _lib.call("daop_host_pool_free", self._ptr, self._nbytes, int(self.pinned))
            self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    def slot(self, layer: int, expert: int) -> torch.Tensor:
        return self.buf[layer * self.shape.num_experts + expert]

    def ptrs(self, layer: int, expert: int):
        b = self.slot(layer, expert).data_ptr()
        fd = self.ffn * self.d
        return b, b + fd * 2, b + 2 * fd * 2


SLOW_SPLIT_FRAC = 0.28  # GPU share of a split slow expert (PCIe ~55 of ~200 GB/s host DRAM)


class SlowSplit:
    """One slow (host-tier) expert of a decode token executed by the host AND
    the GPU together: the GPU pulls rows [0, R) of W1 / W3 and columns [0, R)
    of W2 from the expert's pinned host copy over PCIe
    (daop_slow_split_pull) and runs them through the skinny tcgen05 GEMMs
    as an expert with ffn = R, while the host tier computes rows [R, ffn)
    (daop_host_expert_ffn_rows); y = y_gpu + y_host (fixed order).  Both
    halves read the host's DRAM, which serves ~200 GB/s to the two together
    against ~170 GB/s to the host alone (`scripts/host_pcie_contention.py`),
    so the slow tier -- the whole token time at ECR < 1 -- shrinks.  The
    decisions (which experts are slow, stale inputs) are the reference's;
    only the slow tier's execution changes."""

    def __init__(self, pool: HostExpertPool, rows: int, device, threads: int = 0):
        d, ffn = pool.d, pool.ffn
        if rows <= 0 or rows >= ffn or rows % 128 or d % 128:
            raise ConfigError(f"slow split: {rows} GPU rows of ffn {ffn} (multiple of 128 below ffn)")
        self.pool, self.rows, self.threads = pool, rows, threads
        self.device = torch.device(device)
        self.stream = torch.cuda.Stream(self.device)
        self.stage = torch.empty(3 * rows * d, dtype=torch.bfloat16, device=self.device)
        self.x = torch.empty((1, d), dtype=torch.bfloat16, device=self.device)
        self.x_host = torch.empty((1, d), dtype=torch.int16, pin_memory=True)
        self.off = torch.tensor([0, 1], dtype=torch.int64, device=self.device)
        self.slot = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.y_gpu = torch.empty((1, d), dtype=torch.float32, pin_memory=True)
        self.y_host = np.empty((1, d), dtype=np.float32)
        self.done = torch.cuda.Event()

    def run(self, layer: int, expert: int, x_bf16: np.ndarray) -> np.ndarray:
        """x_bf16: (1, d) bf16 bits -> y (1, d) fp32 of the whole expert."""
        pool, R, d, ffn = self.pool, self.rows, self.pool.d, self.pool.ffn
        x = np.ascontiguousarray(x_bf16, dtype=np.uint16).reshape(1, d)
        w1, w3, w2 = pool.ptrs(layer, expert)
        self.x_host.numpy()[:] = x.view(np.int16)
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self.x.view(torch.int16).copy_(self.x_host, non_blocking=True)
            _lib.call("daop_slow_split_pull", w1, w3, w2, d, ffn, R, self.stage.data_ptr(),
                      self.stream.cuda_stream)
            act = ops.expert_gemm_up_skinny(self.x, self.off, self.slot, self.stage, 1, 3 * R * d,
                                            d, R, nt=32)
            y = ops.expert_gemm_down_skinny(act, self.off, self.slot, self.stage, 1, 3 * R * d, d,
                                            R, nt=32)
            self.y_gpu.copy_(y, non_blocking=True)
            self.done.record(self.stream)
        _lib.call("daop_host_expert_ffn_rows", x.ctypes.data, 1, w1, w3, w2, d, ffn, R, ffn,
                  self.y_host.ctypes.data, self.threads)
        self.done.synchronize()
        return self.y_gpu.numpy() + self.y_host


def host_expert_ffn(pool: HostExpertPool, layer: int, expert: int, x_bf16: np.ndarray,
                    threads: int = 0, out: np.ndarray = None) -> np.ndarray:
    """Slow-tier execution of one expert on (n, d) bf16 inputs -> (n, d) fp32
    (into `out`, a C-contiguous (n, d) fp32 array, when given)."""
    x = np.ascontiguousarray(x_bf16, dtype=np.uint16)
    n = x.shape[0]
    y = np.empty((n, pool.d), dtype=np.float32) if out is None else out
    if y.shape != (n, pool.d) or y.dtype != np.float32 or not y.flags.c_contiguous:
        raise ShapeMismatchError(f"host expert output must be C-contiguous float32 {(n, pool.d)}")
    w1, w3, w2 = pool.ptrs(layer, expert)
    _lib.call("daop_host_expert_ffn", x.ctypes.data, n, w1, w3, w2, pool.d, pool.ffn,
              y.ctypes.data, 0, threads)
    return y


@dataclass
class PrefillResult:
    out: torch.Tensor
    counts: np.ndarray                # (L, E) int64, from the device activation counter
    placement_initial: ExpertPlacement
    placement: ExpertPlacement
    swaps: list
    true_scores: np.ndarray           # (T, L, E) float64 (fp32-exact)
    pred_scores: np.ndarray           # (T, L, E) float64, zero on the last layer
    slow_executions: int
    ms: float
    migration_ms: float = 0.0         # swap copies, serialised on the migration stream
    migration_hidden_ms: float = 0.0  # of which overlapped with compute (simulator.py:495-502)


@dataclass
class DecodeResult:
    out: torch.Tensor
    plans: list                       # L LayerPlans
    true_scores: np.ndarray           # (L, E)
    pred_scores: np.ndarray           # (L, E)
    ms: float


@dataclass
class SequenceRecord:
    prefill: PrefillResult
    decode: list = field(default_factory=list)
    trace: RoutingTrace | None = None
    counts: dict = field(default_factory=dict)
    tokens_per_second: float = float("nan")


class DaopEngine:
    """Executes DAOP (or the Fiddler rule) for one sequence on one B200."""

    def __init__(self, shape: ModelShape, d_model: int, d_ff: int, calib, ecr: float,
                 config: PolicyConfig | None = None, seed: int = 0, device="cuda",
                 swap_in_out: float = SWAP_IN_OUT_DEFAULT, weights_from_pred: bool = True,
                 host_pool: HostExpertPool | None = None, host_threads: int = 0,
                 attention: bool = False, max_seq: int = 1024):
        self.config = config or PolicyConfig("daop")
        self.shape = shape
        self.placement0 = init_from_calibration(calib, ecr, shape)
        self.ecr = ecr
        self.swap_in_out = swap_in_out
        self.weights_from_pred = weights_from_pred
        self.host_threads = host_threads
        # decode slow tier split with the GPU over PCIe (SlowSplit); 0 = host only
        self.slow_split_rows = 0
        self._slow_split = None
        self.host_ms = 0.0  # decode: wall time inside host-tier expert calls
        self.prefill_host_ms = 0.0  # prefill: the same for the slow experts' token batches
        self.prefill_trace = None  # a list: prefill appends each layer's wall-clock timeline
        self._ys_pin = None  # pinned staging of the slow experts' prefill outputs
        # A/B switch: wait for a layer's migrations before its host tier starts
        # (what a pageable index copy used to do implicitly); off = overlapped
        self.prefill_serial_migrations = False
        self._host_exec = None  # one thread feeding the host tier (decode pre-calculation)
        self._host_ms_lock = threading.Lock()
        self.model = MoEModel(shape, d_model, d_ff, seed=seed, device=device,
                              n_slots=self.placement0.slot_budget, resident_layers=[])
        self.pool = host_pool or HostExpertPool(shape, d_model, d_ff, seed)
        self.mig_stream = torch.cuda.Stream(device=self.model.device)
        self.h2d_stream = torch.cuda.Stream(device=self.model.device)
        self.migrations_done = 0
        for l, s in enumerate(self.placement0.on_fast):
            for e in sorted(s):
                self._migrate_in(l, e, self.model._free[0])
        torch.cuda.synchronize()
        self.placement = self.placement0
        self.migrations_done = 0
        E, k = shape.num_experts, shape.top_k
        self.bufs = [ops.DecodeBuffers(d_model, d_ff, E, k, self.model.device) for _ in range(2)]
        # the non-MoE block: attention with a KV cache or,
        # without it, the residual stream goes straight into the MoE block
        self.attn = None
        self.pos = 0
        if attention:
            from .attention import AttentionStack
            heads = d_model // 128
            self.attn = AttentionStack(shape.num_layers, d_model, heads, max(1, heads // 4),
                                       max_seq=max_seq, seed=seed, device=self.model.device)
            self._h_attn = torch.empty(d_model, dtype=torch.float32, device=self.model.device)
            # one-time cuBLAS / kernel setup of the prompt attention here, not in the
            # first timed prefill (position 0 of layer 0 is rewritten by every prefill)
            self.attn.prefill(torch.zeros((1, d_model), device=self.model.device), 0, 0)
        self._lru = None  # LRU planner of the ondemand / prefetch engines (after prefill)
        # fully resident prefill as one CUDA graph per prompt length: bit-identical,
        # but measured no faster (the 256-token layer is GPU-bound, 0.59 ms either
        # way) and the first prompt of a length pays the capture: off by default
        self.prefill_graphs = False
        self._pf_graphs = {}

    # ------------------------------------------------------------ residency
    def _migrate_in(self, layer: int, expert: int, slot: int, wait: bool = True):
        """pinned host pool -> HBM slot on the migration stream; returns its
        event.  wait=False leaves the compute stream free to run other experts
        while the copy lands (the caller orders the expert's first use after
        the event; prefill's swapped-in experts, simulator.py:457-471)."""
        m = self.model
        if slot in m._free:
            m._free.remove(slot)
        # the slot may still be read by work already queued on the compute stream
        self.mig_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.mig_stream):
            m.slab[slot].copy_(self.pool.slot(layer, expert), non_blocking=True)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(self.mig_stream)
        if wait:
            torch.cuda.current_stream().wait_event(ev)  # table update ordered after the copy
        m._bind(layer, expert, slot)
        self.migrations_done += 1
        return ev

    def _apply_swaps(self, layer: int, events):
        """Alg. 1's swaps of one layer, serialised on the migration stream
        (the reference's single interconnect lane, simulator.py:446-456).
        Returns (start event, per-swap completion events)."""
        m = self.model
        self.mig_stream.wait_stream(torch.cuda.current_stream())
        start = torch.cuda.Event(enable_timing=True)
        start.record(self.mig_stream)
        evs = []
        for ev in events:
            slot = m.evict(layer, ev.swapped_out)
            evs.append(self._migrate_in(layer, ev.swapped_in, slot, wait=False))
        return start, evs

    # ------------------------------------------------------------ non-MoE block
    def _non_moe(self, h: torch.Tensor, layer: int, pos: int) -> torch.Tensor:
        """h + Attention(RMSNorm(h)) at position pos (decode, one token)."""
        if self.attn is None:
            return h
        return self.attn.decode(h, layer, pos, out=self._h_attn)

    def _non_moe_prefill(self, h: torch.Tensor, layer: int) -> torch.Tensor:
        """Causal attention over the whole prompt at positions 0 .. T-1 (its
        keys / values land in the layer's cache for the decode tokens)."""
        if self.attn is None:
            return h
        return self.attn.prefill(h, layer, 0)

    # ------------------------------------------------------------ prefill
    def prefill(self, h: torch.Tensor) -> PrefillResult:
        m = self.model
        L, E, k = self.shape.num_layers, self.shape.num_experts, self.shape.top_k
        T, d = h.shape
        t0 = time.perf_counter()
        hist = torch.zeros((1, L, E), dtype=torch.int32, device=m.device)
        # the exported trace's scores: async D2H into one pinned buffer per
        # phase, read once after the last layer (no per-layer host sync)
        p_host = torch.zeros((2, L, T, E), dtype=torch.float32, pin_memory=True)
        swaps_all = []
        new_sets = [set(s) for s in self.placement0.on_fast]
        slow_execs = 0
        mig_timing = []  # per layer: (migration start, copies done, resident GEMMs done)
        if self.prefill_graphs and all(len(s_) == E for s_ in self.placement0.on_fast):
            # every expert in HBM: no host decision, no copy, no slow expert in the
            # whole prompt -> the 32 layers replay as ONE CUDA graph per prompt
            # length (no per-layer Python / launch gaps)
            h, hist, p_host = self._prefill_resident_graph(h)
            L = 0  # the layer loop below has nothing left to do
        tr = self.prefill_trace  # optional per-layer wall-clock timeline (list)
        for l in range(L):
            nvtx_push(f"prefill/L{l}")
            tl = {"layer": l, "t0": time.perf_counter()} if tr is not None else None
            with nvtx_range("attention"):
                h = self._non_moe_prefill(h, l)
            nxt = m.gate[l + 1] if l + 1 < L else None
            with nvtx_range("router"):
                r = ops.router(h, m.norm[l], m.gate[l], nxt, k, hist=hist[:, l],
                               tokens_per_seq=T, hist_seq_stride=L * E)
            swapped_in, mig_evs = [], []
            # a layer whose every expert is cached has no uncached (hot)
            # candidate, so Alg. 1 cannot swap there: no host round trip
            if self.config.engine == "daop" and len(self.placement0.on_fast[l]) < E:
                # only DAOP reallocates (experiment.py:158-163): Alg. 1 for this
                # layer right after its gate (placement.py:188-237)
                counts_l = hist[0, l].to(torch.int64).cpu().numpy()
                if tl is not None:
                    tl["hist_synced"] = time.perf_counter()
                one = ExpertPlacement(ModelShape(1, E, k), [self.placement0.on_fast[l]],
                                      self.placement0.slot_budget)
                after, ev1 = allocate_for_sequence(one, counts_l[None, :], self.swap_in_out)
                evs = [SwapEvent(l, e.swapped_in, e.swapped_out, e.hot_tokens, e.cold_tokens)
                       for e in ev1]
                swaps_all.extend(evs)
                new_sets[l] = set(after.on_fast[0])
                if tl is not None:
                    tl["alg1_done"] = time.perf_counter()
                if evs:
                    mig_start, mig_evs = self._apply_swaps(l, evs)
                    swapped_in = [e.swapped_in for e in evs]
                if tl is not None:
                    tl["swaps_queued"] = time.perf_counter()
            pr = ops.permute(r["topk_idx"], E, r["x"])
            resident = m.resident_mask()[l]  # post-swap residence
            slow = []
            if not resident.all():  # only then does the host need the expert offsets
                off = pr["offsets"].cpu().numpy()
                slow = [e for e in range(E) if off[e + 1] > off[e] and not resident[e]]
                if tl is not None:
                    tl["offsets_synced"] = time.perf_counter()
            # slow experts' rows -> pinned host memory BEFORE the GEMMs are queued,
            # so the host tier runs while the GPU computes
            xs_host = {}
            for e in slow:
                a_, b_ = int(off[e]), int(off[e + 1])
                xs_host[e] = torch.empty((b_ - a_, d), dtype=torch.bfloat16, pin_memory=True)
                xs_host[e].copy_(pr["x_perm"][a_:b_], non_blocking=True)
            x_ready = torch.cuda.Event()
            x_ready.record()
            if tl is not None:
                tl["xs_queued"] = time.perf_counter()
            # experts at the post-swap residence: first every expert whose weights
            # are already in HBM, then the swapped-in ones, each after its copy
            # lands (simulator.py:457-471)
            slot_now = m.slot_of[l]
            if swapped_in:
                # slot tables of the resident and the swapped-in experts, built on
                # the device from a pinned mask (async): indexing a CUDA tensor with
                # a Python list would copy the index from pageable memory, which
                # blocks the host until the stream drains -- i.e. until this
                # layer's migrations landed, serialising them with the host tier
                mask = torch.zeros(E, dtype=torch.bool, pin_memory=True)
                mask[swapped_in] = True
                mask = mask.to(m.device, non_blocking=True)
                slot_now = torch.where(mask, -1, m.slot_of[l])
                slot_mig = torch.where(mask, m.slot_of[l], -1)
            rows = pr["x_perm"].shape[0]
            act = torch.empty((rows, m.ffn), dtype=torch.bfloat16, device=m.device)
            y = torch.empty((rows, d), dtype=torch.float32, device=m.device)
            skinny = rows <= SKINNY_MAX_ROWS  # weights as the M side (engine.py)
            up = ops.expert_gemm_up_skinny if skinny else ops.expert_gemm_up
            down = ops.expert_gemm_down_skinny if skinny else ops.expert_gemm_down
            with nvtx_range("experts/resident"):
                up(pr["x_perm"], pr["offsets"], slot_now, m.slab, m.n_slots, m.slot_elems, d,
                   m.ffn, out=act)
                down(act, pr["offsets"], slot_now, m.slab, m.n_slots, m.slot_elems, d, m.ffn,
                     out=y)
            if swapped_in:
                g1 = torch.cuda.Event(enable_timing=True)
                g1.record()
                mig_timing.append([mig_start, mig_evs[-1], g1, None])
                for ev in mig_evs:
                    torch.cuda.current_stream().wait_event(ev)
                up(pr["x_perm"], pr["offsets"], slot_mig, m.slab, m.n_slots, m.slot_elems, d,
                   m.ffn, out=act)
                down(act, pr["offsets"], slot_mig, m.slab, m.n_slots, m.slot_elems, d, m.ffn,
                     out=y)
            if swapped_in and self.prefill_serial_migrations:  # A/B switch: the r02 behaviour
                for ev in mig_evs:
                    ev.synchronize()
            if tl is not None:
                tl["gemms_queued"] = time.perf_counter()
            if slow:
                nvtx_push("experts/host_tier")
                x_ready.synchronize()
                if tl is not None:
                    tl["host_start"] = time.perf_counter()
                # the host tier's results go up on their own stream, so the GPU
                # clock records when the slow experts finished (for the hidden-
                # migration measurement) independently of the GEMM queue
                # results land in pinned memory and go up asynchronously: a
                # pageable copy would block the host tier behind the H2D copy
                # engine's queue (this layer's migrations).  The staging rows are
                # reused by the next layer only after this layer's combine
                # waited for them (the next x_ready is recorded behind it).
                if self._ys_pin is None or self._ys_pin.shape[0] < rows:
                    self._ys_pin = torch.empty((rows, d), dtype=torch.float32, pin_memory=True)
                ys_np = self._ys_pin.numpy()
                with torch.cuda.stream(self.h2d_stream):
                    for e in slow:
                        a_, b_ = int(off[e]), int(off[e + 1])
                        xs = xs_host[e].view(torch.int16).numpy().view(np.uint16)
                        th0 = time.perf_counter()
                        host_expert_ffn(self.pool, l, e, xs, self.host_threads, out=ys_np[a_:b_])
                        self.prefill_host_ms += 1e3 * (time.perf_counter() - th0)
                        y[a_:b_].copy_(self._ys_pin[a_:b_], non_blocking=True)
                        slow_execs += 1
                    hev = torch.cuda.Event(enable_timing=True)
                    hev.record(self.h2d_stream)
                torch.cuda.current_stream().wait_event(hev)
                if swapped_in:
                    mig_timing[-1][3] = hev
                if tl is not None:
                    tl["host_end"] = time.perf_counter()
                nvtx_pop()
            out = ops.combine(h, y, pr["inv"], r["topk_w"])
            p_host[0, l].copy_(r["p"], non_blocking=True)
            if nxt is not None:
                p_host[1, l].copy_(r["p_pred"], non_blocking=True)
            h = out
            if tl is not None:
                tl.update(t1=time.perf_counter(), swaps=len(swapped_in), slow=len(slow),
                          slow_rows=[int(off[e + 1] - off[e]) for e in slow])
                tr.append(tl)
            nvtx_pop()
        torch.cuda.synchronize()
        true_sc = np.ascontiguousarray(p_host[0].numpy().transpose(1, 0, 2), dtype=np.float64)
        pred_sc = np.ascontiguousarray(p_host[1].numpy().transpose(1, 0, 2), dtype=np.float64)
        self.placement = ExpertPlacement(self.shape, new_sets, self.placement0.slot_budget)
        self.pos = T  # the first decode token's position
        if self.config.engine in ("ondemand", "prefetch"):
            self._lru = make_planner(self.placement, self.config)
        counts = hist[0].to(torch.int64).cpu().numpy()
        # migration time hidden under compute, measured the way the reference
        # prices it (simulator.py:495-502): total copy time minus the time the
        # compute stream actually waited for the copies once its resident
        # experts and the layer's slow (host-tier) experts were done
        mig_total = mig_hidden = 0.0
        for st, done, g1, hev in mig_timing:
            tot = st.elapsed_time(done)
            other = st.elapsed_time(g1)  # resident experts' GEMMs done
            if hev is not None:          # the layer also waits for its slow experts
                other = max(other, st.elapsed_time(hev))
            stall = max(0.0, tot - other)
            mig_total += tot
            mig_hidden += min(max(tot - stall, 0.0), tot)
        return PrefillResult(h, counts, self.placement0, self.placement, swaps_all, true_sc,
                             pred_sc, slow_execs, 1e3 * (time.perf_counter() - t0),
                             mig_total, mig_hidden)

    def _prefill_layers_resident(self, h, hist, p_host):
        """The prefill layer loop for a fully resident model (device work only:
        attention, router + counter, permutation, expert GEMMs, combine, the
        scores' D2H copies) -- the body captured by _prefill_resident_graph."""
        m = self.model
        L, E, k = self.shape.num_layers, self.shape.num_experts, self.shape.top_k
        T, d = h.shape
        for l in range(L):
            h = self._non_moe_prefill(h, l)
            nxt = m.gate[l + 1] if l + 1 < L else None
            r = ops.router(h, m.norm[l], m.gate[l], nxt, k, hist=hist[:, l], tokens_per_seq=T,
                           hist_seq_stride=L * E)
            pr = ops.permute(r["topk_idx"], E, r["x"])
            rows = pr["x_perm"].shape[0]
            skinny = rows <= SKINNY_MAX_ROWS
            up = ops.expert_gemm_up_skinny if skinny else ops.expert_gemm_up
            down = ops.expert_gemm_down_skinny if skinny else ops.expert_gemm_down
            act = up(pr["x_perm"], pr["offsets"], m.slot_of[l], m.slab, m.n_slots, m.slot_elems,
                     d, m.ffn)
            y = down(act, pr["offsets"], m.slot_of[l], m.slab, m.n_slots, m.slot_elems, d, m.ffn)
            h = ops.combine(h, y, pr["inv"], r["topk_w"])
            p_host[0, l].copy_(r["p"], non_blocking=True)
            if nxt is not None:
                p_host[1, l].copy_(r["p_pred"], non_blocking=True)
        return h

    def _prefill_resident_graph(self, h):
        """Capture (first prompt of this length) and replay the resident
        prefill as one CUDA graph.  Returns (h_out, hist, p_host); the
        graph's static buffers are reused by the next prompt of this length,
        so h_out is cloned."""
        m = self.model
        L, E = self.shape.num_layers, self.shape.num_experts
        T, d = h.shape
        ent = self._pf_graphs.get(T)
        if ent is None:
            h_in = torch.empty_like(h)
            hist = torch.zeros((1, L, E), dtype=torch.int32, device=m.device)
            p_host = torch.zeros((2, L, T, E), dtype=torch.float32, pin_memory=True)
            _lib.call("daop_gemm_prepare")  # device-wide setup outside the capture
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=m.device)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                with torch.cuda.graph(g):
                    hist.zero_()
                    out = self._prefill_layers_resident(h_in, hist, p_host)
            torch.cuda.current_stream().wait_stream(side)
            ent = self._pf_graphs[T] = (g, h_in, hist, p_host, out)
        g, h_in, hist, p_host, out = ent
        h_in.copy_(h)
        g.replay()
        return out.clone(), hist, p_host

    # ------------------------------------------------------------ decode
    def _host_views(self):
        """Pinned mirrors of the decode buffers' decision prefix: one row per
        layer of one pinned buffer (one D2H copy per layer), with per-layer
        numpy views and whole-buffer (L, ...) views for reading every deferred
        layer at once at the end of a token."""
        if getattr(self, "_mh", None) is None:
            L, E, k, d = (self.shape.num_layers, self.shape.num_experts, self.shape.top_k,
                          self.model.d)
            b0 = self.bufs[0]
            o = b0.offsets
            self._mh_buf = torch.empty((L, b0.decisions_bytes), dtype=torch.uint8,
                                       pin_memory=True)
            big = self._mh_buf.numpy()

            def fields(a):  # a: (..., decisions_bytes) uint8
                return {"x": a[..., o["x"]: o["x"] + 2 * d].view(np.uint16),
                        "p": a[..., o["p"]: o["p"] + 4 * E].view(np.float32),
                        "p_pred": a[..., o["p_pred"]: o["p_pred"] + 4 * E].view(np.float32),
                        "deg": a[..., o["deg"]: o["deg"] + 4 * (2 * k + 1)].view(np.int32),
                        "is_fast": a[..., o["is_fast"]: o["is_fast"] + k],
                        "sel": a[..., o["sel"]: o["sel"] + 4 * k].view(np.int32)}
            self._mh = [(self._mh_buf[l], fields(big[l])) for l in range(L)]
            self._mh_all = fields(big)
            self._y_host = torch.empty((k, d), dtype=torch.float32, pin_memory=True)
            self._h_pp = [torch.empty(d, dtype=torch.float32, device=self.model.device)
                          for _ in range(2)]
        return self._mh

    def _host_plan(self, layer: int, pred_prev: np.ndarray):
        """The DAOP plan of `layer` from the prediction carried on layer-1
        (policies.py:299-336), computed on the host from the same float32
        values the device planner uses -> identical selection; lets the host
        tier start the pre-calculation before the layer's launch."""
        E, k = self.shape.num_experts, self.shape.top_k
        tr = np.zeros((2, E))
        pr = np.zeros((2, E))
        pr[0] = pred_prev
        pm = np.array([1, 0], dtype=np.uint8)
        fast = np.zeros((2, E), dtype=np.uint8)
        fast[1] = self.model.resident_mask()[layer]
        sel = np.zeros((2, k), dtype=np.int32)
        isf = np.zeros((2, k), dtype=np.uint8)
        drop = np.zeros((2, k), dtype=np.int32)
        sub = np.zeros((2, k), dtype=np.int32)
        nd = np.zeros(2, dtype=np.int32)
        _lib.call("daop_plan_token_f64", tr.ctypes.data, pr.ctypes.data, pm.ctypes.data,
                  fast.ctypes.data, 2, E, k, 1, 3, int(self.config.graceful_degradation),
                  sel.ctypes.data, isf.ctypes.data, drop.ctypes.data, sub.ctypes.data,
                  nd.ctypes.data)
        return sel[1], isf[1]

    def _slow_splitter(self):
        """The SlowSplit for slow_split_rows (None = the host tier alone)."""
        r = int(self.slow_split_rows)
        if r <= 0:
            return None
        sp = self._slow_split
        if sp is None or sp.rows != r or sp.threads != self.host_threads:
            sp = self._slow_split = SlowSplit(self.pool, r, self.model.slab.device,
                                              self.host_threads)
        return sp

    def decode(self, h: torch.Tensor) -> DecodeResult:
        """One decode token (h: (d,) fp32 on device) through every layer.

        Per layer: one decode launch, one D2H of the decisions (+ the layer's
        x for the host tier), one host synchronisation.  From the prediction
        start layer on (DAOP), the plan is known before the launch (it only
        depends on layer l-1's prediction), so the host tier computes the
        slow picks on the stale x_{l-1} while the GPU streams the resident
        picks -- the pre-calculation overlap of PAPER.md:317-339.

        A layer with every expert in HBM needs nothing from the host: when
        the next layer does not need its prediction on the host either, its
        synchronisation is skipped and its decisions are read after the
        token (at ECR 1.0 the whole token runs without a host round trip)."""
        if self.config.engine in ("ondemand", "prefetch"):
            return self._decode_lru(h)
        m = self.model
        cfg = self.config
        L, E, k = self.shape.num_layers, self.shape.num_experts, self.shape.top_k
        start = cfg.prediction_start_layer
        daop = cfg.engine == "daop"
        mh = self._host_views()
        stream = torch.cuda.current_stream()
        t0 = time.perf_counter()
        sel = np.zeros((L, k), dtype=np.int32)
        fast = np.zeros((L, k), dtype=np.uint8)
        drop = np.full((L, k), -1, dtype=np.int32)
        sub = np.full((L, k), -1, dtype=np.int32)
        nd = np.zeros(L, dtype=np.int32)
        true_sc = np.zeros((L, E))
        pred_sc = np.zeros((L, E))

        def read(l, v):  # one layer's decisions out of its pinned mirror
            dg = v["deg"]
            sel[l], fast[l] = v["sel"], v["is_fast"]
            nd[l] = dg[2 * k]
            drop[l, : nd[l]] = dg[: nd[l]]
            sub[l, : nd[l]] = dg[k: k + nd[l]]
            true_sc[l] = v["p"]
            if l + 1 < L:
                pred_sc[l] = v["p_pred"]

        prev_b, prev_v = None, None
        pos = self.pos
        full = m.resident_mask().all(axis=1)
        deferred = []
        queued = {}  # layer -> (sel, is_fast, {pick: Future}) of its host pre-calculation
        if self._host_exec is None:
            self._host_exec = ThreadPoolExecutor(max_workers=1, thread_name_prefix="daop-host")

        split = self._slow_splitter()

        def host_job(l, e, xs):  # one slow expert on the host tier (GIL released)
            th0 = time.perf_counter()
            y = split.run(l, e, xs) if split is not None else \
                host_expert_ffn(self.pool, l, e, xs, self.host_threads)
            with self._host_ms_lock:
                self.host_ms += 1e3 * (time.perf_counter() - th0)
            return y

        def queue_precalc(l, pv):  # DAOP plan of l from layer l-1's mirror pv
            hs, hf = self._host_plan(l, pv["p_pred"].astype(np.float64))
            xs = pv["x"][None, :]
            futs = {q: self._host_exec.submit(host_job, l, int(hs[q]), xs)
                    for q in range(k) if not hf[q]}
            queued[l] = (hs, hf, futs)

        for l in range(L):
            nvtx_push(f"decode/L{l}")
            h = self._non_moe(h, l, pos)
            b = self.bufs[l % 2]
            ht, v = mh[l]
            mode = 1 if (daop and l >= start) else 0
            nxt = m.gate[l + 1] if l + 1 < L else None
            ops.decode_layer(h, m.norm[l], m.gate[l], nxt, m.fast[l], m.slot_of[l], m.slab,
                             m.slot_elems, m.d, m.ffn, k, b,
                             pred_prev=prev_b.p_pred if mode == 1 else None, mode=mode,
                             graceful=cfg.graceful_degradation,
                             weights_from_pred=self.weights_from_pred and mode == 1)
            ht.copy_(b.meta[: b.decisions_bytes], non_blocking=True)
            if full[l] and (l + 1 == L or full[l + 1]):
                deferred.append(l)  # all picks resident: no host work, read later
                h = b.h_out
                prev_b, prev_v = b, v
                nvtx_pop()
                continue
            plan_on_host = mode == 1 and not full[l]
            if plan_on_host and l not in queued:
                # pre-calculation on the host while the GPU streams the layer
                queue_precalc(l, prev_v)
            stream.synchronize()
            s_l, f_l = v["sel"].copy(), v["is_fast"].copy()
            if plan_on_host:
                hs, hf, _ = queued[l]
                if s_l.tolist() != hs.tolist() or f_l.tolist() != hf.tolist():
                    raise ShapeMismatchError(f"layer {l}: host plan differs from the device plan")
            read(l, v)
            futs = dict(queued[l][2]) if plan_on_host else {}
            if mode == 0 and not f_l.all():
                # Fiddler rule: current x_l, after the router -- on the host
                # tier's queue AHEAD of layer l+1's pre-calculation
                xs = v["x"][None, :].copy()
                for q in range(k):
                    if not f_l[q]:
                        futs[q] = self._host_exec.submit(host_job, l, int(s_l[q]), xs)
            # layer l+1's plan and stale input are known now: queue its
            # pre-calculation behind this layer's, so the host tier runs back to
            # back while this thread combines and launches
            if daop and start <= l + 1 < L and not full[l + 1]:
                queue_precalc(l + 1, v)
            ys = {q: f.result() for q, f in futs.items()}
            if not f_l.all():
                for q, yq in ys.items():
                    self._y_host[q].copy_(torch.from_numpy(yq[0]))
                    b.y[q].copy_(self._y_host[q], non_blocking=True)
                out = self._h_pp[l % 2]
                _lib.call("daop_combine_dense", h.data_ptr(), b.y.data_ptr(), b.w.data_ptr(), k,
                          m.d, out.data_ptr(), stream.cuda_stream)
                h = out
            else:
                h = b.h_out
            prev_b, prev_v = b, v
            nvtx_pop()
        torch.cuda.synchronize()
        if deferred:  # every picked expert resident: no degradations to read
            dl = np.asarray(deferred)
            va = self._mh_all
            sel[dl], fast[dl] = va["sel"][dl], va["is_fast"][dl]
            nd[dl] = va["deg"][dl, 2 * k]
            true_sc[dl] = va["p"][dl]
            dp = dl[dl + 1 < L]
            pred_sc[dp] = va["p_pred"][dp]
        h = h.clone()
        self.pos += 1
        plans = plans_from_arrays(sel, fast, drop, sub, nd, pred_sc, cfg)
        return DecodeResult(h, plans, true_sc, pred_sc, 1e3 * (time.perf_counter() - t0))

    def _rebind(self, layer: int, expert: int, evicted: int):
        """Move `expert` of `layer` into the HBM slot of the expert the LRU
        cache evicted (pinned host -> HBM on the migration stream)."""
        m = self.model
        slot = m.evict(layer, evicted) if evicted >= 0 else m._free[0]
        return self._migrate_in(layer, expert, slot)

    def _decode_lru(self, h: torch.Tensor) -> DecodeResult:
        """The ondemand / prefetch baselines on the GPU (policies.py:173-245,
        simulator.py:297-335): every pick runs on the GPU on the current input.
        A pick absent from HBM is a demand migration into the slot of the
        layer's least recently used expert, after which the layer is
        re-launched; the prefetch engine also moves the next layer's predicted
        experts in as soon as layer l's prediction gate ran."""
        m = self.model
        L, E, k = self.shape.num_layers, self.shape.num_experts, self.shape.top_k
        prefetch = self.config.engine == "prefetch"
        t0 = time.perf_counter()
        true_sc = np.zeros((L, E))
        pred_sc = np.zeros((L, E))
        plans = []
        pos = self.pos
        for l in range(L):
            h = self._non_moe(h, l, pos)
            b = self.bufs[l % 2]
            nxt = m.gate[l + 1] if l + 1 < L else None

            def launch():
                ops.decode_layer(h, m.norm[l], m.gate[l], nxt, m.fast[l], m.slot_of[l], m.slab,
                                 m.slot_elems, m.d, m.ffn, k, b, mode=0)

            launch()
            true_sc[l] = b.p.cpu().numpy()
            if nxt is not None:
                pred_sc[l] = b.p_pred.cpu().numpy()
            dec = self._lru.plan_layer(l, true_sc[l],
                                       pred_sc[l] if (prefetch and nxt is not None) else None)
            if tuple(int(x) for x in b.sel.cpu().tolist()) != dec.selection:
                raise ShapeMismatchError(f"layer {l}: device top-k differs from the planner's")
            for e, ev in zip(dec.migrations, dec.migration_evictions):
                self._rebind(l, e, ev)
            if dec.migrations:  # demand migrations block this layer
                launch()
            for e, ev in zip(dec.prefetch_issues, dec.prefetch_evictions):
                self._rebind(l + 1, e, ev)
            h = b.h_out.clone()
            plans.append(LayerPlan(layer=l, executed=tuple(ExecutedExpert(e, "fast", "current")
                                                           for e in dec.selection),
                                   migrations=dec.migrations,
                                   prefetch_issues=dec.prefetch_issues))
        torch.cuda.synchronize()
        self.pos += 1
        return DecodeResult(h, plans, true_sc, pred_sc, 1e3 * (time.perf_counter() - t0))

    # ------------------------------------------------------------ sequence
    def run_sequence(self, h_prompt: torch.Tensor, decode_inputs, sequence_id: str = "seq"):
        """prefill + decode of one sequence; returns a SequenceRecord whose
        trace / placements / swaps / plans / counters mirror run_single."""
        pre = self.prefill(h_prompt)
        rec = SequenceRecord(prefill=pre)
        lat = 0.0
        for h in decode_inputs:
            dr = self.decode(h)
            rec.decode.append(dr)
            lat += dr.ms
        L = self.shape.num_layers
        pm = np.zeros(pre.true_scores.shape[:2], dtype=bool)
        pm[:, : L - 1] = True
        n = len(rec.decode)
        dt = np.stack([r.true_scores for r in rec.decode]) if n else np.zeros((0, L, self.shape.num_experts))
        dp = np.stack([r.pred_scores for r in rec.decode]) if n else np.zeros_like(dt)
        dm = np.zeros(dt.shape[:2], dtype=bool)
        dm[:, : L - 1] = True
        rec.trace = RoutingTrace(self.shape, sequence_id, pre.true_scores, dt, pre.pred_scores,
                                 pm, dp, dm)
        rec.counts = decode_counters([r.plans for r in rec.decode], self.config)
        rec.tokens_per_second = 1e3 * n / lat if lat > 0 else float("nan")
        return rec

    def run_single(self, h_prompt: torch.Tensor, decode_inputs, sequence_id: str = "seq",
                   seed: int = 0) -> dict:
        """experiment.run_single (moesim/experiment.py:145-211) EXECUTED:
        prefill + decode of one sequence on the B200, returned as the
        reference's flat run record.  Decision fields (placements, swaps,
        counters, set_fidelity, score_mass, similarity_prefill_decode,
        swap_count) come from the kernels' own decisions; the timing fields
        are measured (per-token wall latency, tokens/s, prefill latency,
        hidden migration time).  Extra keys: ``_trace`` (the exported
        RoutingTrace: re-running the reference's run_single on it with the
        same calibration reproduces every decision field), ``_sequence``."""
        from .experiment import make_record
        rec = self.run_sequence(h_prompt, decode_inputs, sequence_id)
        pre = rec.prefill
        lat = [d.ms for d in rec.decode]
        total = pre.ms + sum(lat)
        out = make_record(rec.trace, self.ecr, self.config.engine, seed, pre.placement_initial,
                          pre.placement, pre.swaps, [d.plans for d in rec.decode], self.config,
                          per_token_latency_ms=lat, prefill_latency_ms=pre.ms,
                          prefill_hidden_migration_ms=pre.migration_hidden_ms,
                          busy_fraction={"host_tier": (self.host_ms / sum(lat)) if lat else 0.0,
                                         "host_tier_prefill": (self.prefill_host_ms / total)
                                         if total else 0.0})
        out["_prefill_result"] = pre
        out["_trace"] = rec.trace
        out["_sequence"] = rec
        return out

