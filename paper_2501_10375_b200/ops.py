"""Device operations of the MoE-block hot path (torch CUDA tensors in/out).

Each function is a thin marshalling layer over one C-ABI entry point of
libdaop_b200.so -- torch owns device memory and streams, the kernels do the
work.  No function here has a CPU path: inputs must already be on the
device, and a missing device raises DeviceError.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import DeviceError, ShapeMismatchError

RMS_EPS = 1e-5


def _dev(*ts):
    for t in ts:
        if t is not None and (not isinstance(t, torch.Tensor) or not t.is_cuda):
            raise DeviceError("hot-path ops take CUDA tensors (there is no CPU fallback)")
        if t is not None and not t.is_contiguous():
            raise ShapeMismatchError("hot-path ops take contiguous tensors")


def _p(t):
    return 0 if t is None else t.data_ptr()


def _s():
    return torch.cuda.current_stream().cuda_stream


def fill_uniform_bf16(out: torch.Tensor, seed: int, tag: int, scale: float, offset: int = 0):
    _dev(out)
    _lib.call("daop_fill_uniform_bf16", out.data_ptr(), out.numel(), seed, tag, float(scale),
              offset, _s())
    return out


def fill_uniform_f32(out: torch.Tensor, seed: int, tag: int, scale: float, offset: int = 0):
    _dev(out)
    _lib.call("daop_fill_uniform_f32", out.data_ptr(), out.numel(), seed, tag, float(scale),
              offset, _s())
    return out


def fill_norm_bf16(out: torch.Tensor, seed: int, layer: int):
    _dev(out)
    _lib.call("daop_fill_norm_bf16", out.data_ptr(), out.numel(), seed, layer, _s())
    return out


def router(h, gamma, wg, wg_next, k, *, hist=None, tokens_per_seq=0, hist_seq_stride=0,
           write_x=True, eps=RMS_EPS):
    """Fused router over T tokens (see daop_router)."""
    _dev(h, gamma, wg, wg_next)
    if hist is not None and not hist.is_cuda:  # hist may be a strided (seq, E) view
        raise DeviceError("hist must live on the device")
    t, d = h.shape
    e = wg.shape[0]
    dev = h.device
    x = torch.empty((t, d), dtype=torch.bfloat16, device=dev) if write_x else None
    p = torch.empty((t, e), dtype=torch.float32, device=dev)
    pp = torch.empty((t, e), dtype=torch.float32, device=dev) if wg_next is not None else None
    idx = torch.empty((t, k), dtype=torch.int32, device=dev)
    w = torch.empty((t, k), dtype=torch.float32, device=dev)
    _lib.call("daop_router", h.data_ptr(), gamma.data_ptr(), wg.data_ptr(), _p(wg_next), t, d,
              e, k, float(eps), _p(x), p.data_ptr(), _p(pp), idx.data_ptr(), w.data_ptr(),
              _p(hist), int(tokens_per_seq), int(hist_seq_stride), _s())
    return {"x": x, "p": p, "p_pred": pp, "topk_idx": idx, "topk_w": w}


def set_router_mode(single_pass: bool, prefetch: int = -1, bulk: bool = True) -> None:
    """Tuning switch: single-pass tensor-core router (default) or two-pass;
    prefetch >= 0 sets the register-resident single-pass kernel's L2 prefetch
    distance; bulk=False turns the bulk-copy (shared-memory ring) router off,
    leaving the register-resident single-pass kernel."""
    mode = (int(bool(single_pass)) | (0 if bulk else 4)
            | ((prefetch + 1) << 4 if prefetch >= 0 else 0))
    _lib.call("daop_set_router_mode", mode)


def set_stream_mode(gather: int = 0, combine: int = 0, gather_ctas_per_sm: int = 0,
                    combine_stages: int = 0) -> None:
    """Tuning switch for the gather / combine kernels (daop_set_stream_mode)."""
    _lib.call("daop_set_stream_mode", gather, combine, gather_ctas_per_sm, combine_stages)


def permute(topk_idx, num_experts, x=None):
    """Stable (expert, token, j) permutation; gathers x rows when given."""
    _dev(topk_idx, x)
    t, k = topk_idx.shape
    dev = topk_idx.device
    ws_bytes = torch.zeros(1, dtype=torch.int64)
    _lib.call("daop_permute_workspace", t, k, num_experts, ws_bytes.data_ptr())
    ws = torch.empty(int(ws_bytes[0]), dtype=torch.uint8, device=dev)
    offsets = torch.empty(num_experts + 1, dtype=torch.int64, device=dev)
    perm = torch.empty(t * k, dtype=torch.int32, device=dev)
    inv = torch.empty(t * k, dtype=torch.int32, device=dev)
    x_perm = None
    d = 0
    if x is not None:
        d = x.shape[1]
        x_perm = torch.empty((t * k, d), dtype=x.dtype, device=dev)
    _lib.call("daop_permute", topk_idx.data_ptr(), t, k, num_experts, _p(x), d,
              offsets.data_ptr(), perm.data_ptr(), inv.data_ptr(), _p(x_perm), ws.data_ptr(),
              ws.numel(), _s())
    return {"offsets": offsets, "perm": perm, "inv": inv.view(t, k), "x_perm": x_perm}


SPLITK_MAX = 8


def splitk_parts(m: int, k: int, n: int) -> int:
    """The K split daop_gemm_bf16_f32_ws uses for an (m, k) x (n, k)^T product
    (1 = none): the idle SM pairs over the n / 256 tiles of a <= 256-row M."""
    if m > 256:
        return 1
    pairs = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count // 2
    return max(1, min(SPLITK_MAX, pairs // (n // 256), (k // 64) // 4))


def gemm_bf16_f32(a, w, resid=None, out=None, ws=None):
    """out (M, N) fp32 = a (M, K) bf16 . w (N, K)^T [+ resid (M, N) fp32] on the
    tcgen05 GEMM pipeline (daop_gemm_bf16_f32); N % 256 == 0, K % 64 == 0.
    ws: fp32 workspace for the split-K path of prompt-sized M
    (daop_gemm_bf16_f32_ws; True = allocate splitk_parts x M x N)."""
    _dev(a, w, resid, out)
    m, k = a.shape
    n = w.shape[0]
    if w.shape[1] != k or (resid is not None and tuple(resid.shape) != (m, n)):
        raise ShapeMismatchError(f"gemm: a {tuple(a.shape)}, w {tuple(w.shape)}")
    out = torch.empty((m, n), dtype=torch.float32, device=a.device) if out is None else out
    if ws is None:
        _lib.call("daop_gemm_bf16_f32", a.data_ptr(), m, k, w.data_ptr(), n, _p(resid),
                  out.data_ptr(), _s())
        return out
    if ws is True:
        ws = torch.empty(max(1, splitk_parts(m, k, n)) * m * n, dtype=torch.float32,
                         device=a.device)
    _dev(ws)
    _lib.call("daop_gemm_bf16_f32_ws", a.data_ptr(), m, k, w.data_ptr(), n, _p(resid),
              out.data_ptr(), ws.data_ptr(), ws.numel() * 4, _s())
    return out


def set_gemm_mode(mode: int) -> None:
    """0: tcgen05 CTA-pair grouped GEMM (default), 1: single-CTA kernel."""
    _lib.call("daop_set_gemm_mode", int(mode))


def expert_gemm_up(x_perm, offsets, slot_of, slab, n_slots, slot_elems, d, ffn, group_m=0,
                   out=None):
    """act rows of every expert with an HBM slot in `slot_of` (experts with
    slot -1 get no tiles: their rows of `out` are left untouched)."""
    _dev(x_perm, offsets, slot_of, slab, out)
    rows = x_perm.shape[0]
    act = torch.empty((rows, ffn), dtype=torch.bfloat16, device=x_perm.device) if out is None \
        else out
    _lib.call("daop_expert_gemm_up", x_perm.data_ptr(), rows, d, ffn, slab.data_ptr(), n_slots,
              slot_elems, offsets.data_ptr(), slot_of.data_ptr(), offsets.numel() - 1,
              act.data_ptr(), group_m, _s())
    return act


def expert_gemm_up_gather(x, perm, k, offsets, slot_of, slab, n_slots, slot_elems, d, ffn,
                          group_m=0):
    """Up GEMM whose A rows are TMA-gathered from x (T, d) by the permutation
    (sorted row r = token perm[r] // k): no x_perm.  Raises DeviceError in the
    single-CTA tuning mode."""
    _dev(x, perm, offsets, slot_of, slab)
    rows = perm.numel()
    act = torch.empty((rows, ffn), dtype=torch.bfloat16, device=x.device)
    _lib.call("daop_expert_gemm_up_gather", x.data_ptr(), x.shape[0], perm.data_ptr(), k, rows, d,
              ffn, slab.data_ptr(), n_slots, slot_elems, offsets.data_ptr(), slot_of.data_ptr(),
              offsets.numel() - 1, act.data_ptr(), group_m, _s())
    return act


SKINNY_NTS = (32, 48, 64, 80, 96, 128)


def skinny_nt(rows: int, experts: int = 0) -> int:
    """Token block (the MMA's N) of the skinny GEMMs for `rows` permuted rows
    (T * k) over `experts` experts: the smallest instantiated block holding
    1.25x the mean rows per expert, so one block usually covers an expert's
    tokens and the stages stream few empty token rows (256-token prompt:
    64 rows per expert -> 80).  experts = 0: by rows alone (32 / 64 / 128)."""
    if experts <= 0:
        return 32 if rows <= 32 else 64 if rows <= SKINNY_NT128_ROWS else 128
    want = -(-5 * rows // (4 * experts))
    return next((nt for nt in SKINNY_NTS if nt >= want), 128)


SKINNY_NT128_ROWS = 384


def expert_gemm_up_skinny(x_perm, offsets, slot_of, slab, n_slots, slot_elems, d, ffn, nt=0,
                          out=None):
    """Up GEMM for small token counts (weights as the M side); like
    expert_gemm_up, rows of experts with slot -1 in `out` are left untouched."""
    _dev(x_perm, offsets, slot_of, slab, out)
    rows = x_perm.shape[0]
    act = torch.empty((rows, ffn), dtype=torch.bfloat16, device=x_perm.device) if out is None \
        else out
    _lib.call("daop_expert_gemm_up_skinny", x_perm.data_ptr(), rows, d, ffn, slab.data_ptr(),
              n_slots, slot_elems, offsets.data_ptr(), slot_of.data_ptr(), offsets.numel() - 1,
              act.data_ptr(), nt or skinny_nt(rows, offsets.numel() - 1), _s())
    return act


def expert_gemm_down_skinny(act, offsets, slot_of, slab, n_slots, slot_elems, d, ffn, nt=0,
                            out=None):
    _dev(act, offsets, slot_of, slab, out)
    rows = act.shape[0]
    y = torch.empty((rows, d), dtype=torch.float32, device=act.device) if out is None else out
    _lib.call("daop_expert_gemm_down_skinny", act.data_ptr(), rows, d, ffn, slab.data_ptr(),
              n_slots, slot_elems, offsets.data_ptr(), slot_of.data_ptr(), offsets.numel() - 1,
              y.data_ptr(), nt or skinny_nt(rows, offsets.numel() - 1), _s())
    return y


def expert_gemm_down(act, offsets, slot_of, slab, n_slots, slot_elems, d, ffn, group_m=0,
                     out=None):
    _dev(act, offsets, slot_of, slab, out)
    rows = act.shape[0]
    y = torch.empty((rows, d), dtype=torch.float32, device=act.device) if out is None else out
    _lib.call("daop_expert_gemm_down", act.data_ptr(), rows, d, ffn, slab.data_ptr(), n_slots,
              slot_elems, offsets.data_ptr(), slot_of.data_ptr(), offsets.numel() - 1,
              y.data_ptr(), group_m, _s())
    return y


def expert_gemm_down_combine(act, offsets, slot_of, slab, n_slots, slot_elems, d, ffn, perm,
                             inv, h, w, group_m=0):
    """Down GEMM + combine in one kernel (daop_expert_gemm_down_combine):
    returns (out (T, d) = h + sum_j w_j y_j, y).  Raises DeviceError when the
    fused form is unavailable (single-CTA tuning mode)."""
    _dev(act, offsets, slot_of, slab, perm, inv, h, w)
    rows = act.shape[0]
    t, k = inv.shape
    y = torch.empty((rows, d), dtype=torch.float32, device=act.device)
    out = torch.empty_like(h)
    cnt = torch.zeros((t, d // 256), dtype=torch.int32, device=act.device)
    _lib.call("daop_expert_gemm_down_combine", act.data_ptr(), rows, d, ffn, slab.data_ptr(),
              n_slots, slot_elems, offsets.data_ptr(), slot_of.data_ptr(), offsets.numel() - 1,
              y.data_ptr(), perm.data_ptr(), inv.data_ptr(), h.data_ptr(), w.data_ptr(), k,
              out.data_ptr(), cnt.data_ptr(), group_m, _s())
    return out, y


def combine(h, y_sorted, inv, w, out=None):
    _dev(h, y_sorted, inv, w, out)
    t, d = h.shape
    k = inv.shape[1]
    out = torch.empty_like(h) if out is None else out
    _lib.call("daop_combine", h.data_ptr(), y_sorted.data_ptr(), inv.data_ptr(), w.data_ptr(),
              t, k, d, out.data_ptr(), _s())
    return out


def _pad16(n: int) -> int:
    return (n + 15) // 16 * 16


class DecodeBuffers:
    """Preallocated outputs + self-resetting workspace of one decode layer call
    (fixed addresses, so a decode step can be captured in a CUDA graph).

    All outputs live in ONE device buffer so the host reads what it needs in
    one copy:  [x | p | p_pred | w | deg | is_fast | sel | h_out]  (16-byte
    aligned fields).  The DAOP engine copies the prefix up to `sel` (the
    decisions + the stale input of the host tier); the end-to-end host call
    copies the suffix [sel | h_out]."""

    def __init__(self, d, ffn, num_experts, k, device):
        nb = torch.zeros(1, dtype=torch.int64)
        _lib.call("daop_decode_workspace", d, ffn, num_experts, k, nb.data_ptr())
        self.ws = torch.zeros(int(nb[0]), dtype=torch.uint8, device=device)
        e = num_experts
        sizes = [("x", 2 * d), ("p", 4 * e), ("p_pred", 4 * e), ("w", 4 * k),
                 ("deg", 4 * (2 * k + 1)), ("is_fast", k), ("sel", 4 * k), ("h_out", 4 * d)]
        off, o = {}, 0
        for name, n in sizes:
            off[name] = o
            o += _pad16(n)
        self.meta = torch.zeros(o, dtype=torch.uint8, device=device)
        self.offsets = off
        dt = {"x": torch.bfloat16, "p": torch.float32, "p_pred": torch.float32,
              "w": torch.float32, "deg": torch.int32, "is_fast": torch.uint8,
              "sel": torch.int32, "h_out": torch.float32}
        for name, n in sizes:
            setattr(self, name, self.meta[off[name]: off[name] + n].view(dt[name]))
        self.decisions_bytes = off["sel"] + _pad16(4 * k)  # prefix: x .. sel
        self.io_offset = off["sel"]                         # suffix: sel | h_out
        self.y = torch.zeros((k, d), dtype=torch.float32, device=device)


def decode_layer(h, gamma, wg, wg_next, fast_row, slot_of, slab, slot_elems, d, ffn, k,
                 bufs: DecodeBuffers, *, pred_prev=None, mode=0, graceful=True,
                 weights_from_pred=False, variant=0, eps=RMS_EPS, h_out=None, sel_out=None):
    """One decode token through one MoE layer in a single launch.

    h_out / sel_out (optional) redirect the residual and the selection to
    other buffers -- e.g. pinned host memory, which the kernel then writes
    directly over the bus (the end-to-end call needs no D2H copy)."""
    _dev(h, gamma, wg, wg_next, pred_prev, fast_row, slot_of, slab)
    for t in (h_out, sel_out):
        if t is not None and not (t.is_cuda or t.is_pinned()):
            raise DeviceError("h_out / sel_out must be device or pinned host memory")
    e = wg.shape[0]
    _lib.call("daop_decode_layer", h.data_ptr(), gamma.data_ptr(), wg.data_ptr(), _p(wg_next),
              _p(pred_prev), fast_row.data_ptr(), slot_of.data_ptr(), slab.data_ptr(),
              slot_elems, d, ffn, e, k, mode, int(graceful), int(weights_from_pred), float(eps),
              bufs.x.data_ptr(), bufs.p.data_ptr(), bufs.p_pred.data_ptr(),
              (bufs.sel if sel_out is None else sel_out).data_ptr(),
              bufs.w.data_ptr(), bufs.is_fast.data_ptr(), bufs.deg.data_ptr(),
              bufs.y.data_ptr(), (bufs.h_out if h_out is None else h_out).data_ptr(),
              bufs.ws.data_ptr(), variant, _s())
    return bufs
