"""Operator table -- drop-in for ``moesim._kernels`` (_kernels.py:104-126).

Module-level functions with the reference's names and signatures, resolved
at call time exactly like the reference resolves its own (metrics.py:59,70,
policies.py:180,302,318).  Every call runs the sm_100a kernels in
libdaop_b200.so; numpy inputs are staged through the device and results come
back as freshly allocated caller-owned numpy arrays (the reference's ownership
rule, _kernels.py:37,105).  torch CUDA tensors are accepted without copies and
return torch tensors.  There is no CPU backend: without a CUDA device these
raise DeviceError.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import DeviceError

BACKEND = "cuda-sm100a"
HAVE_NUMBA = False
NUMBA_DISABLED = True


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("the operator table runs on an sm_100a CUDA device; none is visible")
    return torch


def _to_dev(a, dtype):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous(), True
    arr = np.ascontiguousarray(a)
    if not arr.flags.writeable:  # read-only trace arrays: torch wants a writable buffer
        arr = arr.copy()
    return torch.from_numpy(arr).to(device="cuda", dtype=dtype).contiguous(), False


def topk_rows(scores, k: int):
    """(N, E) scores -> (N, k) int64 ids, highest first, ties to lower index."""
    torch = _torch()
    is_t = isinstance(scores, torch.Tensor)
    dtype = scores.dtype if is_t and scores.dtype in (torch.float32, torch.float64) else torch.float64
    s, _ = _to_dev(scores, dtype)
    if s.dim() != 2:
        s = s.reshape(-1, s.shape[-1])
    n, e = s.shape
    out = torch.empty((n, k), dtype=torch.int64, device=s.device)
    fn = "daop_topk_rows_f32" if s.dtype == torch.float32 else "daop_topk_rows_f64"
    _lib.call(fn, s.data_ptr(), n, e, int(k), out.data_ptr(), _lib.stream_handle())
    return out if is_t else out.cpu().numpy()


def activation_counts(topk, num_experts: int):
    """(T, L, k) ids -> (L, E) float64 counts (dtype as _kernels.py:55)."""
    torch = _torch()
    is_t = isinstance(topk, torch.Tensor)
    ids, _ = _to_dev(topk, torch.int64)
    t, l, k = ids.shape
    counts = torch.zeros((l, num_experts), dtype=torch.int64, device=ids.device)
    _lib.call("daop_activation_counts", ids.data_ptr(), t, l, k, int(num_experts),
              counts.data_ptr(), _lib.stream_handle())
    out = counts.to(torch.float64)
    return out if is_t else out.cpu().numpy()


def pair_overlap(a, b):
    """Per-row |a ∩ b| of two (N, ka) / (N, kb) id arrays -> (N,) int64."""
    torch = _torch()
    is_t = isinstance(a, torch.Tensor)
    da, _ = _to_dev(a, torch.int64)
    db, _ = _to_dev(b, torch.int64)
    n, ka = da.shape
    out = torch.empty((n,), dtype=torch.int64, device=da.device)
    _lib.call("daop_pair_overlap", da.data_ptr(), db.data_ptr(), n, ka, db.shape[1],
              out.data_ptr(), _lib.stream_handle())
    return out if is_t else out.cpu().numpy()


def warmup() -> None:
    """Load the module and touch every kernel once (no JIT to warm)."""
    s = np.array([[0.5, 0.3, 0.2], [0.1, 0.1, 0.8]])
    idx = topk_rows(s, 2)
    pair_overlap(idx, idx)
    activation_counts(idx[:, None, :], 3)
