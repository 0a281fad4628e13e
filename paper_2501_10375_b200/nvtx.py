"""NVTX ranges per layer and phase (SURVEY §5 tracing): `DAOP_NVTX=1` turns
them on for a profiler (ncu --nvtx / nsys); off by default, where a range
costs one flag test.  Names: "prefill/L{l}/router", "decode/L{l}", ..."""

from __future__ import annotations

import contextlib
import os

ENABLED = os.environ.get("DAOP_NVTX", "0") == "1"


@contextlib.contextmanager
def nvtx_range(name: str):
    if not ENABLED:
        yield
        return
    import torch
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()


def nvtx_push(name: str) -> None:
    if ENABLED:
        import torch
        torch.cuda.nvtx.range_push(name)


def nvtx_pop() -> None:
    if ENABLED:
        import torch
        torch.cuda.nvtx.range_pop()
