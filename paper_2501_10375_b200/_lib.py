"""ctypes binding of libdaop_b200.so (the C ABI in include/daop_b200.h).

There is exactly one backend: if the shared library is missing the import
fails loudly -- there is no Python/CPU fallback for any hot-path operation.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import errors as E

LIB_PATH = Path(__file__).resolve().parent / "libdaop_b200.so"

P = C.c_void_p
I32, I64, U64, F32, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double

# name -> argtypes (every function returns int status)
PROTOS = {
    "daop_version": [],
    "daop_device_info": [P, P, P],
    "daop_graph_step": [P, P, P, P, I64],
    "daop_graph_step_mode": [I32],
    "daop_server_start": [P, P, P, P, P, P, I64, I32, I32, I32, I32, F32, P, P, P, P, P, P, P,
                          P, P, P, F64, P, P],
    "daop_server_step": [P, P, F64],
    "daop_server_stop": [P],
    "daop_attn_workspace": [I32, I32, I32, P],
    "daop_attn_norm_rows": [P, I64, P, I32, F32, P, P],
    "daop_attn_prefill": [P, I64, I32, P, P, I32, I32, I32, F32, P, P],
    "daop_attn_decode": [P, P, P, P, P, P, I32, I32, I32, I32, I32, F32, F32, P, P, P, P],
    "daop_server_trace": [P, I32],
    "daop_set_attn_fused": [I32],
    "daop_attn_timeline": [I32, P],
    "daop_gemm_timeline": [I32, P],
    "daop_die_map": [P, I32, P],
    "daop_set_gemm_die_table": [P, I32],
    "daop_die_pair_probe": [P, I64, I32, I32, P, P],
    "daop_die_probe": [P, I32, I32, I32, P, P, P],
    "daop_topk_rows_f64": [P, I64, I32, I32, P, P],
    "daop_topk_rows_f32": [P, I64, I32, I32, P, P],
    "daop_activation_counts": [P, I64, I32, I32, I32, P, P],
    "daop_pair_overlap": [P, P, I64, I32, I32, P, P],
    "daop_slot_budget": [F64, I32, I32, P],
    "daop_placement_init": [P, I32, I32, F64, P, P],
    "daop_allocate": [P, P, I32, I32, I64, I64, P, P, P],
    "daop_degrade_f64": [P, I32, P, I32, P, P, P, P],
    "daop_plan_token_f64": [P, P, P, P, I32, I32, I32, I32, I32, I32, P, P, P, P, P],
    "daop_plan_layer_f32": [P, P, P, I64, I32, I32, I32, I32, I32, I32, P, P, P, P, P, P],
    "daop_fill_uniform_bf16": [P, I64, U64, U64, F32, I64, P],
    "daop_fill_uniform_f32": [P, I64, U64, U64, F32, I64, P],
    "daop_fill_norm_bf16": [P, I64, U64, I32, P],
    "daop_fill_uniform_bf16_host": [P, I64, U64, U64, F32, I64, I32],
    "daop_router": [P, P, P, P, I64, I32, I32, I32, F32, P, P, P, P, P, P, I64, I64, P],
    "daop_permute_workspace": [I64, I32, I32, P],
    "daop_permute": [P, I64, I32, I32, P, I32, P, P, P, P, P, I64, P],
    "daop_combine": [P, P, P, P, I64, I32, I32, P, P],
    "daop_set_gemm_mode": [I32],
    "daop_expert_gemm_up": [P, I64, I32, I32, P, I64, I64, P, P, I32, P, I32, P],
    "daop_expert_gemm_up_gather": [P, I64, P, I32, I64, I32, I32, P, I64, I64, P, P, I32, P, I32,
                                   P],
    "daop_expert_gemm_down": [P, I64, I32, I32, P, I64, I64, P, P, I32, P, I32, P],
    "daop_gemm_bf16_f32": [P, I64, I32, P, I32, P, P, P],
    "daop_gemm_bf16_f32_ws": [P, I64, I32, P, I32, P, P, P, I64, P],
    "daop_set_router_mode": [I32],
    "daop_set_stream_mode": [I32, I32, I32, I32],
    "daop_l2_prefetch": [P, I64, P, I64, P],
    "daop_gemm_prepare": [],
    "daop_host_pool_alloc": [I64, I32, P, P],
    "daop_host_pool_free": [P, I64, I32],
    "daop_expert_gemm_up_skinny": [P, I64, I32, I32, P, I64, I64, P, P, I32, P, I32, P],
    "daop_expert_gemm_down_skinny": [P, I64, I32, I32, P, I64, I64, P, P, I32, P, I32, P],
    "daop_expert_gemm_down_combine": [P, I64, I32, I32, P, I64, I64, P, P, I32, P, P, P, P, P,
                                      I32, P, P, I32, P],
    "daop_ep_ws_layout": [I32, I32, I32, I64, I64, P, P, P, P],
    "daop_ep_publish": [P, I32, I32, I32, P, C.c_uint32, P],
    "daop_ep_dispatch": [P, I32, I32, I32, I32, I32, P, P, I64, I64, C.c_uint32, P],
    "daop_ep_recv": [P, I32, I32, I32, I32, I64, C.c_uint32, P],
    "daop_ep_expert_gemm_down": [P, I64, I32, I32, P, I64, I64, P, I32, P, P, I32, I32,
                                 C.c_uint32, I32, P],
    "daop_ep_wait_back": [P, I32, C.c_uint32, P],
    "daop_ep_expert_gemm_down_skinny": [P, I64, I32, I32, P, I64, I64, P, I32, P, P, I32, I32,
                                        C.c_uint32, I32, P],
    "daop_ep_status": [P, P],
    "daop_ep_decode_ws_bytes": [I32, I32, P],
    "daop_ep_decode_share": [P, I32, I32, I32, I32, P, P, C.c_uint32, P],
    "daop_ep_decode_wait": [P, I32, C.c_uint32, P],
    "daop_ep_decode_layer": [P, I32, I32, C.c_uint32, P, P, P, P, P, P, P, I64, I32, I32, I32,
                             I32, F32, P, P, P, P, P, P, P, P, P, P, P],
    "daop_ep_decode_finish": [P, I32, I32, I32, P, P, P, C.c_uint32, P],
    "daop_ep_ipc_handle": [P, P, P],
    "daop_ep_ipc_open": [P, I64, P, P],
    "daop_ep_ipc_close": [P],
    "daop_decode_workspace": [I32, I32, I32, I32, P],
    "daop_decode_timeline": [I32, P, I32],
    "daop_combine_dense": [P, P, P, I32, I32, P, P],
    "daop_host_expert_ffn": [P, I64, P, P, P, I32, I32, P, P, I32],
    "daop_host_expert_ffn_rows": [P, I64, P, P, P, I32, I32, I32, I32, P, I32],
    "daop_slow_split_pull": [P, P, P, I32, I32, I32, P, P],
    "daop_host_caps": [P, P],
    "daop_host_set_grain": [I64, I64],
    "daop_host_stream_read": [P, I64, I32, P],
    "daop_lru_plan_layer": [I32, I32, I32, I32, I32, I32, P, P, P, P, P, P, P, P, P, P, P, P],
    "daop_trace_format_phase": [P, P, P, I64, I32, I32, I32, P, I64, P],
    "daop_decode_layer": [P, P, P, P, P, P, P, P, I64, I32, I32, I32, I32, I32, I32, I32, F32,
                          P, P, P, P, P, P, P, P, P, P, I32, P],
}

_CODES = {
    -1: E.ShapeMismatchError,
    -2: E.NormalizationError,
    -3: E.BudgetError,
    -4: E.PredictionMissingError,
    -5: E.ConfigError,
    -6: E.EmptyPhaseError,
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH.name} is not built; run `python paper_2501_10375_b200/build.py` "
            "(nvcc, sm_100a). There is no CPU fallback."
        )
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, args in PROTOS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.daop_last_error.argtypes = []
    lib.daop_last_error.restype = C.c_char_p
    return lib


LIB = _load()


def exported_symbols():
    return sorted(PROTOS) + ["daop_last_error"]


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = LIB.daop_last_error().decode(errors="replace")
    cls = _CODES.get(rc)
    if cls is not None:
        raise cls(msg)
    raise E.DeviceError(f"{what}: {msg} (code {rc})")


def call(name: str, *args) -> None:
    check(getattr(LIB, name)(*args), name)


def ptr(a) -> int:
    """Raw address of a numpy array or torch tensor (no copies)."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
