"""The drop-in boundary, CPU-side: the library loads and binds every symbol,
errors map onto the reference's exception classes, and the hot path fails
loudly instead of falling back to the CPU."""

import numpy as np
import pytest
import torch

import paper_2501_10375_b200 as P
from paper_2501_10375_b200 import _lib, ops
from paper_2501_10375_b200.errors import DeviceError


def test_reference_api_names_present():
    # the hot-path subset of moesim/__init__.py:87-151
    for name in ["ModelShape", "MIXTRAL_SHAPE", "PHI_SHAPE", "RoutingTrace", "TokenRouting",
                 "ExpertPlacement", "SwapEvent", "init_from_calibration",
                 "allocate_for_sequence", "slot_budget_for_ecr", "PolicyConfig",
                 "make_planner", "plan_token_daop", "plan_token_fiddler", "plan_trace_decode",
                 "degrade_selection", "DaopPlanner", "FiddlerPlanner", "LayerPlan",
                 "ExecutedExpert", "Degradation", "expert_counts", "activation_matrix",
                 "prediction_accuracy", "routing_fidelity", "ActivationMatrix",
                 "MoesimError", "ShapeMismatchError", "BudgetError", "ConfigError",
                 "PredictionMissingError", "NormalizationError", "EmptyPhaseError",
                 "SWAP_IN_OUT_DEFAULT", "PREDICTION_START_LAYER_DEFAULT", "ENGINES"]:
        assert hasattr(P, name), name
    assert P.MIXTRAL_SHAPE == P.ModelShape(32, 8, 2)
    assert P.SWAP_IN_OUT_DEFAULT == 1.05 and P.PREDICTION_START_LAYER_DEFAULT == 4


def test_error_codes_map_to_reference_classes():
    with pytest.raises(P.BudgetError) as ei:
        P.init_from_calibration(np.ones((4, 4)), 0.1, P.ModelShape(4, 4, 2))
    # the native code's message is carried into the raised exception
    msg = _lib.LIB.daop_last_error().decode()
    assert "budget" in msg.lower() and msg in str(ei.value)
    with pytest.raises(P.BudgetError):
        P.init_from_calibration(np.ones((4, 4)), float("nan"), P.ModelShape(4, 4, 2))
    with pytest.raises(P.ShapeMismatchError):
        P.init_from_calibration(np.ones((2, 4)), 0.5, P.ModelShape(3, 4, 2))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_hot_path_fails_loudly_without_gpu():
    with pytest.raises(DeviceError):
        P._kernels.topk_rows(np.array([[0.5, 0.5]]), 1)
    h = torch.zeros((4, 64))
    g = torch.zeros(64, dtype=torch.bfloat16)
    w = torch.zeros((8, 64), dtype=torch.bfloat16)
    with pytest.raises(DeviceError):
        ops.router(h, g, w, None, 2)
    with pytest.raises(DeviceError):
        ops.combine(h, h, torch.zeros((4, 1), dtype=torch.int32), torch.zeros((4, 1)))


def test_no_cpu_compute_symbols_hidden_behind_python():
    # every device op in ops.py goes through the C ABI (no torch math fallback)
    import inspect
    src = inspect.getsource(ops)
    for banned in ("torch.matmul", "torch.softmax", "F.silu", "torch.topk", "@ "):
        assert banned not in src, banned


def test_routing_trace_validation_matches_reference_rules():
    shape = P.ModelShape(2, 4, 2)
    good = np.array([0.4, 0.3, 0.2, 0.1])
    with pytest.raises(P.NormalizationError):
        P.TokenRouting(np.array([0.5, 0.5, 0.5, 0.5]))
    with pytest.raises(P.ShapeMismatchError):  # prediction on the last layer
        P.RoutingTrace(shape, "x", good[None, None, :].repeat(2, 1), np.zeros((0, 2, 4)),
                       prefill_predicted=good[None, None, :].repeat(2, 1),
                       prefill_mask=np.array([[True, True]]))
    t = P.RoutingTrace.from_token_lists(shape, "y", [[P.TokenRouting(good, good),
                                                     P.TokenRouting(good)]])
    assert t.num_prefill_tokens == 1 and t.prefill_mask.tolist() == [[True, False]]


def test_ep_workspace_layout_host_rules():
    """The symmetric EP workspace layout is host arithmetic: offsets are
    aligned, the receive buffer and y_back fit, bad worlds are refused."""
    import torch
    from paper_2501_10375_b200 import _lib
    from paper_2501_10375_b200.errors import DeviceError
    out = [torch.zeros(1, dtype=torch.int64) for _ in range(4)]
    ptrs = [o.data_ptr() for o in out]
    _lib.call("daop_ep_ws_layout", 4, 8, 4096, 1000, 500, *ptrs)
    total, recv_off, yback_off, local_off = (int(o[0]) for o in out)
    assert recv_off % 4096 == 0 and yback_off % 4096 == 0 and total % 4096 == 0
    assert yback_off >= recv_off + 1000 * 4096 * 2
    assert total >= yback_off + 500 * 4096 * 4
    assert local_off < 16384  # local offsets live in the header, before the row table
    for bad in [(3, 8), (16, 16), (2, 65)]:  # E % G != 0, G > 8, E > 64
        with pytest.raises(DeviceError):
            _lib.call("daop_ep_ws_layout", bad[0], bad[1], 4096, 10, 10, *ptrs)


def test_attention_workspace_size():
    import torch
    from paper_2501_10375_b200 import _lib
    nb = torch.zeros(1, dtype=torch.int64)
    _lib.call("daop_attn_workspace", 32, 8, 4096, nb.data_ptr())
    q, kv = 32 * 128, 8 * 128
    # qkv fp32 + split partials (8 kv heads x 64 splits x 4 heads x 130) + o bf16 + counters
    assert int(nb[0]) >= (q + 2 * kv) * 4 + 8 * 64 * 4 * 130 * 4 + q * 2 + 4 * 8


def test_skinny_token_block_rule():
    """The skinny GEMMs' token block covers ~1.25x the mean rows per expert
    with an instantiated NT (decode b = 64 -> 32; 256-token prompt -> 80)."""
    assert ops.skinny_nt(128, 8) == 32
    assert ops.skinny_nt(512, 8) == 80
    assert ops.skinny_nt(768, 8) == 128
    assert ops.skinny_nt(10_000, 8) == 128
    assert all(ops.skinny_nt(r, e) in ops.SKINNY_NTS for r in range(1, 2000, 37) for e in (1, 4, 8, 16))
    assert ops.skinny_nt(64) == 64 and ops.skinny_nt(16) == 32  # by rows alone
