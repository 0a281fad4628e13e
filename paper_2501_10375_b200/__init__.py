"""paper_2501_10375_b200 -- B200-native DAOP MoE-block hot path.

Drop-in for the hot path of the reference package ``moesim`` (DAOP,
arXiv 2501.10375): the same names for the routing/placement/planning API
(moesim/__init__.py:87-151), backed by hand-written sm_100a CUDA kernels and
native host code in libdaop_b200.so, plus the numeric engine the reference
only simulates (fused router, permutation, grouped SwiGLU experts, combine,
expert migration) -- see DESIGN.md.
"""

from .errors import (BudgetError, ConfigError, DeviceError, EmptyPhaseError,
                     GeneratorTargetError, MoesimError, NormalizationError,
                     PredictionMissingError, ShapeMismatchError,
                     TooShortSequenceError, TraceParseError)
from .trace import (MIXTRAL_SHAPE, PHI_SHAPE, SCORE_SUM_TOL, ModelShape,
                    RoutingTrace, TokenRouting, load_trace, parse_shape,
                    save_trace, softmax)
from . import kernels as _kernels
from .metrics import (ActivationMatrix, activation_matrix, expert_counts,
                      mean_prediction_accuracy, pooled_decode_probabilities,
                      prediction_accuracy, routing_fidelity, row_cosines,
                      similarity)
from .placement import (SWAP_IN_OUT_DEFAULT, ExpertPlacement, SwapEvent,
                        allocate_for_sequence, init_from_calibration,
                        slot_budget_for_ecr)
from .policies import (ENGINES, PREDICTION_START_LAYER_DEFAULT, DaopPlanner,
                       Degradation, ExecutedExpert, FiddlerPlanner, LayerPlan,
                       OnDemandPlanner, PolicyConfig, PrefetchPlanner,
                       decode_counters, degrade_selection, make_planner,
                       plan_token_daop, plan_token_fiddler, plan_token_ondemand,
                       plan_token_prefetch, plan_trace_decode)

from .experiment import CSV_SCHEMA_VERSION, TimelineResult, run_single

__version__ = "0.2.0"

__all__ = [
    "BudgetError", "ConfigError", "DeviceError", "EmptyPhaseError",
    "GeneratorTargetError", "MoesimError", "NormalizationError",
    "PredictionMissingError", "ShapeMismatchError", "TooShortSequenceError",
    "TraceParseError", "MIXTRAL_SHAPE", "PHI_SHAPE", "SCORE_SUM_TOL",
    "ModelShape", "RoutingTrace", "TokenRouting", "softmax", "save_trace",
    "load_trace", "parse_shape", "ActivationMatrix",
    "activation_matrix", "expert_counts", "mean_prediction_accuracy",
    "pooled_decode_probabilities", "prediction_accuracy", "routing_fidelity",
    "SWAP_IN_OUT_DEFAULT", "ExpertPlacement", "SwapEvent",
    "allocate_for_sequence", "init_from_calibration", "slot_budget_for_ecr",
    "ENGINES", "PREDICTION_START_LAYER_DEFAULT", "DaopPlanner", "Degradation",
    "ExecutedExpert", "FiddlerPlanner", "LayerPlan", "PolicyConfig",
    "decode_counters", "degrade_selection", "make_planner", "plan_token_daop",
    "plan_token_fiddler", "plan_trace_decode", "OnDemandPlanner", "PrefetchPlanner",
    "plan_token_ondemand", "plan_token_prefetch", "row_cosines", "similarity",
    "CSV_SCHEMA_VERSION", "TimelineResult", "run_single",
]
