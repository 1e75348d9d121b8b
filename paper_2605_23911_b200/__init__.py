"""B200-native fused MoE-layer forward (sm_100a), drop-in for the reference
``moeperf`` hot path (``moeperf/pipeline.py:572`` ``moe_forward``).

Public API mirrors the reference's names (``moeperf/__init__.py:56-78``):
``moe_forward``, ``route``, ``ModelConfig``, ``Gating``, ``ExpertWeights``,
``PipelineParams``, ``RoutingResult``, the error classes, and the trace
types.  ``MoELayer`` is the resident-weights device layer used by the bench.
"""

from .errors import (
    AllZero,
    DegenerateStage,
    DeviceError,
    IndexOutOfRange,
    InvalidBlockM,
    InvalidK,
    InvalidSpec,
    MissingPeakFlops,
    MoeperfError,
    NativeLibraryMissing,
    NonFiniteInput,
    ScheduleMismatch,
    ShapeMismatch,
)
from .trace import (
    DEVICE_STAGES,
    PipelineTrace,
    StageRecord,
    TrafficReport,
    activation_traffic_closed_form,
    build_block_schedule,
    expert_offsets,
    stage_bytes,
    stage_flops,
    trace_from_counts,
    traffic_from_measured,
    traffic_from_traces,
)
from .types import (
    MODEL_PRESETS,
    BlockSchedule,
    ExpertOffsets,
    ExpertWeights,
    Gating,
    ModelConfig,
    Permutation,
    PipelineParams,
    RoutingResult,
    preset,
)

__version__ = "0.1.0"


_LAYER_NAMES = ("MoELayer", "HostPipeline", "DeviceExpertWeights", "upload_weights", "moe_forward", "route")
# the reference's stage-level API (moeperf/__init__.py:56-78) on the device
_STAGE_NAMES = ("gate_scores", "stable_softmax_row", "topk_select", "expert_histogram", "build_permutation",
                "permute_tokens", "fused_gate_up", "unfused_gate_up", "grouped_gemm", "unpermute_combine",
                "sigmoid", "silu", "dense_matmul", "dense_moe_oracle")


def __getattr__(name):
    # Device-facing symbols import torch lazily so host-only users (trace,
    # types) do not pay for it.
    if name in _LAYER_NAMES:
        from . import layer

        return getattr(layer, name)
    if name in _STAGE_NAMES:
        from . import stages

        return getattr(stages, name)
    raise AttributeError(name)
