"""B200-native Krul state-restoration hot path (arxiv 2507.08045).

The product is libkrul_b200.so (sm_100a CUDA kernels + C++ host behind the C
ABI in include/krul_b200.h). This package is its Python mirror; see native.py.
"""
from . import native  # noqa: F401
from .native import (  # noqa: F401
    AccountingError, ClassificationError, CompressionStrategy, ConfigError, Context, Conversation,
    CostModel, KrulError, KVSnapshot, ModelConfig, PlanInvalidError, RestorationGapError,
    SnapshotError, StateCorruptionError, StreamingEstimator, build_plan, calibrate_rc,
    default_rc_grid, plan_blob_specs, select_strategy, shared_layer_quota, simulate_pipeline,
    uniform_plan, validate_plan,
)
