"""paper_2211_00391_b200: B200-native (sm_100a) oblivious-ensemble predict.

A drop-in for the reference ``obtree`` package's model-loading and predict surface
(pkg/src/obtree/__init__.py): the same model types, document format, configuration
and ``Evaluator`` / ``evaluate`` calls, with quantize -> leaf index -> leaf
gather/accumulate running as hand-written CUDA kernels behind a C ABI
(include/obtree_b200.h).  There is no CPU compute path.
"""

from .config import BLOCK_SIZES, EvalConfig, LeafStrategy, TailPolicy
from .evaluate import DeviceModel, Evaluator, ModelTables, evaluate
from .matrix import FeatureMatrix, Layout, VectorWidth
from .metrics import DeviationMetrics, classification_flip_count, deviation_metrics
from .model import (
    HALF_MAX,
    MAX_BORDERS,
    MAX_DEPTH,
    FloatFeatureBorders,
    LeafBank,
    LeafPrecision,
    ObliviousModel,
    ObliviousTree,
    SplitCondition,
    build_leaf_bank,
    require_valid,
    validate_model,
)
from .serialize import ModelFormatError, deserialize_model, load_model, save_model, serialize_model
from ._native import NativeError, NativeUnavailable

__version__ = "0.1.0"

__all__ = [
    "BLOCK_SIZES",
    "DeviationMetrics",
    "DeviceModel",
    "EvalConfig",
    "Evaluator",
    "FeatureMatrix",
    "FloatFeatureBorders",
    "HALF_MAX",
    "Layout",
    "LeafBank",
    "LeafPrecision",
    "LeafStrategy",
    "MAX_BORDERS",
    "MAX_DEPTH",
    "ModelFormatError",
    "ModelTables",
    "NativeError",
    "NativeUnavailable",
    "ObliviousModel",
    "ObliviousTree",
    "SplitCondition",
    "TailPolicy",
    "VectorWidth",
    "build_leaf_bank",
    "classification_flip_count",
    "deserialize_model",
    "deviation_metrics",
    "evaluate",
    "load_model",
    "require_valid",
    "save_model",
    "serialize_model",
    "validate_model",
]
