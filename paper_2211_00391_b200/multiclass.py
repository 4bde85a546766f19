"""Multi-output oblivious ensembles (BASELINE config 5: 10 outputs, depth 10).

The reference cannot express these models (depth <= 8, one output: model.py:21-22,
SPEC.md:15), so this module extends its semantics the natural way, as the CPU
restatement in oracle/ does: every tree has one leaf table per output,
all outputs share the tree's splits, each output folds its leaves in tree order in
binary64, and prediction[o][c] = scale * sum_t leaf[t][c][index_t(o)] + bias.

The binary16 family (``EvalConfig(strategy=NAIVE16 | PERMUTE16)``) extends the same way:
each output's leaves go through the reference's binary16 bank (model.py:262-268: RNE,
saturation to +/-65504) and fold in binary32 (accumulate.py:94-97) -- the multiclass
FP16 permutation the paper leaves as future work ("if each leaf holds 2 or
4 values, combine the 16-bit numbers into 32- or 64-bit words").  On the GPU a leaf's C
binary16 values sit two per 32-bit word in one record, and the fold adds two outputs
per packed FADD2.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _checks, _native
from .config import EvalConfig, LeafPrecision
from .matrix import FeatureMatrix, Layout, layout_code
from .model import MAX_BORDERS, half_bank_values

MAX_MULTI_DEPTH = 12
MAX_OUTPUTS = 16
SENTINEL = 255


@dataclass
class MultiOutputModel:
    borders: list            # per feature: float32 strictly ascending, <= 254
    split_feature: np.ndarray  # int32 [T][D]
    split_ordinal: np.ndarray  # int [T][D]; 255 marks an unused (shallower-tree) level
    leaves: np.ndarray       # float64 [T][C][2^D]
    scale: float = 1.0
    bias: float = 0.0

    def __post_init__(self):
        self.borders = [np.ascontiguousarray(b, dtype=np.float32) for b in self.borders]
        self.split_feature = np.ascontiguousarray(self.split_feature, dtype=np.int32)
        self.split_ordinal = np.ascontiguousarray(self.split_ordinal, dtype=np.int32)
        self.leaves = np.ascontiguousarray(self.leaves, dtype=np.float64)
        self.scale, self.bias = float(self.scale), float(self.bias)

    @property
    def n_features(self) -> int:
        return len(self.borders)

    @property
    def n_trees(self) -> int:
        return self.split_feature.shape[0]

    @property
    def depth(self) -> int:
        return self.split_feature.shape[1] if self.split_feature.ndim == 2 else 0

    @property
    def n_outputs(self) -> int:
        return self.leaves.shape[1]

    def validate(self) -> list:
        errors = []
        if self.n_features == 0:
            errors.append("model: at least one float feature is required")
        for f, b in enumerate(self.borders):
            if b.size > MAX_BORDERS:
                errors.append(f"float_features[{f}]: {b.size} borders exceed the limit of {MAX_BORDERS}")
            if np.isnan(b).any():
                errors.append(f"float_features[{f}]: NaN border")
            elif b.size > 1 and not bool(np.all(np.diff(b) > 0)):
                errors.append(f"float_features[{f}]: non-ascending borders")
        T, D = self.split_feature.shape if self.split_feature.ndim == 2 else (0, 0)
        if not 1 <= D <= MAX_MULTI_DEPTH and T:
            errors.append(f"depth {D} outside 1..{MAX_MULTI_DEPTH}")
        if self.leaves.shape != (T, self.leaves.shape[1] if self.leaves.ndim == 3 else 0, 1 << D) or self.leaves.ndim != 3:
            errors.append(f"leaves must be [T][C][2^depth] = [{T}][C][{1 << D}]")
        elif not 2 <= self.leaves.shape[1] <= MAX_OUTPUTS:
            errors.append(f"{self.leaves.shape[1]} outputs outside 2..{MAX_OUTPUTS}")
        if np.isnan(self.leaves).any():
            errors.append("NaN leaf value")
        counts = np.array([b.size for b in self.borders])
        used = self.split_ordinal != SENTINEL
        if used.any():
            f = self.split_feature[used]
            o = self.split_ordinal[used]
            if f.min() < 0 or f.max() >= self.n_features:
                errors.append("split feature index out of range")
            elif (o < 0).any() or (o >= counts[f]).any():
                errors.append("split border ordinal out of range")
        return errors

    def require_valid(self) -> None:
        errors = self.validate()
        if errors:
            raise ValueError("invalid model: " + "; ".join(errors))

    def subset(self, begin: int, end: int, raw: bool = True) -> "MultiOutputModel":
        """Trees [begin, end); with raw=True scale 1 / bias 0 (partial sums for sharding)."""
        return MultiOutputModel(self.borders, self.split_feature[begin:end], self.split_ordinal[begin:end],
                                self.leaves[begin:end], 1.0 if raw else self.scale, 0.0 if raw else self.bias)


class MultiOutputEvaluator:
    """A multi-output model resident on one GPU (K5 staged kernel, K4 where K5 does not
    apply).  ``config`` selects the precision family as EvalConfig does for one output
    (evaluate.py:106-135): NAIVE / GATHER / PERMUTE64 binary64, NAIVE16 / PERMUTE16
    binary16 (depth <= 10 and <= 10 outputs)."""

    def __init__(self, model: MultiOutputModel, device: Optional[int] = None, config: Optional[EvalConfig] = None):
        model.require_valid()
        self.config = config if config is not None else EvalConfig()
        self.precision = self.config.strategy.precision
        lib = _native.require_gpu()
        import torch

        self.device = torch.cuda.current_device() if device is None else int(device)
        self.model = model
        counts = np.array([b.size for b in model.borders], dtype=np.int32)
        stride = max(1, int(counts.max()))
        borders = np.full((model.n_features, stride), np.inf, dtype=np.float32)
        for f, b in enumerate(model.borders):
            borders[f, : b.size] = b
        so = model.split_ordinal.astype(np.uint8)
        half = self.precision is LeafPrecision.BINARY16
        bank = np.ascontiguousarray(half_bank_values(model.leaves)[0].view(np.uint16)) if half else None
        keep = (counts, borders, model.split_feature, so, model.leaves, bank)
        desc = _native.ModelDesc()
        desc.n_features, desc.n_trees = model.n_features, model.n_trees
        desc.max_depth, desc.n_outputs = model.depth if model.n_trees else 0, model.n_outputs
        desc.border_counts, desc.borders, desc.border_stride = counts.ctypes.data, borders.ctypes.data, stride
        desc.split_feature = model.split_feature.ctypes.data if model.n_trees else None
        desc.split_ordinal = so.ctypes.data if model.n_trees else None
        desc.leaves = model.leaves.ctypes.data if model.n_trees else None
        desc.leaves_f16 = bank.ctypes.data if half and model.n_trees else None
        desc.scale, desc.bias = model.scale, model.bias
        desc.precision = _native.PRECISION_BINARY16 if half else _native.PRECISION_BINARY64
        handle = ctypes.c_void_p()
        _native.check(lib.obt_model_create(ctypes.byref(desc), self.device, ctypes.byref(handle)))
        del keep
        self._lib, self.handle = lib, handle

    def quantize_kernel(self) -> tuple[str, int]:
        """("cells", compares) or ("eytzinger", levels): the predict path's quantize search."""
        kind, param = ctypes.c_int32(), ctypes.c_int32()
        _native.check(self._lib.obt_model_quantize_kernel(self.handle, ctypes.byref(kind), ctypes.byref(param)))
        return ({1: "cells", 2: "cells1024", 3: "cells512"}.get(kind.value, "eytzinger"), param.value)

    def apply_kernel(self) -> str:
        """The multi-output apply kernel this model runs: "staged" (K5) or "gather" (K4)."""
        kind = ctypes.c_int32()
        _native.check(self._lib.obt_model_multi_kernel(self.handle, ctypes.byref(kind)))
        return {2: "staged", 0: "gather"}.get(kind.value, "none")

    def predict_device(self, x, layout: Layout = Layout.OBJECT_MAJOR, out=None, workspace=None):
        """float32 CUDA tensor [n][F] (or [F][n]) -> float64 CUDA tensor [n][C]."""
        x, n, out, ws_ptr, ws_bytes = _checks.device_inputs(x, layout, self.model.n_features, self.device,
                                                             self.model.n_outputs, out, workspace)
        if n:
            _native.check(self._lib.obt_predict_dev(self.handle, x.data_ptr(), n, layout_code(layout), out.data_ptr(),
                                                    ws_ptr, ws_bytes, _native.current_stream_handle(x.device)))
        return out

    def predict_device_marked(self, x, events, layout: Layout = Layout.OBJECT_MAJOR, out=None, workspace=None):
        """predict_device recording three _native.Event's around the two kernels."""
        x, n, out, ws_ptr, ws_bytes = _checks.device_inputs(x, layout, self.model.n_features, self.device,
                                                             self.model.n_outputs, out, workspace)
        if n == 0:
            return out
        ev = [e.handle if e is not None else None for e in events]
        _native.check(self._lib.obt_predict_dev_marked(self.handle, x.data_ptr(), n, layout_code(layout), out.data_ptr(),
                                                       ws_ptr, ws_bytes, _native.current_stream_handle(x.device), *ev))
        return out

    def workspace_bytes(self, n_objects: int) -> int:
        size = ctypes.c_size_t()
        _native.check(self._lib.obt_workspace_size(self.handle, int(n_objects), ctypes.byref(size)))
        return size.value

    def last_launch_count(self) -> int:
        return int(self._lib.obt_last_launch_count())

    @property
    def leaf_storage(self) -> str:
        info = [ctypes.c_int32() for _ in range(7)]
        _native.check(self._lib.obt_model_info(self.handle, *[ctypes.byref(v) for v in info]))
        return _native.LEAF_STORAGE_NAMES[info[5].value]

    def predict(self, matrix: FeatureMatrix, out: Optional[np.ndarray] = None) -> np.ndarray:
        if not isinstance(matrix, FeatureMatrix):
            return self.predict_device(matrix)
        _checks.check_features(matrix.n_features, self.model.n_features)
        out = _checks.host_out(out, matrix.n_objects, self.model.n_outputs)
        if matrix.n_objects:
            import torch

            with torch.cuda.device(self.device):
                _native.check(self._lib.obt_predict_host(self.handle, matrix.values.ctypes.data, matrix.n_objects,
                                                         layout_code(matrix.layout), out.ctypes.data,
                                                         _native.current_stream_handle(self.device)))
        return out

    def close(self):
        if self.handle.value:
            self._lib.obt_model_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def from_arrays(arrays: dict) -> MultiOutputModel:
    """From synthetic.model_arrays(...) output."""
    return MultiOutputModel(arrays["borders"], arrays["split_feature"], arrays["split_ordinal"], arrays["leaves"],
                            arrays["scale"], arrays["bias"])
