"""The drop-in evaluator: reference names, B200 kernels underneath.

``ModelTables``, ``Evaluator`` and ``evaluate`` keep the reference signatures and
error behaviour (pkg/src/obtree/evaluate.py:138-166, 251-307).  ``Evaluator.predict``
takes the reference's host ``FeatureMatrix`` and returns a float64 ndarray in input
order; ``predict_device`` is the HBM-resident path (torch CUDA tensors in and out,
asynchronous on the current stream).  Both go through the C ABI
(include/obtree_b200.h); nothing here computes a prediction on the CPU.
"""

from __future__ import annotations

import ctypes
import threading
from typing import Optional

import numpy as np

from . import _checks, _native
from .config import EvalConfig
from .matrix import FeatureMatrix, Layout, layout_code
from .model import LeafBank, LeafPrecision, ObliviousModel, build_leaf_bank, half_bank_values, require_valid

SENTINEL_ORDINAL = 255  # reference evaluate.py:32: never true, quantiles are <= 254


def _ptr(arr: np.ndarray) -> int:
    return int(arr.ctypes.data) if arr is not None and arr.size else 0


class DeviceModel:
    """An ``obt_model`` handle: the model's tables resident on one GPU."""

    def __init__(self, tables: "ModelTables", precision: LeafPrecision, device: int):
        lib = _native.require_gpu()
        packed = tables.packed()
        desc = _native.ModelDesc()
        desc.n_features = tables.n_features
        desc.n_trees = tables.n_trees
        desc.max_depth = tables.max_depth
        desc.n_outputs = 1
        desc.border_counts = _ptr(packed["border_counts"])
        desc.borders = _ptr(packed["borders"])
        desc.border_stride = packed["borders"].shape[1]
        desc.split_feature = _ptr(packed["split_feature"])
        desc.split_ordinal = _ptr(packed["split_ordinal"])
        desc.leaves = _ptr(packed["leaves"])
        half = precision is LeafPrecision.BINARY16
        desc.leaves_f16 = _ptr(packed["leaves_f16"]) if half else 0
        desc.scale = tables.model.scale
        desc.bias = tables.model.bias
        desc.precision = _native.PRECISION_BINARY16 if half else _native.PRECISION_BINARY64
        handle = ctypes.c_void_p()
        _native.check(lib.obt_model_create(ctypes.byref(desc), int(device), ctypes.byref(handle)))
        self._lib = lib
        self.handle = handle
        self.device = int(device)
        self.precision = precision
        info = [ctypes.c_int32() for _ in range(7)]
        _native.check(lib.obt_model_info(handle, *[ctypes.byref(v) for v in info]))
        self.leaf_storage = _native.LEAF_STORAGE_NAMES[info[5].value]
        self.compare_mode = info[6].value

    def quantize_kernel(self) -> tuple[str, int]:
        """The predict path's quantize search for TMA-eligible inputs: ("cells", compares
        per value) for the cell-table kernel, ("eytzinger", levels) otherwise."""
        kind, param = ctypes.c_int32(), ctypes.c_int32()
        _native.check(self._lib.obt_model_quantize_kernel(self.handle, ctypes.byref(kind), ctypes.byref(param)))
        return ({1: "cells", 2: "cells1024", 3: "cells512"}.get(kind.value, "eytzinger"), param.value)

    def close(self) -> None:
        if getattr(self, "handle", None) and self.handle.value:
            self._lib.obt_model_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ModelTables:
    """Derived arrays shared by every evaluation of one model (reference evaluate.py:138-166).

    ``split_feature`` int32 [T][Dmax] / ``split_ordinal`` uint8 [T][Dmax] with the 255
    sentinel padding shallow trees; leaf banks per precision built on first use; the
    device-resident copy per (precision, device) uploaded on first use."""

    def __init__(self, model: ObliviousModel):
        require_valid(model)
        self.model = model
        self.borders = [ff.borders for ff in model.float_features]
        self.n_trees = model.n_trees
        self.n_features = model.n_features
        self.max_depth = max((t.depth for t in model.trees), default=0)
        shape = (self.n_trees, self.max_depth)
        self.split_feature = np.zeros(shape, dtype=np.int32)
        self.split_ordinal = np.full(shape, SENTINEL_ORDINAL, dtype=np.uint8)
        for t, tree in enumerate(model.trees):
            for d, split in enumerate(tree.splits):
                self.split_feature[t, d] = split.feature_index
                self.split_ordinal[t, d] = split.border_ordinal
        self._banks: dict = {}
        self._packed: Optional[dict] = None
        self._device: dict = {}
        self._lock = threading.Lock()

    def bank(self, precision: LeafPrecision) -> LeafBank:
        with self._lock:
            if precision not in self._banks:
                self._banks[precision] = build_leaf_bank(self.model, precision)
            return self._banks[precision]

    def packed(self) -> dict:
        """Flat host arrays in the C ABI's obt_model_desc layout."""
        if self._packed is None:
            F, T, D = self.n_features, self.n_trees, self.max_depth
            counts = np.array([b.size for b in self.borders], dtype=np.int32)
            stride = max(1, int(counts.max()) if counts.size else 1)
            borders = np.full((F, stride), np.inf, dtype=np.float32)
            for f, b in enumerate(self.borders):
                borders[f, : b.size] = b
            width = 1 << D if T else 1
            leaves = np.zeros((T, width), dtype=np.float64)
            for t, tree in enumerate(self.model.trees):
                leaves[t, : tree.leaf_values.size] = tree.leaf_values
            halves, _ = half_bank_values(leaves)
            self._packed = {
                "border_counts": counts,
                "borders": borders,
                "split_feature": np.ascontiguousarray(self.split_feature),
                "split_ordinal": np.ascontiguousarray(self.split_ordinal),
                "leaves": leaves,
                "leaves_f16": np.ascontiguousarray(halves.view(np.uint16)),
            }
        return self._packed

    def device_model(self, precision: LeafPrecision, device: int) -> DeviceModel:
        key = (precision, int(device))
        with self._lock:
            if key not in self._device:
                self._device[key] = DeviceModel(self, precision, device)
            return self._device[key]


def _check_features(matrix_features: int, model: ObliviousModel) -> None:
    _checks.check_features(matrix_features, model.n_features)


class Evaluator:
    """A model prepared for repeated evaluation under one configuration, on one GPU."""

    def __init__(self, model, config: Optional[EvalConfig] = None, device: Optional[int] = None):
        self.tables = model if isinstance(model, ModelTables) else ModelTables(model)
        self.config = config or EvalConfig()
        self.config.validate()
        self.precision = self.config.strategy.precision
        if device is None:
            import torch

            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = int(device)
        self._dev = self.tables.device_model(self.precision, self.device)

    def quantize_kernel(self) -> tuple[str, int]:
        """("cells", compares) or ("eytzinger", levels): the predict path's quantize search."""
        return self._dev.quantize_kernel()

    @property
    def model(self) -> ObliviousModel:
        return self.tables.model

    @property
    def bank(self) -> LeafBank:
        return self.tables.bank(self.precision)

    @property
    def leaf_storage(self) -> str:
        return self._dev.leaf_storage

    def predict(self, matrix, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Raw scores for every object, in input order (reference evaluate.py:268-300).

        A ``FeatureMatrix`` (host memory) returns a float64 ndarray (written into
        ``out`` when given, e.g. a pinned buffer); a CUDA tensor is routed to
        ``predict_device`` and returns a CUDA float64 tensor."""
        if not isinstance(matrix, FeatureMatrix):
            return self.predict_device(matrix)
        _check_features(matrix.n_features, self.model)
        n = matrix.n_objects
        out = _checks.host_out(out, n, 1)
        if n == 0:
            return out
        import torch

        lib = self._dev._lib
        with torch.cuda.device(self.device):
            stream = _native.current_stream_handle(self.device)
            _native.check(
                lib.obt_predict_host(
                    self._dev.handle, _ptr(matrix.values), n, layout_code(matrix.layout), _ptr(out), stream
                )
            )
        return out

    def predict_device(self, x, layout: Layout = Layout.OBJECT_MAJOR, out=None, workspace=None):
        """HBM-resident predict: ``x`` float32 CUDA tensor [n][F] (object-major) or
        [F][n] (feature-major) -> float64 CUDA tensor [n]; asynchronous on the
        current stream.  ``workspace`` (uint8 CUDA tensor) avoids pool allocation."""
        x, n, out, ws_ptr, ws_bytes = _checks.device_inputs(x, layout, self.model.n_features, self.device, 1, out,
                                                             workspace)
        if n == 0:
            return out
        lib = self._dev._lib
        stream = _native.current_stream_handle(x.device)
        _native.check(
            lib.obt_predict_dev(
                self._dev.handle, x.data_ptr(), n, layout_code(layout), out.data_ptr(), ws_ptr, ws_bytes, stream
            )
        )
        return out

    def predict_device_marked(self, x, events, layout: Layout = Layout.OBJECT_MAJOR, out=None, workspace=None):
        """``predict_device`` recording three ``_native.Event``s around the two kernels."""
        x, n, out, ws_ptr, ws_bytes = _checks.device_inputs(x, layout, self.model.n_features, self.device, 1, out,
                                                             workspace)
        if n == 0:
            return out
        stream = _native.current_stream_handle(x.device)
        ev = [e.handle if e is not None else None for e in events]
        _native.check(
            self._dev._lib.obt_predict_dev_marked(
                self._dev.handle, x.data_ptr(), n, layout_code(layout), out.data_ptr(), ws_ptr, ws_bytes, stream, *ev
            )
        )
        return out

    def last_launch_count(self) -> int:
        return int(self._dev._lib.obt_last_launch_count())

    def workspace_bytes(self, n_objects: int) -> int:
        size = ctypes.c_size_t()
        _native.check(self._dev._lib.obt_workspace_size(self._dev.handle, int(n_objects), ctypes.byref(size)))
        return size.value


def evaluate(model: ObliviousModel, matrix: FeatureMatrix, config: Optional[EvalConfig] = None) -> np.ndarray:
    """One-shot evaluation (reference evaluate.py:303-307)."""
    return Evaluator(model, config).predict(matrix)
