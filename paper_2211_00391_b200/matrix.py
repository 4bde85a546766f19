"""Feature batches and the configuration enums of the reference engine.

``FeatureMatrix`` / ``Layout`` follow the reference (pkg/src/obtree/quantize.py:25-90):
a C-contiguous binary32 matrix, object-major (element (o, f) at o*F + f) or
feature-major (f*N + o).  ``VectorWidth`` is kept for configuration compatibility
(quantize.py:32-56); on the GPU the lane width is a property of the kernels, so it
never changes a result -- exactly the reference's own width-invariance contract.
"""

from __future__ import annotations

from enum import Enum

import numpy as np


class Layout(Enum):
    OBJECT_MAJOR = "object-major"
    FEATURE_MAJOR = "feature-major"


class VectorWidth(Enum):
    SCALAR = "scalar"
    W128 = "w128"
    W256 = "w256"
    W512 = "w512"

    @property
    def byte_lanes(self) -> int:
        return {"scalar": 1, "w128": 16, "w256": 32, "w512": 64}[self.value]

    def is_supported(self) -> bool:
        return True

    @classmethod
    def widest_supported(cls) -> "VectorWidth":
        return cls.W512


class FeatureMatrix:
    """A batch of binary32 feature values in one contiguous layout."""

    __slots__ = ("layout", "values", "n_objects", "n_features")

    def __init__(self, values, layout: Layout):
        arr = np.ascontiguousarray(values, dtype=np.float32)
        if arr.ndim != 2:
            raise ValueError("feature matrix must be 2-D")
        self.layout = layout
        self.values = arr
        if layout is Layout.OBJECT_MAJOR:
            self.n_objects, self.n_features = arr.shape
        else:
            self.n_features, self.n_objects = arr.shape

    def feature_values(self, feature: int, begin: int, end: int) -> np.ndarray:
        if self.layout is Layout.OBJECT_MAJOR:
            return self.values[begin:end, feature]
        return self.values[feature, begin:end]

    def transposed(self) -> "FeatureMatrix":
        flipped = Layout.FEATURE_MAJOR if self.layout is Layout.OBJECT_MAJOR else Layout.OBJECT_MAJOR
        return FeatureMatrix(np.ascontiguousarray(self.values.T), flipped)


def layout_code(layout: Layout) -> int:
    return 0 if layout is Layout.OBJECT_MAJOR else 1
