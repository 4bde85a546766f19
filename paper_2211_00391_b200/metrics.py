"""FP16-trade-off reporting: the paper's Table 9.2 deviation metrics and class flips.

Same definitions as the reference (pkg/src/obtree/oracle.py:57-92): absolute
deviations, median = lower middle element, RMS over all objects; a flip is a sign
change of (score - threshold).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class DeviationMetrics:
    max_abs: float
    mean_abs: float
    median_abs: float
    rms: float


def deviation_metrics(a, b) -> DeviationMetrics:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError("prediction vectors must be 1-D and the same length")
    if a.size == 0:
        raise ValueError("prediction vectors must not be empty")
    dev = np.abs(a - b)
    ranked = np.sort(dev)
    return DeviationMetrics(
        max_abs=float(ranked[-1]),
        mean_abs=float(dev.mean()),
        median_abs=float(ranked[(dev.size - 1) // 2]),
        rms=float(math.sqrt(float(np.mean(dev * dev)))),
    )


def classification_flip_count(a, b, threshold: float) -> int:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("prediction vectors must be the same length")
    return int(np.count_nonzero(np.sign(a - threshold) != np.sign(b - threshold)))
