"""CPU oracle for the oblivious-ensemble apply path -- TEST INFRASTRUCTURE ONLY.

Restates the reference package (pkg/src/obtree, pure Python + numpy) in plain C
(obtree_oracle.c, built by oracle/Makefile into oracle/_build/liborc.so) plus a few
numpy restatements for cross-checks.  Parity of the restatement is pinned by the
fixtures under tests/golden, which were produced by running the reference itself
(tests/golden/make_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
``--impl reference``) may import this package, and only as the checker / the CPU
baseline.  The product package paper_2211_00391_b200 never imports it.
"""

from __future__ import annotations

import ctypes
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liborc.so"

OBJECT_MAJOR = 0
FEATURE_MAJOR = 1
BINARY64 = 0
BINARY16 = 1
SENTINEL = 255

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.orc_quantize_value.restype = i32
        L.orc_quantize_value.argtypes = [ctypes.c_float, vp, i32]
        L.orc_quantize_matrix.restype = None
        L.orc_quantize_matrix.argtypes = [vp, i64, i32, ctypes.c_int, vp, vp, i32, vp]
        L.orc_leaf_indices.restype = None
        L.orc_leaf_indices.argtypes = [vp, i64, i32, i32, vp, vp, vp]
        L.orc_evaluate_scalar.restype = ctypes.c_int
        L.orc_evaluate_scalar.argtypes = [vp, i64, i32, ctypes.c_int, vp, i32, i32, i32, vp, vp, vp, vp, i32,
                                          f64, f64, ctypes.c_int, vp]
        L.orc_half_from_double.restype = ctypes.c_uint16
        L.orc_half_from_double.argtypes = [f64]
        L.orc_half_saturated.restype = ctypes.c_uint16
        L.orc_half_saturated.argtypes = [f64]
        L.orc_half_to_float.restype = ctypes.c_float
        L.orc_half_to_float.argtypes = [ctypes.c_uint16]
        L.orc_half_bank.restype = i64
        L.orc_half_bank.argtypes = [vp, i64, vp]
        L.orc_synthetic_model.restype = ctypes.c_int
        L.orc_synthetic_model.argtypes = [i32, i32, i32, i32, ctypes.c_uint64, vp, vp, vp, vp,
                                          ctypes.POINTER(f64), ctypes.POINTER(f64)]
        L.orc_feature_matrix.restype = None
        L.orc_feature_matrix.argtypes = [i64, i32, ctypes.c_uint64, f64, f64, f64, f64, vp]
        L.orc_xoshiro_seed.restype = None
        L.orc_xoshiro_seed.argtypes = [vp, ctypes.c_uint64]
        L.orc_xoshiro_next.restype = ctypes.c_uint64
        L.orc_xoshiro_next.argtypes = [vp]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_set_threads.restype = None
        L.orc_set_threads.argtypes = [i32]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return int(a.ctypes.data) if a.size else 0


@dataclass
class FlatModel:
    """The oracle's model layout (see obtree_oracle.c header)."""

    borders: np.ndarray        # float32 [F][stride], +inf padded
    border_counts: np.ndarray  # int32 [F]
    depths: np.ndarray         # int32 [T]
    split_feature: np.ndarray  # int32 [T][Dmax]
    split_ordinal: np.ndarray  # int32 [T][Dmax]
    leaves: np.ndarray         # float64 [T][C][2^Dmax]
    scale: float
    bias: float

    @property
    def n_features(self) -> int:
        return self.borders.shape[0]

    @property
    def n_trees(self) -> int:
        return self.depths.shape[0]

    @property
    def max_depth(self) -> int:
        return self.split_feature.shape[1] if self.split_feature.ndim == 2 else 0

    @property
    def n_outputs(self) -> int:
        return self.leaves.shape[1] if self.leaves.ndim == 3 else 1


def flatten(model) -> FlatModel:
    """Duck-typed: any object with float_features / trees / scale / bias in the
    reference's shape (reference model.py:93-124, or the product's mirror)."""
    F = len(model.float_features)
    counts = np.array([ff.borders.size for ff in model.float_features], dtype=np.int32)
    stride = max(1, int(counts.max()) if F else 1)
    borders = np.full((F, stride), np.inf, dtype=np.float32)
    for f, ff in enumerate(model.float_features):
        borders[f, : ff.borders.size] = ff.borders
    T = len(model.trees)
    D = max((t.depth for t in model.trees), default=0)
    depths = np.array([t.depth for t in model.trees], dtype=np.int32)
    sf = np.zeros((T, D), dtype=np.int32)
    so = np.full((T, D), SENTINEL, dtype=np.int32)
    leaves = np.zeros((T, 1, 1 << D), dtype=np.float64)
    for t, tree in enumerate(model.trees):
        for d, s in enumerate(tree.splits):
            sf[t, d] = s.feature_index
            so[t, d] = s.border_ordinal
        leaves[t, 0, : tree.leaf_values.size] = tree.leaf_values
    return FlatModel(borders, counts, depths, sf, so, leaves, float(model.scale), float(model.bias))


def evaluate_scalar(fm: FlatModel, x: np.ndarray, layout: int = OBJECT_MAJOR, precision: int = BINARY64) -> np.ndarray:
    """oracle.py:21-54 restated in C (raw compares, tree-order fold, two-rounding finalize).
    Returns [n] for single-output models, else [n][C]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = x.shape[0] if layout == OBJECT_MAJOR else x.shape[1]
    F = x.shape[1] if layout == OBJECT_MAJOR else x.shape[0]
    if F != fm.n_features:
        raise ValueError(f"matrix has {F} features, model expects {fm.n_features}")
    C = fm.n_outputs
    out = np.empty((n, C), dtype=np.float64)
    if n:
        rc = lib().orc_evaluate_scalar(
            _p(x), n, F, layout, _p(fm.borders), fm.borders.shape[1], fm.n_trees, fm.max_depth,
            _p(fm.depths), _p(np.ascontiguousarray(fm.split_feature)), _p(np.ascontiguousarray(fm.split_ordinal)),
            _p(np.ascontiguousarray(fm.leaves)), C, fm.scale, fm.bias, precision, _p(out))
        if rc != 0:
            raise RuntimeError(f"orc_evaluate_scalar failed: {rc}")
    return out[:, 0] if C == 1 else out


def quantize(fm: FlatModel, x: np.ndarray, layout: int = OBJECT_MAJOR) -> np.ndarray:
    """quantize.py:164-172 restated: uint8 [F][n] exhaustive border counts."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = x.shape[0] if layout == OBJECT_MAJOR else x.shape[1]
    out = np.zeros((fm.n_features, n), dtype=np.uint8)
    if n:
        lib().orc_quantize_matrix(_p(x), n, fm.n_features, layout, _p(fm.borders), _p(fm.border_counts),
                                  fm.borders.shape[1], _p(out))
    return out


def leaf_indices(fm: FlatModel, buckets: np.ndarray) -> np.ndarray:
    """indexer.py:39-57 / evaluate.py:199-207 restated: uint16 [T][n]."""
    buckets = np.ascontiguousarray(buckets, dtype=np.uint8)
    n = buckets.shape[1]
    out = np.zeros((fm.n_trees, n), dtype=np.uint16)
    if n and fm.n_trees:
        lib().orc_leaf_indices(_p(buckets), n, fm.n_trees, fm.max_depth,
                               _p(np.ascontiguousarray(fm.split_feature)),
                               _p(np.ascontiguousarray(fm.split_ordinal)), _p(out))
    return out


def quantize_value(value: float, borders) -> int:
    b = np.ascontiguousarray(borders, dtype=np.float32)
    return int(lib().orc_quantize_value(float(value), _p(b), b.size))


def half_bits(x: float) -> int:
    return int(lib().orc_half_from_double(float(x)))


def half_bank(leaves: np.ndarray):
    leaves = np.ascontiguousarray(leaves, dtype=np.float64)
    out = np.zeros(leaves.shape, dtype=np.uint16)
    sat = lib().orc_half_bank(_p(leaves), leaves.size, _p(out))
    return out, int(sat)


# ---------------------------------------------------------------------------
# seeded generators (synthetic.py:28-167 restated)

class Xoshiro:
    def __init__(self, seed: int):
        self._state = (ctypes.c_uint64 * 4)()
        lib().orc_xoshiro_seed(ctypes.addressof(self._state), ctypes.c_uint64(seed & (2**64 - 1)))

    def next_u64(self) -> int:
        return int(lib().orc_xoshiro_next(ctypes.addressof(self._state)))

    def unit(self) -> float:
        return (self.next_u64() >> 11) * 2.0**-53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + self.unit() * (hi - lo)

    def below(self, n: int) -> int:
        return (self.next_u64() * n) >> 64


def synthetic_model(n_features: int, borders_per_feature: int, n_trees: int, depth: int, seed: int) -> FlatModel:
    """generate_synthetic_model (synthetic.py:87-133) restated; flat layout."""
    F, B, T, D = n_features, borders_per_feature, n_trees, depth
    borders = np.zeros((F, B), dtype=np.float32)
    sf = np.zeros((T, D), dtype=np.int32)
    so = np.zeros((T, D), dtype=np.int32)
    leaves = np.zeros((T, 1, 1 << D), dtype=np.float64)
    scale, bias = ctypes.c_double(), ctypes.c_double()
    rc = lib().orc_synthetic_model(F, B, T, D, ctypes.c_uint64(seed), _p(borders), _p(sf), _p(so), _p(leaves),
                                   ctypes.byref(scale), ctypes.byref(bias))
    if rc != 0:
        raise ValueError("synthetic model spec out of range")
    counts = np.full(F, B, dtype=np.int32)
    return FlatModel(borders, counts, np.full(T, D, dtype=np.int32), sf, so, leaves, scale.value, bias.value)


def feature_matrix(n_objects: int, n_features: int, seed: int, lo: float = -0.25, hi: float = 1.25,
                   nan_fraction: float = 0.0, inf_fraction: float = 0.0) -> np.ndarray:
    """generate_feature_matrix (synthetic.py:136-167) restated; object-major [n][F]."""
    out = np.empty((n_objects, n_features), dtype=np.float32)
    if out.size:
        lib().orc_feature_matrix(n_objects, n_features, ctypes.c_uint64(seed), lo, hi, nan_fraction,
                                 inf_fraction, _p(out))
    return out


def to_model(fm: FlatModel, types):
    """Build an ObliviousModel from a flat model using the given types module
    (the product package or any module exposing the reference names)."""
    feats = tuple(
        types.FloatFeatureBorders(f, fm.borders[f, : fm.border_counts[f]].copy()) for f in range(fm.n_features)
    )
    trees = []
    for t in range(fm.n_trees):
        d = int(fm.depths[t])
        splits = tuple(types.SplitCondition(int(fm.split_feature[t, k]), int(fm.split_ordinal[t, k])) for k in range(d))
        trees.append(types.ObliviousTree(depth=d, splits=splits, leaf_values=fm.leaves[t, 0, : 1 << d].copy()))
    return types.ObliviousModel(float_features=feats, trees=tuple(trees), scale=fm.scale, bias=fm.bias)


def model_digest(model) -> str:
    """sha256 over a canonical byte encoding of a model (duck-typed)."""
    import hashlib

    h = hashlib.sha256()
    for ff in model.float_features:
        h.update(np.int64(ff.feature_index).tobytes())
        h.update(np.ascontiguousarray(ff.borders, dtype=np.float32).tobytes())
    for tree in model.trees:
        h.update(np.int64(tree.depth).tobytes())
        for s in tree.splits:
            h.update(np.array([s.feature_index, s.border_ordinal], dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(tree.leaf_values, dtype=np.float64).tobytes())
    h.update(np.float64(model.scale).tobytes())
    h.update(np.float64(model.bias).tobytes())
    return h.hexdigest()


def max_threads() -> int:
    return int(lib().orc_max_threads())


def set_threads(n: int) -> None:
    """OpenMP threads for the oracle's parallel loops (overrides OMP_NUM_THREADS)."""
    lib().orc_set_threads(int(n))


def host_cores() -> int:
    """Cores this process may run on."""
    import os

    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover - non-Linux
        return os.cpu_count() or 1
