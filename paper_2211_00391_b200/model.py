"""Ensemble model types, validation and the binary16 leaf bank.

Mirrors the reference model core (pkg/src/obtree/model.py) name for name so a
user can switch imports:

* ``FloatFeatureBorders`` / ``SplitCondition`` / ``ObliviousTree`` /
  ``ObliviousModel`` -- frozen value types with read-only ndarray payloads
  (reference model.py:39-124);
* ``validate_model`` / ``require_valid`` -- every invariant, with the same
  violation texts (reference model.py:131-184);
* ``build_leaf_bank`` / ``LeafBank`` -- per-tree leaf tables in binary64, or
  binary16 with round-to-nearest-even and +/-65504 saturation (reference
  model.py:195-277).  On the GPU path the binary16 bank bits are what gets
  uploaded, so the device sees exactly the reference's half values.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

MAX_BORDERS = 254  # a quantile must fit one byte with every comparison representable
MAX_DEPTH = 8      # leaf indices fit one byte in the reference engine
HALF_MAX = 65504.0
BANK_TAIL_PAD = 256  # zero elements kept after the last table (reference model.py:26)


class LeafPrecision(Enum):
    BINARY64 = "binary64"
    BINARY16 = "binary16"


def _frozen_array(values, dtype) -> np.ndarray:
    arr = np.array(values, dtype=dtype, copy=True, order="C")
    if arr.ndim != 1:
        arr = arr.reshape(-1)
    arr.flags.writeable = False
    return arr


def _f64_bits(x: float) -> int:
    return int(np.array(x, dtype=np.float64).view(np.uint64))


@dataclass(frozen=True, eq=False)
class FloatFeatureBorders:
    """Strictly ascending binary32 thresholds of one feature (at most 254)."""

    feature_index: int
    borders: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "borders", _frozen_array(self.borders, np.float32))

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, FloatFeatureBorders):
            return NotImplemented
        return self.feature_index == other.feature_index and (
            self.borders.tobytes() == other.borders.tobytes()
        )

    __hash__ = None  # mutable-looking payload; equality is by value


@dataclass(frozen=True)
class SplitCondition:
    """True for an object iff quantile(feature) > border_ordinal,
    i.e. iff value > borders[feature][border_ordinal]."""

    feature_index: int
    border_ordinal: int


@dataclass(frozen=True, eq=False)
class ObliviousTree:
    depth: int
    splits: tuple
    leaf_values: np.ndarray  # binary64, 2**depth entries, bit d of the index = split d

    def __post_init__(self) -> None:
        object.__setattr__(self, "splits", tuple(self.splits))
        object.__setattr__(self, "leaf_values", _frozen_array(self.leaf_values, np.float64))

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, ObliviousTree):
            return NotImplemented
        return (
            self.depth == other.depth
            and self.splits == other.splits
            and self.leaf_values.tobytes() == other.leaf_values.tobytes()
        )

    __hash__ = None


@dataclass(frozen=True, eq=False)
class ObliviousModel:
    """prediction = scale * (sum of one leaf per tree, in tree order) + bias."""

    float_features: tuple
    trees: tuple
    scale: float
    bias: float

    def __post_init__(self) -> None:
        object.__setattr__(self, "float_features", tuple(self.float_features))
        object.__setattr__(self, "trees", tuple(self.trees))
        object.__setattr__(self, "scale", float(self.scale))
        object.__setattr__(self, "bias", float(self.bias))

    @property
    def n_features(self) -> int:
        return len(self.float_features)

    @property
    def n_trees(self) -> int:
        return len(self.trees)

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, ObliviousModel):
            return NotImplemented
        return (
            self.float_features == other.float_features
            and self.trees == other.trees
            and _f64_bits(self.scale) == _f64_bits(other.scale)
            and _f64_bits(self.bias) == _f64_bits(other.bias)
        )

    __hash__ = None


def _feature_errors(position: int, ff: FloatFeatureBorders) -> list:
    where = f"float_features[{position}]"
    out = []
    if ff.feature_index != position:
        out.append(f"{where}: feature index {ff.feature_index} does not match position {position}")
    count = ff.borders.size
    if count > MAX_BORDERS:
        out.append(f"{where}: {count} borders exceed the limit of {MAX_BORDERS}")
    if np.isnan(ff.borders).any():
        out.append(f"{where}: NaN border")
    elif count > 1 and not bool(np.all(np.diff(ff.borders) > 0)):
        out.append(f"{where}: non-ascending borders")
    return out


def _tree_errors(position: int, tree: ObliviousTree, features: tuple) -> list:
    where = f"trees[{position}]"
    if not 1 <= tree.depth <= MAX_DEPTH:
        return [f"{where}: depth {tree.depth} outside 1..{MAX_DEPTH}"]
    out = []
    if len(tree.splits) != tree.depth:
        out.append(f"{where}: {len(tree.splits)} splits for depth {tree.depth}")
    expected = 1 << tree.depth
    if tree.leaf_values.size != expected:
        out.append(f"{where}: {tree.leaf_values.size} leaf values, expected {expected}")
    if np.isnan(tree.leaf_values).any():
        out.append(f"{where}: NaN leaf value")
    for s, split in enumerate(tree.splits):
        swhere = f"{where}.splits[{s}]"
        f = split.feature_index
        if not 0 <= f < len(features):
            out.append(f"{swhere}: feature index {f} out of range")
            continue
        n_borders = features[f].borders.size
        if not 0 <= split.border_ordinal < n_borders:
            out.append(
                f"{swhere}: border ordinal out of range "
                f"({split.border_ordinal} vs {n_borders} borders on feature {f})"
            )
    return out


def validate_model(model: ObliviousModel) -> list:
    """All invariant violations of ``model`` (empty list = valid)."""
    errors = []
    if model.n_features == 0:
        errors.append("model: at least one float feature is required")
    for i, ff in enumerate(model.float_features):
        errors.extend(_feature_errors(i, ff))
    for t, tree in enumerate(model.trees):
        errors.extend(_tree_errors(t, tree, model.float_features))
    return errors


def require_valid(model: ObliviousModel) -> None:
    errors = validate_model(model)
    if errors:
        raise ValueError("invalid model: " + "; ".join(errors))


def aligned_zeros(n: int, dtype, alignment: int = 64) -> np.ndarray:
    """Zero-filled 1-D array whose first element sits on an ``alignment`` boundary."""
    itemsize = np.dtype(dtype).itemsize
    raw = np.zeros(n * itemsize + alignment, dtype=np.uint8)
    skip = (-raw.ctypes.data) % alignment
    return raw[skip : skip + n * itemsize].view(dtype)


def half_bank_values(leaves: np.ndarray):
    """binary64 leaves -> (binary16 values, saturation count): numpy's RNE cast, every
    infinite result -- finite overflow and infinite leaves alike -- clamped to +/-65504
    and counted (reference model.py:262-268 tests isinf on the cast values only)."""
    leaves = np.asarray(leaves, dtype=np.float64)
    with np.errstate(over="ignore"):
        halves = leaves.astype(np.float16)
    overflow = np.isinf(halves)
    if overflow.any():
        halves[overflow] = np.where(leaves[overflow] > 0, np.float16(HALF_MAX), np.float16(-HALF_MAX))
    return halves, int(overflow.sum())


@dataclass(frozen=True, eq=False)
class LeafBank:
    """Flat per-tree leaf tables: tree t owns values[offsets[t] : offsets[t] + padded_lengths[t]].

    Tables start on 64-byte boundaries and are zero padded to whole 64-byte
    groups (8 binary64 or 32 binary16 lanes)."""

    precision: LeafPrecision
    values: np.ndarray
    offsets: np.ndarray
    padded_lengths: np.ndarray
    max_abs_leaf: float
    saturation_count: int

    def table(self, tree_index: int) -> np.ndarray:
        start = int(self.offsets[tree_index])
        return self.values[start : start + int(self.padded_lengths[tree_index])]

    @property
    def n_trees(self) -> int:
        return self.offsets.size


def build_leaf_bank(model: ObliviousModel, precision: LeafPrecision) -> LeafBank:
    require_valid(model)
    wide = precision is LeafPrecision.BINARY64
    lanes = 8 if wide else 32
    dtype = np.float64 if wide else np.float16
    sizes = np.array([t.leaf_values.size for t in model.trees], dtype=np.int64)
    padded = -(-sizes // lanes) * lanes
    offsets = np.concatenate(([0], np.cumsum(padded)[:-1])).astype(np.int64) if sizes.size else sizes
    total = int(padded.sum()) if sizes.size else 0
    values = aligned_zeros(total + BANK_TAIL_PAD, dtype)
    max_abs = 0.0
    saturated = 0
    for t, tree in enumerate(model.trees):
        leaves = tree.leaf_values
        if leaves.size:
            max_abs = max(max_abs, float(np.abs(leaves).max()))
        start = int(offsets[t])
        if wide:
            values[start : start + leaves.size] = leaves
        else:
            halves, sat = half_bank_values(leaves)
            saturated += sat
            values[start : start + leaves.size] = halves
    for arr in (values, offsets, padded):
        arr.flags.writeable = False
    return LeafBank(
        precision=precision,
        values=values,
        offsets=offsets,
        padded_lengths=padded,
        max_abs_leaf=max_abs,
        saturation_count=saturated,
    )
