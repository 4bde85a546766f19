"""Evaluation configuration, kept call-compatible with the reference.

``EvalConfig`` / ``LeafStrategy`` / ``TailPolicy`` / ``BLOCK_SIZES`` follow the
reference (pkg/src/obtree/evaluate.py:27-135, accumulate.py:34-60) including the
validation errors.  On the GPU only the strategy's *precision family* changes
arithmetic (binary64 leaves + binary64 fold, or binary16 leaves + binary32 fold);
block size, vector width and tail policy are CPU cache/lane mechanics whose
results the reference proves invariant (tests/test_evaluate.py:172-213), so they
are validated and otherwise ignored.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

from .matrix import VectorWidth
from .model import LeafPrecision

BLOCK_SIZES = (64, 128, 256, 512)


class LeafStrategy(Enum):
    NAIVE = "naive"
    GATHER = "gather"
    PERMUTE64 = "permute64"
    PERMUTE16 = "permute16"
    NAIVE16 = "naive16"

    @property
    def precision(self) -> LeafPrecision:
        half = (LeafStrategy.PERMUTE16, LeafStrategy.NAIVE16)
        return LeafPrecision.BINARY16 if self in half else LeafPrecision.BINARY64

    def allows_width(self, width: VectorWidth) -> bool:
        if self is LeafStrategy.GATHER:
            return width in (VectorWidth.W256, VectorWidth.W512)
        if self in (LeafStrategy.PERMUTE64, LeafStrategy.PERMUTE16):
            return width is VectorWidth.W512
        return True

    def object_group(self, width: VectorWidth) -> int:
        if self is LeafStrategy.PERMUTE64:
            return 8
        if self is LeafStrategy.PERMUTE16:
            return 32
        return width.byte_lanes


class TailPolicy(Enum):
    SCALAR_TAIL = "scalar"
    PADDED_GROUP = "padded"


@dataclass(frozen=True)
class EvalConfig:
    block_size: int = 128
    width: VectorWidth = field(default_factory=VectorWidth.widest_supported)
    strategy: LeafStrategy = LeafStrategy.NAIVE
    tail_policy: TailPolicy = TailPolicy.SCALAR_TAIL

    @property
    def object_group(self) -> int:
        return self.strategy.object_group(self.width)

    def validate(self) -> None:
        if self.block_size not in BLOCK_SIZES:
            raise ValueError(f"block size must be one of {BLOCK_SIZES}")
        if not self.width.is_supported():
            raise ValueError(f"vector width {self.width.value} not supported on this host")
        if not self.strategy.allows_width(self.width):
            raise ValueError(
                f"strategy {self.strategy.value} is incompatible with width {self.width.value}"
            )
        if self.block_size < self.object_group:
            raise ValueError(
                f"block size {self.block_size} below the object group of {self.object_group}"
            )

    def describe(self) -> str:
        return f"{self.strategy.value}-{self.width.value}-b{self.block_size}-{self.tail_policy.value}"
