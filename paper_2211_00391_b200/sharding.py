"""Multi-GPU partitioning of the apply path: one process per GPU (torch.distributed).

Object sharding (BASELINE configs 1-4): every prediction depends only on its own
feature row (reference oracle.py:42-51), so rank r evaluates objects
[begin_r, end_r) of the batch on its own GPU with a replicated model and there is
no collective on the data path.  ``gather=True`` assembles the full score vector on
every rank afterwards (an all_gather outside the compute path).

Tree sharding (BASELINE config 5): rank r owns trees [t_r, t_{r+1}) and evaluates
every object against them with scale 1 and bias 0, producing per-object binary64
partial sums; one all_reduce(SUM) over NCCL combines them and the affine finalize
runs on the reduced sums (two roundings, as evaluate.py:298-299).  Summing per-rank
partials reassociates the reference's tree-order fold, so results agree with the
oracle to ~1e-16 relative of the partial magnitudes rather than bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .config import EvalConfig
from .matrix import FeatureMatrix, Layout
from .model import ObliviousModel


def balanced_ranges(total: int, parts: int, quantum: int = 1) -> list:
    """Contiguous [begin, end) ranges covering 0..total, sizes in multiples of
    ``quantum`` except the last, as even as possible."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    units = -(-total // quantum) if total else 0
    base, extra = divmod(units, parts)
    out, pos = [], 0
    for r in range(parts):
        n_units = base + (1 if r < extra else 0)
        end = min(total, pos + n_units * quantum)
        out.append((pos, end))
        pos = end
    return out


def object_shard(n: int, rank: int, world: int) -> tuple:
    # 256-object quanta keep every shard on whole quantize CTAs
    return balanced_ranges(n, world, quantum=256)[rank]


def tree_shard(n_trees: int, rank: int, world: int) -> tuple:
    return balanced_ranges(n_trees, world, quantum=4)[rank]


def tree_submodel(model, begin: int, end: int):
    """The trees [begin, end) with scale 1 / bias 0: its predictions are raw partial sums.
    Works for ObliviousModel and multiclass.MultiOutputModel."""
    if hasattr(model, "subset"):
        return model.subset(begin, end, raw=True)
    return ObliviousModel(model.float_features, model.trees[begin:end], scale=1.0, bias=0.0)


def _rows(matrix: FeatureMatrix, begin: int, end: int) -> FeatureMatrix:
    if matrix.layout is Layout.OBJECT_MAJOR:
        return FeatureMatrix(matrix.values[begin:end], Layout.OBJECT_MAJOR)
    return FeatureMatrix(np.ascontiguousarray(matrix.values[:, begin:end]), Layout.FEATURE_MAJOR)


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised (one process per GPU)")
    return dist


@dataclass
class ShardPlan:
    rank: int
    world: int
    begin: int
    end: int


class ObjectShardedEvaluator:
    """Data-parallel predict: this rank's object shard on this rank's GPU.

    ``local_predict(model, matrix) -> np.ndarray`` defaults to a GPU ``Evaluator``;
    it is injectable so the partitioning and gather logic is testable on CPU."""

    def __init__(self, model: ObliviousModel, config: Optional[EvalConfig] = None,
                 local_predict: Optional[Callable] = None, device: Optional[int] = None):
        dist = _dist()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.model = model
        if local_predict is None:
            if hasattr(model, "subset"):  # a multi-output model (config 5): [n][C] scores per shard
                from .multiclass import MultiOutputEvaluator

                ev = MultiOutputEvaluator(model, device=device)
            else:
                from .evaluate import Evaluator

                ev = Evaluator(model, config, device=device)
            local_predict = lambda m, x: ev.predict(x)  # noqa: E731
        self._predict = local_predict

    def plan(self, n: int) -> ShardPlan:
        b, e = object_shard(n, self.rank, self.world)
        return ShardPlan(self.rank, self.world, b, e)

    def predict(self, matrix: FeatureMatrix, gather: bool = True) -> np.ndarray:
        plan = self.plan(matrix.n_objects)
        local = np.asarray(self._predict(self.model, _rows(matrix, plan.begin, plan.end)), dtype=np.float64)
        if not gather:
            return local
        import torch

        dist = _dist()
        pieces = [None] * self.world
        dist.all_gather_object(pieces, local)  # assembly only; no collective on the compute path
        return np.concatenate([np.asarray(p, dtype=np.float64) for p in pieces]) if pieces else local


class TreeShardedEvaluator:
    """Model-parallel predict: this rank's trees over every object, partial binary64 sums
    all-reduced (sum) across ranks, then scale/bias.

    ``local_predict(submodel, matrix) -> np.ndarray`` returns the raw partial sums of a
    scale-1 bias-0 sub-model; it defaults to a GPU ``Evaluator``.  ``reduce_device`` chooses
    where the all_reduce runs (a CUDA device for NCCL, "cpu" for gloo)."""

    def __init__(self, model: ObliviousModel, config: Optional[EvalConfig] = None,
                 local_predict: Optional[Callable] = None, device: Optional[int] = None, reduce_device=None):
        dist = _dist()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.model = model
        b, e = tree_shard(model.n_trees, self.rank, self.world)
        self.tree_range = (b, e)
        self.submodel = tree_submodel(model, b, e)
        if local_predict is None:
            if hasattr(self.submodel, "subset"):
                from .multiclass import MultiOutputEvaluator

                ev = MultiOutputEvaluator(self.submodel, device=device)
            else:
                from .evaluate import Evaluator

                ev = Evaluator(self.submodel, config, device=device)
            local_predict = lambda m, x: ev.predict(x)  # noqa: E731
            reduce_device = reduce_device or f"cuda:{ev.device}"
        self._predict = local_predict
        self.reduce_device = reduce_device or "cpu"

    def predict(self, matrix: FeatureMatrix) -> np.ndarray:
        import torch

        dist = _dist()
        partial = np.asarray(self._predict(self.submodel, matrix), dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(partial)).to(self.reduce_device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        sums = t.cpu().numpy()
        return sums * self.model.scale + self.model.bias
