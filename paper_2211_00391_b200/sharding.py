"""Multi-GPU partitioning of the apply path: one process per GPU (torch.distributed).

Object sharding (BASELINE configs 1-4): every prediction depends only on its own
feature row (reference oracle.py:42-51), so rank r evaluates objects
[begin_r, end_r) of the batch on its own GPU with a replicated model and there is
no collective on the data path.  ``gather=True`` assembles the full score vector on
every rank afterwards (one tensor all_gather outside the compute path).

Tree sharding (BASELINE config 5): rank r owns trees [t_r, t_{r+1}) and evaluates
every object against them with scale 1 and bias 0, producing per-object binary64
partial sums; one all_reduce(SUM) over NCCL combines them and the affine finalize
runs on the reduced sums (two roundings, as evaluate.py:298-299).  Summing per-rank
partials reassociates the reference's tree-order fold.  For the binary64 family
(binary64 partials) results agree with the oracle to ~1e-16 relative of the partial
magnitudes rather than bit for bit.  For the binary16 family (NAIVE16/PERMUTE16) each
rank folds its trees in binary32, so the error is that of binary32 partial sums,
~1e-7 relative of the partial magnitudes (the reference's single binary32 fold has
errors of the same order, but not the same ones).

Grid sharding (config 5 comparison): G_o x G_t ranks; rank
r = o * G_t + t evaluates object shard o against tree shard t and the G_t ranks of
object shard o all_reduce their partials (one process group per object shard).
G_t = 1 is object sharding, G_o = 1 tree sharding.

``LocalShardedEvaluator`` is the one-process form of object and tree sharding: one
model handle per device of this process behind the C ABI's ``obt_predict_sharded`` (host
threads per object shard; peer copies of the tree shards' partial sums to the first
device, added there in shard order).  It needs no process group.

Every distributed class has a host path (``predict(FeatureMatrix)``, the reference's call) and a
device path (``predict_device(cuda tensor)``) whose collectives run on the tensors in
HBM (NCCL) or, for gloo test runs, through host copies.
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
        self._ev, self.device = None, device
        if local_predict is None:
            if hasattr(model, "subset"):  # a multi-output model (config 5): [n][C] scores per shard
                from .multiclass import MultiOutputEvaluator

                ev = MultiOutputEvaluator(model, device=device, config=config)
            else:
                from .evaluate import Evaluator

                ev = Evaluator(model, config, device=device)
            local_predict = lambda m, x: ev.predict(x)  # noqa: E731
            self._ev, self.device = ev, ev.device
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

        return _gather_rows(torch.from_numpy(np.ascontiguousarray(local)), matrix.n_objects, self.world,
                            self._gather_device).numpy()

    @property
    def _gather_device(self):
        dist = _dist()
        return f"cuda:{self.device}" if dist.get_backend() == "nccl" and self.device is not None else "cpu"

    def predict_device(self, x_local, layout: Layout = Layout.OBJECT_MAJOR, out=None, workspace=None):
        """This rank's shard, already resident on its GPU -> its scores (no collective)."""
        if self._ev is None:
            raise RuntimeError("predict_device needs the GPU evaluator (no local_predict injection)")
        return self._ev.predict_device(x_local, layout, out=out, workspace=workspace)


def _gather_rows(local, n_total: int, world: int, device):
    """Concatenate every rank's rows (ranks hold object_shard ranges, in rank order) with
    one tensor all_gather; shards are padded to the largest one."""
    import torch

    dist = _dist()
    sizes = [e - b for b, e in (object_shard(n_total, r, world) for r in range(world))]
    width = max(sizes) if sizes else 0
    tail = tuple(local.shape[1:])
    buf = torch.zeros((width,) + tail, dtype=torch.float64, device=device)
    buf[: local.shape[0]].copy_(local)
    pieces = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(pieces, buf)
    return torch.cat([p[:k] for p, k in zip(pieces, sizes)]).cpu()


def _all_reduce_sum(t, group=None):
    """In-place SUM all_reduce of a float64 tensor: on the tensor's GPU under NCCL, through
    a host copy under gloo (functional test runs)."""
    dist = _dist()
    if t.is_cuda and dist.get_backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def _finalize_(sums, scale: float, bias: float):
    # sum * scale + bias with two roundings (evaluate.py:298-299): two separate kernels
    return sums.mul_(scale).add_(bias)


class TreeShardedEvaluator:
    """Model-parallel predict: this rank's trees over every object, partial binary64 sums
    all-reduced (sum) across ranks, then scale/bias.

    ``local_predict(submodel, matrix) -> np.ndarray`` returns the raw partial sums of a
    scale-1 bias-0 sub-model; it defaults to a GPU ``Evaluator``.  ``reduce_device`` chooses
    where the all_reduce runs (a CUDA device for NCCL, "cpu" for gloo)."""

    def __init__(self, model: ObliviousModel, config: Optional[EvalConfig] = None,
                 local_predict: Optional[Callable] = None, device: Optional[int] = None, reduce_device=None,
                 tree_groups: Optional[int] = None, tree_group_index: Optional[int] = None, group=None):
        dist = _dist()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.model = model
        self.group = group
        n_groups = self.world if tree_groups is None else tree_groups
        index = self.rank if tree_group_index is None else tree_group_index
        b, e = tree_shard(model.n_trees, index, n_groups)
        self.tree_range = (b, e)
        self.submodel = tree_submodel(model, b, e)
        self._ev = None
        if local_predict is None:
            if hasattr(self.submodel, "subset"):
                from .multiclass import MultiOutputEvaluator

                ev = MultiOutputEvaluator(self.submodel, device=device, config=config)
            else:
                from .evaluate import Evaluator

                ev = Evaluator(self.submodel, config, device=device)
            local_predict = lambda m, x: ev.predict(x)  # noqa: E731
            self._ev = ev
            if reduce_device is None:
                reduce_device = f"cuda:{ev.device}" if dist.get_backend(group) == "nccl" else "cpu"
        self._predict = local_predict
        self.reduce_device = reduce_device or "cpu"

    @property
    def local_evaluator(self):
        """The GPU evaluator of this rank's tree shard (None under local_predict injection)."""
        return self._ev

    def predict(self, matrix: FeatureMatrix) -> np.ndarray:
        import torch

        partial = np.asarray(self._predict(self.submodel, matrix), dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(partial)).to(self.reduce_device)
        _all_reduce_sum(t, self.group)
        return _finalize_(t, self.model.scale, self.model.bias).cpu().numpy()

    def predict_device(self, x, layout: Layout = Layout.OBJECT_MAJOR, out=None, workspace=None):
        """Partial sums of this rank's trees in HBM, all_reduced in place (NCCL over
        NVLink), then the affine finalize on the device; returns the finished scores."""
        if self._ev is None:
            raise RuntimeError("predict_device needs the GPU evaluator (no local_predict injection)")
        out = self._ev.predict_device(x, layout, out=out, workspace=workspace)
        _all_reduce_sum(out, self.group)
        return _finalize_(out, self.model.scale, self.model.bias)


def grid_groups(object_groups: int, tree_groups: int):
    """One process group per object shard: ranks o * tree_groups + t, t < tree_groups.
    Every rank must call this (new_group is collective), in the same order."""
    dist = _dist()
    if object_groups * tree_groups != dist.get_world_size():
        raise ValueError(f"grid {object_groups} x {tree_groups} does not match world size {dist.get_world_size()}")
    groups = [dist.new_group(list(range(o * tree_groups, (o + 1) * tree_groups))) for o in range(object_groups)]
    return groups


class GridShardedEvaluator:
    """2-D sharding, object shards x tree shards: rank
    r = o * G_t + t evaluates object shard o of the batch against tree shard t; the G_t
    ranks of an object shard all_reduce their binary64 partials and finalize.
    ``predict`` returns this rank's object shard of the finished scores (``gather=True``:
    the whole batch, in object order)."""

    def __init__(self, model, object_groups: int, tree_groups: int, config: Optional[EvalConfig] = None,
                 local_predict: Optional[Callable] = None, device: Optional[int] = None, reduce_device=None):
        dist = _dist()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.object_groups, self.tree_groups = object_groups, tree_groups
        groups = grid_groups(object_groups, tree_groups)
        self.object_index, self.tree_index = divmod(self.rank, tree_groups)
        self.model = model
        self._trees = TreeShardedEvaluator(model, config, local_predict, device, reduce_device,
                                           tree_groups=tree_groups, tree_group_index=self.tree_index,
                                           group=groups[self.object_index])
        self.tree_range = self._trees.tree_range

    @property
    def trees(self) -> TreeShardedEvaluator:
        """This rank's tree-shard evaluator (reduce group = its object shard's ranks)."""
        return self._trees

    def object_range(self, n: int) -> tuple:
        return balanced_ranges(n, self.object_groups, quantum=256)[self.object_index]

    def predict(self, matrix: FeatureMatrix, gather: bool = True) -> np.ndarray:
        import torch

        b, e = self.object_range(matrix.n_objects)
        local = self._trees.predict(_rows(matrix, b, e))
        if not gather:
            return local
        # one representative per object shard (tree index 0) contributes rows; the others
        # contribute empty slots, so a world-wide gather assembles the batch in order
        dist = _dist()
        sizes = [e2 - b2 for b2, e2 in balanced_ranges(matrix.n_objects, self.object_groups, quantum=256)]
        width = max(sizes) if sizes else 0
        tail = tuple(local.shape[1:])
        buf = torch.zeros((width,) + tail, dtype=torch.float64)
        buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local))
        dev = self._trees.reduce_device
        buf = buf.to(dev)
        pieces = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(pieces, buf)
        rows = [pieces[o * self.tree_groups][: sizes[o]] for o in range(self.object_groups)]
        return torch.cat(rows).cpu().numpy()

    def predict_device(self, x_local, layout: Layout = Layout.OBJECT_MAJOR, out=None, workspace=None):
        """This rank's object shard (resident on its GPU) against its tree shard, reduced
        within the object shard's group and finalized: the shard's finished scores."""
        return self._trees.predict_device(x_local, layout, out=out, workspace=workspace)


class LocalShardedEvaluator:
    """One process, several GPUs, through ``obt_predict_sharded`` (include/obtree_b200.h).

    ``mode="objects"``: the whole model on every device of ``devices``; a predict splits
    the batch into contiguous object ranges (256-object quanta), one host thread and one
    host->device pipeline per device, bit-identical to a single device.
    ``mode="trees"``: device i holds trees ``tree_shard(T, i, len(devices))`` as a raw
    partial-sum model; partial sums are peer-copied to ``devices[0]``, added in shard order
    and finalized there (reassociates the fold, as ``TreeShardedEvaluator``).
    ``devices`` may repeat a device (functional tests on a one-GPU box)."""

    def __init__(self, model, devices, mode: str = "objects", config: Optional[EvalConfig] = None):
        if mode not in ("objects", "trees"):
            raise ValueError(f"unknown shard mode {mode!r}")
        devices = [int(d) for d in devices]
        if not 1 <= len(devices) <= 16:
            raise ValueError("devices must name 1..16 GPUs")
        self.model, self.mode, self.devices = model, mode, devices
        multi = hasattr(model, "subset")
        self.n_outputs = model.n_outputs if multi else 1

        def make(sub, device):
            if multi:
                from .multiclass import MultiOutputEvaluator

                return MultiOutputEvaluator(sub, device=device, config=config)
            from .evaluate import Evaluator

            return Evaluator(sub, config, device=device)

        if mode == "objects":
            self.tree_ranges = [(0, model.n_trees)] * len(devices)
            self._evs = [make(model, d) for d in devices]
        else:
            self.tree_ranges = [tree_shard(model.n_trees, i, len(devices)) for i in range(len(devices))]
            self._evs = [make(tree_submodel(model, b, e), d) for (b, e), d in zip(self.tree_ranges, devices)]
        handles = [ev.handle if multi else ev._dev.handle for ev in self._evs]
        import ctypes

        self._handles = (ctypes.c_void_p * len(handles))(*[h.value for h in handles])

    def predict(self, matrix: FeatureMatrix, out: Optional[np.ndarray] = None) -> np.ndarray:
        from . import _checks, _native
        from .matrix import layout_code

        _checks.check_features(matrix.n_features, self.model.n_features)
        out = _checks.host_out(out, matrix.n_objects, self.n_outputs)
        if matrix.n_objects:
            lib = _native.require_gpu()
            code = _native.SHARD_OBJECTS if self.mode == "objects" else _native.SHARD_TREES
            _native.check(lib.obt_predict_sharded(self._handles, len(self.devices), code, matrix.values.ctypes.data,
                                                  matrix.n_objects, layout_code(matrix.layout),
                                                  float(self.model.scale), float(self.model.bias), out.ctypes.data))
        return out
