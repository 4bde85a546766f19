"""The N>1 path on CPU: two processes over gloo exercise object sharding (no data-path
collective, results assembled in order) and tree sharding (partial binary64 sums,
all_reduce, affine finalize).  The per-rank compute is the CPU oracle (test-only
injection); on GPUs the same classes call the sm_100a Evaluator and reduce over NCCL."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import sharding


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _flat(model):
    if not hasattr(model, "subset"):
        return oracle.flatten(model)
    return oracle.FlatModel(np.stack(model.borders), np.array([b.size for b in model.borders], np.int32),
                            np.full(model.n_trees, model.depth, np.int32), model.split_feature, model.split_ordinal,
                            model.leaves, model.scale, model.bias)


def _oracle_predict(model, matrix):
    layout = oracle.OBJECT_MAJOR if matrix.layout is obt.Layout.OBJECT_MAJOR else oracle.FEATURE_MAJOR
    return oracle.evaluate_scalar(_flat(model), matrix.values, layout)


def _worker(rank, world, port, case):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fm = oracle.synthetic_model(9, 13, 203, 6, 4242)
        model = oracle.to_model(fm, obt)
        x = oracle.feature_matrix(1301, 9, 77, nan_fraction=0.02, inf_fraction=0.01)
        full = oracle.evaluate_scalar(fm, x)
        if case == "objects":
            ev = sharding.ObjectShardedEvaluator(model, local_predict=_oracle_predict)
            for layout in (obt.Layout.OBJECT_MAJOR, obt.Layout.FEATURE_MAJOR):
                m = obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)
                m = m if layout is obt.Layout.OBJECT_MAJOR else m.transposed()
                got = ev.predict(m)
                assert np.array_equal(got, full), "object sharding must be bit-exact"
                local = ev.predict(m, gather=False)
                b, e = sharding.object_shard(x.shape[0], rank, world)
                assert np.array_equal(local, full[b:e])
        elif case == "objects_multi":
            from paper_2211_00391_b200 import multiclass, synthetic

            spec = synthetic.WorkloadSpec("m", 1, 9, 40, 101, 10, 0.01, n_outputs=10, cfg=5)
            mm = multiclass.from_arrays(synthetic.model_arrays(spec, seed=3, affine=True))
            full_m = oracle.evaluate_scalar(_flat(mm), x)
            ev = sharding.ObjectShardedEvaluator(mm, local_predict=_oracle_predict)
            got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
            assert got.shape == (x.shape[0], 10)
            assert np.array_equal(got, full_m), "object sharding of a multi-output model must be bit-exact"
        elif case == "trees_multi":
            from paper_2211_00391_b200 import multiclass, synthetic

            spec = synthetic.WorkloadSpec("m", 1, 9, 40, 101, 10, 0.01, n_outputs=10, cfg=5)
            mm = multiclass.from_arrays(synthetic.model_arrays(spec, seed=3, affine=True))
            full_m = oracle.evaluate_scalar(_flat(mm), x)
            ev = sharding.TreeShardedEvaluator(mm, local_predict=_oracle_predict, reduce_device="cpu")
            got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
            assert got.shape == full_m.shape == (x.shape[0], 10)
            rel = np.abs(got - full_m) / np.maximum(np.maximum(np.abs(got), np.abs(full_m)), 1e-300)
            assert rel.max() <= 1e-12, rel.max()
        elif case.startswith("grid"):
            from paper_2211_00391_b200 import multiclass, synthetic

            go, gt = (int(v) for v in case.split("_")[1].split("x"))
            spec = synthetic.WorkloadSpec("m", 1, 9, 40, 101, 10, 0.01, n_outputs=10, cfg=5)
            mm = multiclass.from_arrays(synthetic.model_arrays(spec, seed=3, affine=True))
            full_m = oracle.evaluate_scalar(_flat(mm), x)
            ev = sharding.GridShardedEvaluator(mm, go, gt, local_predict=_oracle_predict, reduce_device="cpu")
            assert ev.tree_range == sharding.tree_shard(mm.n_trees, rank % gt, gt)
            got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
            assert got.shape == full_m.shape
            rel = np.abs(got - full_m) / np.maximum(np.maximum(np.abs(got), np.abs(full_m)), 1e-300)
            assert rel.max() <= 1e-12, rel.max()
            if gt == 1:
                assert np.array_equal(got, full_m), "a 1-tree-group grid is object sharding: bit-exact"
            local = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR), gather=False)
            b, e = ev.object_range(x.shape[0])
            assert np.allclose(local, full_m[b:e], rtol=1e-12, atol=0)
        else:
            ev = sharding.TreeShardedEvaluator(model, local_predict=_oracle_predict, reduce_device="cpu")
            got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
            rel = np.abs(got - full) / np.maximum(np.maximum(np.abs(got), np.abs(full)), 1e-300)
            assert rel.max() <= 1e-12, rel.max()
            b, e = ev.tree_range
            assert (b, e) == sharding.tree_shard(model.n_trees, rank, world)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["objects", "objects_multi", "trees", "trees_multi", "grid_1x2", "grid_2x1"])
def test_two_rank_gloo(case):
    mp.spawn(_worker, args=(2, _free_port(), case), nprocs=2, join=True)


def test_four_rank_grid_gloo():
    """2 object shards x 2 tree shards: each object shard reduces within its own group."""
    mp.spawn(_worker, args=(4, _free_port(), "grid_2x2"), nprocs=4, join=True)


def test_balanced_ranges_cover_exactly():
    for total in (0, 1, 255, 256, 257, 10_000, 1_000_000):
        for parts in (1, 2, 3, 8):
            r = sharding.balanced_ranges(total, parts, quantum=256)
            assert r[0][0] == 0 and r[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert all((e - b) % 256 == 0 or e == total for b, e in r)
    assert sharding.tree_shard(4000, 7, 8) == (3500, 4000)
