"""obt_predict_sharded (one process, several devices) on a 1-GPU box: the handles share
cuda:0, which exercises the object ranges, the per-shard host pipelines and threads, the
peer copies and the shard-order fold -- a functional check, never a measurement."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import _native, multiclass, sharding, synthetic

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _single(n=70_001, trees=301, depth=7, features=24):
    spec = synthetic.WorkloadSpec("t", 1, features, 60, trees, depth, 0.1, cfg=1)
    model = synthetic.build_model(spec, seed=5, affine=True)
    x = synthetic.host_features(synthetic.WorkloadSpec("t", n, features, 1, 1, 1, 0.1, cfg=1), seed=6)
    x = synthetic.sprinkle_specials(x, [ff.borders for ff in model.float_features], seed=7)
    return model, x


def _rel(a, b):
    return (np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)).max()


@pytest.mark.parametrize("n_shards", [1, 2, 3])
@pytest.mark.parametrize("layout", [obt.Layout.OBJECT_MAJOR, obt.Layout.FEATURE_MAJOR])
def test_object_shards_bit_exact(n_shards, layout):
    model, x = _single()
    full = oracle.evaluate_scalar(oracle.flatten(model), x)
    values = x if layout is obt.Layout.OBJECT_MAJOR else np.ascontiguousarray(x.T)
    ev = sharding.LocalShardedEvaluator(model, [0] * n_shards, mode="objects")
    got = ev.predict(obt.FeatureMatrix(values, layout))
    assert np.array_equal(got, full)
    # ragged tails: fewer 256-object quanta than shards, and an empty batch
    small = ev.predict(obt.FeatureMatrix(values[:300] if layout is obt.Layout.OBJECT_MAJOR
                                         else np.ascontiguousarray(values[:, :300]), layout))
    assert np.array_equal(small, full[:300])
    empty = np.empty((0, x.shape[1]), np.float32) if layout is obt.Layout.OBJECT_MAJOR else np.empty((x.shape[1], 0), np.float32)
    assert ev.predict(obt.FeatureMatrix(empty, layout)).shape == (0,)


def test_object_shards_multi_chunk_pipeline():
    """A batch large enough that every shard runs the chunked (double-buffered) host
    pipeline: 3 shards x ~3 chunks of 128 MB of features."""
    spec = synthetic.WorkloadSpec("t", 1, 200, 64, 64, 6, 0.05, cfg=2)
    model = synthetic.build_model(spec, seed=3, affine=True)
    n = 1_300_000
    x = synthetic.host_features(synthetic.WorkloadSpec("t", n, 200, 1, 1, 1, 0.1, cfg=2), seed=4)
    ev = sharding.LocalShardedEvaluator(model, [0, 0, 0], mode="objects")
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    one = obt.Evaluator(model, device=0).predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, one)
    idx = np.r_[0:2048, n - 2048:n, 0:n:997]
    assert np.array_equal(got[idx], oracle.evaluate_scalar(oracle.flatten(model), x[idx]))


@pytest.mark.parametrize("n_shards", [2, 3])
@pytest.mark.parametrize("layout", [obt.Layout.OBJECT_MAJOR, obt.Layout.FEATURE_MAJOR])
@pytest.mark.parametrize("strategy", [obt.LeafStrategy.NAIVE, obt.LeafStrategy.NAIVE16])
def test_tree_shards_match_shard_order_sum(n_shards, layout, strategy):
    model, x = _single(n=9_001)
    cfg = obt.EvalConfig(strategy=strategy)
    values = x if layout is obt.Layout.OBJECT_MAJOR else np.ascontiguousarray(x.T)
    m = obt.FeatureMatrix(values, layout)
    ev = sharding.LocalShardedEvaluator(model, [0] * n_shards, mode="trees", config=cfg)
    got = ev.predict(m)
    # exactly the shard-order binary64 sum of the shards' raw partial sums, then scale/bias
    parts = [obt.Evaluator(sharding.tree_submodel(model, b, e), cfg, device=0).predict(m) for b, e in ev.tree_ranges]
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = acc + p
    assert np.array_equal(got, acc * model.scale + model.bias)
    half = strategy is obt.LeafStrategy.NAIVE16
    full = oracle.evaluate_scalar(oracle.flatten(model), x, precision=oracle.BINARY16 if half else oracle.BINARY64)
    assert _rel(got, full) <= (1e-5 if half else 1e-12)


def test_tree_shards_multi_output_and_chunks():
    """Config-5 style: 10 outputs, tree shards, several object chunks per shard."""
    spec = synthetic.WorkloadSpec("m", 1, 1000, 60, 24, 9, 0.01, n_outputs=10, cfg=5)
    mm = multiclass.from_arrays(synthetic.model_arrays(spec, seed=11, affine=True))
    n = 80_000  # 320 MB of features: 3 chunks
    x = synthetic.host_features(synthetic.WorkloadSpec("m", n, 1000, 1, 1, 1, 0.1, cfg=5), seed=12)
    ev = sharding.LocalShardedEvaluator(mm, [0, 0], mode="trees")
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert got.shape == (n, 10)
    idx = np.r_[0:1024, n - 1024:n, 0:n:401]
    counts = np.array([b.size for b in mm.borders], np.int32)
    borders = np.full((mm.n_features, int(counts.max())), np.inf, np.float32)
    for f, b in enumerate(mm.borders):
        borders[f, : b.size] = b
    flat = oracle.FlatModel(borders, counts, np.full(mm.n_trees, mm.depth, np.int32), mm.split_feature,
                            mm.split_ordinal, mm.leaves, mm.scale, mm.bias)
    assert _rel(got[idx], oracle.evaluate_scalar(flat, x[idx])) <= 1e-12
    # object shards of the same multi-output model are bit-exact
    evo = sharding.LocalShardedEvaluator(mm, [0, 0], mode="objects")
    goto = evo.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(goto[idx], oracle.evaluate_scalar(flat, x[idx]))


def test_sharded_entry_error_texts():
    model, x = _single(n=512)
    ev = sharding.LocalShardedEvaluator(model, [0, 0], mode="objects")
    with pytest.raises(ValueError, match="matrix has 3 features, model expects 24"):
        ev.predict(obt.FeatureMatrix(np.zeros((4, 3), np.float32), obt.Layout.OBJECT_MAJOR))
    # whole-model handles are not raw partial-sum models: the tree mode refuses them
    lib = _native.load_library()
    out = np.empty(512)
    rc = lib.obt_predict_sharded(ev._handles, 2, _native.SHARD_TREES, x.ctypes.data, 512, 0, 1.0, 0.0, out.ctypes.data)
    assert rc == _native.OBT_E_INVALID and b"raw partial-sum" in lib.obt_last_error()
