"""Every BASELINE configuration's full model shape (trees, depth, borders, features,
outputs) on the GPU against the oracle, bit for bit; and batches whose bucket matrix
passes 4 GiB (64-bit tile offsets in the quantize and apply kernels).

The reference's own acceptance sweep checks every batch against evaluate_scalar
(/root/reference/pkg/tests/test_acceptance.py:99-161, oracle.py:21-54); these are the
same checks at the BASELINE shapes (cfg5: the multi-output restatement, oracle.py:42-54
generalised to C outputs and depth 10)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import multiclass, synthetic

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _flat_multi(model):
    counts = np.array([b.size for b in model.borders], np.int32)
    borders = np.full((model.n_features, max(1, int(counts.max()))), np.inf, np.float32)
    for f, b in enumerate(model.borders):
        borders[f, : b.size] = b
    return oracle.FlatModel(borders, counts, np.full(model.n_trees, model.depth, np.int32), model.split_feature,
                            model.split_ordinal, model.leaves, model.scale, model.bias)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_full_model_shape_bit_exact(cfg):
    """The configuration's full model (config 1: 500 x depth 6 over 50 features ...
    config 4: 8,000 x depth 8 over 500 features, 128 borders) on 8,191 objects of its
    feature distribution with NaN / inf / border-hit / denormal specials, both layouts."""
    spec = synthetic.CONFIGS[cfg]
    model = synthetic.build_model(spec)
    x = synthetic.host_features(spec, n_objects=8191, seed=spec.data_seed + 11)
    x = synthetic.sprinkle_specials(x, [ff.borders for ff in model.float_features], seed=cfg)
    prec = oracle.BINARY16 if spec.half_leaves else oracle.BINARY64
    strategy = obt.LeafStrategy.NAIVE16 if spec.half_leaves else obt.LeafStrategy.NAIVE
    oracle.set_threads(oracle.host_cores())
    want = oracle.evaluate_scalar(oracle.flatten(model), x, oracle.OBJECT_MAJOR, prec)
    ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy), device=0)
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, want), int(np.count_nonzero(got != want))
    xt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    dev = ev.predict_device(xt, layout=obt.Layout.FEATURE_MAJOR).cpu().numpy()
    assert np.array_equal(dev, want)


def test_full_model_shape_config5_bit_exact():
    """Config 5's full model: 4,000 depth-10 trees over 1,000 features (254 borders), 10
    outputs; 4,097 objects against the multi-output restatement."""
    spec = synthetic.CONFIGS[5]
    model = multiclass.from_arrays(synthetic.model_arrays(spec))
    x = synthetic.host_features(spec, n_objects=4097, seed=spec.data_seed + 11)
    x = synthetic.sprinkle_specials(x, list(model.borders), seed=5)
    oracle.set_threads(oracle.host_cores())
    want = oracle.evaluate_scalar(_flat_multi(model), x).reshape(4097, spec.n_outputs)
    ev = multiclass.MultiOutputEvaluator(model, device=0)
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert ev.apply_kernel() == "staged"
    assert np.array_equal(got, want), int(np.count_nonzero(got != want))


def _rows(n: int, edge: int = 4096, step: int = 997) -> np.ndarray:
    return np.unique(np.concatenate([np.arange(edge), np.arange(n - edge, n), np.arange(0, n, n // step)]))


@pytest.mark.parametrize("kind", ["single", "multi"])
def test_bucket_matrix_past_4gib(kind):
    """A batch whose tiled bucket matrix passes 2^32 bytes (single output: F = 500 x 8.7M
    objects, the K1L quantize and K2w apply; multi-output: F = 1,000 x 4.4M objects,
    K5): the first and last tiles and a stride of rows equal the oracle bit for bit."""
    if kind == "single":
        spec = synthetic.WorkloadSpec("big", 8_700_000, 500, 128, 96, 8, 0.02, cfg=4)
        model = synthetic.build_model(spec)
        fm = oracle.flatten(model)
        ev = obt.Evaluator(model, device=0)
    else:
        spec = synthetic.WorkloadSpec("bigm", 4_400_000, 1000, 254, 24, 10, 0.01, n_outputs=10, cfg=5)
        model = multiclass.from_arrays(synthetic.model_arrays(spec))
        fm = _flat_multi(model)
        ev = multiclass.MultiOutputEvaluator(model, device=0)
    n, F = spec.n_objects, spec.n_features
    assert n * F > 2**32
    x = synthetic.device_features(spec, n_objects=n, seed=spec.data_seed, device="cuda:0")
    out = ev.predict_device(x)
    rows = _rows(n)
    idx = torch.from_numpy(rows).cuda()
    xs = x.index_select(0, idx).cpu().numpy()
    got = out.index_select(0, idx).cpu().numpy()
    del x, out
    torch.cuda.empty_cache()
    oracle.set_threads(oracle.host_cores())
    want = oracle.evaluate_scalar(fm, xs).reshape(got.shape)
    assert np.array_equal(got, want), int(np.count_nonzero(got != want))
