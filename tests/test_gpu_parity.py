"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bucket ids and leaf indices must be bit-exact; predictions are bit-exact too for
both precision families (binary64 tree-order fold of binary64/fp32-exact leaves;
binary16 leaves with a binary32 fold), which is stricter than the reference's own
1e-12 / 1e-6 tolerances (SPEC.md acceptance 3).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import _native, stages, synthetic

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _model(F, B, T, D, seed, affine=True, sigma=0.1):
    spec = synthetic.WorkloadSpec("t", 1, F, B, T, D, sigma, cfg=1)
    return synthetic.build_model(spec, seed=seed, affine=affine)


def _features(model, n, seed, specials=True):
    spec = synthetic.WorkloadSpec("t", n, model.n_features, 1, 1, 1, 0.1, cfg=1)
    x = synthetic.host_features(spec, seed=seed)
    if specials:
        x = synthetic.sprinkle_specials(x, [ff.borders for ff in model.float_features], seed=seed + 1)
    return x


def _mixed_depth_model(F, B, T, seed):
    rng = np.random.default_rng(seed)
    base = _model(F, B, 1, 1, seed)
    trees = []
    for _ in range(T):
        d = int(rng.integers(1, 9))
        splits = tuple(obt.SplitCondition(int(rng.integers(0, F)), int(rng.integers(0, B))) for _ in range(d))
        trees.append(obt.ObliviousTree(depth=d, splits=splits, leaf_values=rng.uniform(-1, 1, 1 << d)))
    return obt.ObliviousModel(base.float_features, tuple(trees), scale=1.25, bias=-0.5)


def test_smoke():
    import __graft_entry__ as ge

    ge.smoke()


@pytest.mark.parametrize("layout", [obt.Layout.OBJECT_MAJOR, obt.Layout.FEATURE_MAJOR])
@pytest.mark.parametrize("B", [1, 7, 16, 64, 127, 128, 200, 254])
def test_quantize_bit_exact(layout, B):
    model = _model(23, B, 3, 2, seed=B)
    x = _features(model, 1537, seed=100 + B)
    fm = oracle.flatten(model)
    xin = x if layout is obt.Layout.OBJECT_MAJOR else np.ascontiguousarray(x.T)
    got = stages.quantize(model, torch.from_numpy(xin).cuda(), layout).cpu().numpy()
    want = oracle.quantize(fm, xin, oracle.OBJECT_MAJOR if layout is obt.Layout.OBJECT_MAJOR else oracle.FEATURE_MAJOR)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


@pytest.mark.parametrize("D", [1, 2, 3, 5, 6, 7, 8])
@pytest.mark.parametrize("B", [16, 128, 254])
def test_leaf_indices_bit_exact(D, B):
    model = _model(17, B, 37, D, seed=D * 7 + B)
    x = _features(model, 777, seed=D)
    fm = oracle.flatten(model)
    got = stages.as_uint16(stages.leaf_indices(model, torch.from_numpy(x).cuda()))
    want = oracle.leaf_indices(fm, oracle.quantize(fm, x))
    assert np.array_equal(got, want)


def test_leaf_indices_tree_range_and_mixed_depth():
    model = _mixed_depth_model(9, 30, 50, seed=3)
    x = _features(model, 300, seed=4)
    fm = oracle.flatten(model)
    want = oracle.leaf_indices(fm, oracle.quantize(fm, x))
    got = stages.as_uint16(stages.leaf_indices(model, torch.from_numpy(x).cuda(), tree_begin=11, tree_end=29))
    assert np.array_equal(got, want[11:29])


@pytest.mark.parametrize("strategy", [obt.LeafStrategy.NAIVE, obt.LeafStrategy.NAIVE16])
@pytest.mark.parametrize("n", [1, 7, 31, 32, 33, 100, 128, 257, 4099])
def test_predict_bit_exact_batch_sizes(strategy, n):
    model = _model(31, 40, 90, 6, seed=n)
    x = _features(model, n, seed=n + 5)
    prec = oracle.BINARY64 if strategy is obt.LeafStrategy.NAIVE else oracle.BINARY16
    want = oracle.evaluate_scalar(oracle.flatten(model), x, oracle.OBJECT_MAJOR, prec)
    got = obt.Evaluator(model, obt.EvalConfig(strategy=strategy)).predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("D", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("B", [5, 64, 128, 254])
def test_predict_bit_exact_depth_borders(D, B):
    model = _model(13, B, 61, D, seed=1000 + D * 10 + B)
    x = _features(model, 513, seed=D + B)
    fm = oracle.flatten(model)
    for strategy, prec in ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.PERMUTE16, oracle.BINARY16)):
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy, width=obt.VectorWidth.W512))
        got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
        want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
        assert np.array_equal(got, want), (strategy, int(np.count_nonzero(got != want)))


def test_predict_binary64_leaves_not_fp32_exact():
    """Arbitrary binary64 leaves (not fp32-representable) use the fp64 table."""
    rng = np.random.default_rng(11)
    base = _model(8, 20, 1, 1, seed=11)
    trees = tuple(
        obt.ObliviousTree(
            depth=5,
            splits=tuple(obt.SplitCondition(int(rng.integers(0, 8)), int(rng.integers(0, 20))) for _ in range(5)),
            leaf_values=rng.standard_normal(32) * 10.0 ** rng.integers(-8, 3),
        )
        for _ in range(70)
    )
    model = obt.ObliviousModel(base.float_features, trees, scale=0.75, bias=0.125)
    x = _features(model, 999, seed=12)
    ev = obt.Evaluator(model)
    assert ev.leaf_storage == "fp64"
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, oracle.evaluate_scalar(oracle.flatten(model), x))


def test_predict_mixed_depth_and_layouts():
    model = _mixed_depth_model(11, 25, 120, seed=21)
    x = _features(model, 1000, seed=22)
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    ev = obt.Evaluator(model)
    om = obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)
    assert np.array_equal(ev.predict(om), want)
    assert np.array_equal(ev.predict(om.transposed()), want)


def test_predict_zero_trees_and_empty_batch():
    model = obt.ObliviousModel(
        float_features=(obt.FloatFeatureBorders(0, np.array([0.5], dtype=np.float32)),), trees=(), scale=2.0, bias=0.75
    )
    ev = obt.Evaluator(model)
    x = np.zeros((5, 1), dtype=np.float32)
    assert np.all(ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)) == 0.75)
    assert ev.predict(obt.FeatureMatrix(np.zeros((0, 1), np.float32), obt.Layout.OBJECT_MAJOR)).shape == (0,)


def test_depth3_known_answer():
    # (root, d1, d2) conditions (1, 0, 1) address leaf 0b101 = 5 (test_acceptance.py:194-214)
    features = tuple(obt.FloatFeatureBorders(i, np.array([0.5], dtype=np.float32)) for i in range(3))
    tree = obt.ObliviousTree(
        depth=3,
        splits=(obt.SplitCondition(0, 0), obt.SplitCondition(1, 0), obt.SplitCondition(2, 0)),
        leaf_values=np.arange(10.0, 18.0),
    )
    model = obt.ObliviousModel(features, (tree,), scale=2.0, bias=1.0)
    x = np.array([[1.0, 0.0, 1.0]], dtype=np.float32)
    assert obt.evaluate(model, obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))[0] == 15.0 * 2.0 + 1.0
    idx = stages.as_uint16(stages.leaf_indices(model, torch.from_numpy(x).cuda()))
    assert idx[0, 0] == 5


def test_binary16_infinite_leaves_saturate_like_the_reference():
    """Infinite leaves become +/-65504 in the binary16 bank (model.py:262-268), so the
    NAIVE16 predictions are the reference's finite sums (golden from the reference)."""
    import json
    from pathlib import Path

    g = json.loads((Path(__file__).parent / "golden" / "known_answers.json").read_text())["half_saturation_inf"]
    from test_host_api import _inf_leaf_model

    model = _inf_leaf_model()
    x = np.array([[0.25], [0.75], [np.nan], [0.5]], np.float32)
    ev = obt.Evaluator(model, obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16), device=0)
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert got.tolist() == g["predictions_naive16"] == g["predictions_scalar16"]
    want = oracle.evaluate_scalar(oracle.flatten(model), x, oracle.OBJECT_MAJOR, oracle.BINARY16)
    assert np.array_equal(got, want)


def test_device_entry_points_check_every_buffer():
    """out / workspace / x are checked before a pointer reaches the kernels: wrong dtype,
    short or non-contiguous outputs and foreign devices raise instead of writing."""
    from paper_2211_00391_b200 import multiclass

    model = _model(8, 16, 12, 4, seed=5)
    ev = obt.Evaluator(model, device=0)
    x = torch.from_numpy(_features(model, 300, seed=6)).cuda()
    good = ev.predict_device(x)
    bad_outs = [torch.empty(300, dtype=torch.float32, device="cuda"), torch.empty(299, dtype=torch.float64, device="cuda"),
                torch.empty(600, dtype=torch.float64, device="cuda")[::2], torch.empty(300, dtype=torch.float64)]
    for out in bad_outs:
        with pytest.raises(ValueError):
            ev.predict_device(x, out=out)
        with pytest.raises(ValueError):
            ev.predict_device_marked(x, [None, None, None], out=out)
    with pytest.raises(ValueError):
        ev.predict_device(x, workspace=torch.empty(1 << 20, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        ev.predict_device(x.double())
    with pytest.raises(ValueError, match="features"):
        ev.predict_device(x[:, :7])
    with pytest.raises(ValueError):
        ev.predict(obt.FeatureMatrix(x.cpu().numpy(), obt.Layout.OBJECT_MAJOR), out=np.empty(300, np.float32))
    assert torch.equal(ev.predict_device(x[::1]), good)
    mm = multiclass.from_arrays(synthetic.model_arrays(synthetic.WorkloadSpec("m", 1, 8, 16, 12, 4, 0.1, cfg=5,
                                                                               n_outputs=3)))
    mev = multiclass.MultiOutputEvaluator(mm, device=0)
    with pytest.raises(ValueError):
        mev.predict_device(x, out=torch.empty(300, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        mev.predict(obt.FeatureMatrix(x.cpu().numpy(), obt.Layout.OBJECT_MAJOR), out=np.empty(300, np.float64))
    assert mev.predict_device(x).shape == (300, 3)


def test_predict_device_matches_host_path():
    model = _model(40, 64, 200, 6, seed=5, affine=False)
    x = _features(model, 20000, seed=6, specials=False)
    ev = obt.Evaluator(model)
    host = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    dev = ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(host, dev)
    ws = torch.empty(ev.workspace_bytes(x.shape[0]), dtype=torch.uint8, device="cuda")
    dev2 = ev.predict_device(torch.from_numpy(x).cuda(), workspace=ws).cpu().numpy()
    assert np.array_equal(host, dev2)


@pytest.mark.parametrize("D", [9, 10, 12])
def test_predict_deeper_than_reference(D):
    """Depths 9..12 (the multiclass config needs 10) through the padded instantiations."""
    rng = np.random.default_rng(D)
    F, B, T = 10, 30, 25
    borders = tuple(obt.FloatFeatureBorders(f, np.sort(rng.standard_normal(B)).astype(np.float32)) for f in range(F))
    fm = oracle.FlatModel(
        borders=np.stack([b.borders for b in borders]),
        border_counts=np.full(F, B, np.int32),
        depths=np.full(T, D, np.int32),
        split_feature=rng.integers(0, F, (T, D)).astype(np.int32),
        split_ordinal=rng.integers(0, B, (T, D)).astype(np.int32),
        leaves=rng.standard_normal((T, 1, 1 << D)).astype(np.float32).astype(np.float64),
        scale=1.0,
        bias=0.0,
    )
    x = rng.standard_normal((700, F)).astype(np.float32)
    want = oracle.evaluate_scalar(fm, x)
    from paper_2211_00391_b200.evaluate import DeviceModel  # noqa: F401 (low-level path below)
    import ctypes

    from paper_2211_00391_b200 import _native

    lib = _native.require_gpu()
    desc = _native.ModelDesc()
    so = fm.split_ordinal.astype(np.uint8)
    leaves = np.ascontiguousarray(fm.leaves[:, 0, :])
    desc.n_features, desc.n_trees, desc.max_depth, desc.n_outputs = F, T, D, 1
    desc.border_counts = fm.border_counts.ctypes.data
    desc.borders = fm.borders.ctypes.data
    desc.border_stride = B
    desc.split_feature = fm.split_feature.ctypes.data
    desc.split_ordinal = so.ctypes.data
    desc.leaves = leaves.ctypes.data
    desc.leaves_f16 = None
    desc.scale, desc.bias, desc.precision = 1.0, 0.0, 0
    h = ctypes.c_void_p()
    _native.check(lib.obt_model_create(ctypes.byref(desc), 0, ctypes.byref(h)))
    try:
        xd = torch.from_numpy(x).cuda()
        out = torch.empty(x.shape[0], dtype=torch.float64, device="cuda")
        _native.check(lib.obt_predict_dev(h, xd.data_ptr(), x.shape[0], 0, out.data_ptr(), None, 0,
                                          _native.current_stream_handle()))
        got = out.cpu().numpy()
    finally:
        lib.obt_model_destroy(h)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("source", ["param", "smem"])
@pytest.mark.parametrize("strategy", [obt.LeafStrategy.NAIVE, obt.LeafStrategy.NAIVE16])
def test_descriptor_sources_and_multi_launch_fold(paths, source, strategy):
    """3,000 depth-6 trees exceed one launch's parameter bank (about 1,300 trees), so the
    parameter path folds across 3 launches through the carried accumulators; the
    shared-memory path streams all descriptors in one launch.  Both are bit-exact."""
    paths(desc_source=1 if source == "param" else 0)
    paths(fan=0)  # the K2 / K2s paths, not the small-batch K2f
    model = _model(12, 50, 3001, 6, seed=77)
    x = _features(model, 2500, seed=78)
    prec = oracle.BINARY64 if strategy is obt.LeafStrategy.NAIVE else oracle.BINARY16
    want = oracle.evaluate_scalar(oracle.flatten(model), x, oracle.OBJECT_MAJOR, prec)
    ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy))
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, want)
    idx = stages.as_uint16(stages.leaf_indices(model, torch.from_numpy(x).cuda(), tree_begin=1290, tree_end=1400))
    fm = oracle.flatten(model)
    assert np.array_equal(idx, oracle.leaf_indices(fm, oracle.quantize(fm, x))[1290:1400])


@pytest.mark.parametrize("kernel", ["staged", "k4"])
@pytest.mark.parametrize("D,C,F,B", [(10, 10, 40, 254), (6, 3, 17, 64), (8, 16, 9, 128), (3, 2, 5, 7), (12, 7, 13, 30),
                                     (10, 9, 33, 100), (4, 5, 8, 200), (10, 4, 2, 254)])  # last: 8-bit compare
def test_multi_output_bit_exact(paths, kernel, D, C, F, B):
    """Multi-output (config 5 shape family): K5 (staged tables, default where it applies:
    fp32 records, C <= 10, depth <= 10) and K4 (path option multi_staged=0) against the
    oracle restatement, both layouts, with the binary64 leaf tables too (leaf_storage=0,
    which K5 leaves to K4)."""
    from paper_2211_00391_b200 import multiclass

    paths(multi_staged=1 if kernel == "staged" else 0)

    spec = synthetic.WorkloadSpec("m", 1, F, B, 57, D, 0.01, n_outputs=C, cfg=5)
    arrays = synthetic.model_arrays(spec, seed=D * 100 + C, affine=True)
    model = multiclass.from_arrays(arrays)
    x = _features(obt.ObliviousModel(tuple(obt.FloatFeatureBorders(f, b) for f, b in enumerate(arrays["borders"])),
                                      (), 1.0, 0.0), 4097, seed=D + C)
    fm = oracle.FlatModel(np.stack(arrays["borders"]), np.full(F, B, np.int32), np.full(57, D, np.int32),
                          arrays["split_feature"], arrays["split_ordinal"], arrays["leaves"], model.scale, model.bias)
    want = oracle.evaluate_scalar(fm, x)
    ev = multiclass.MultiOutputEvaluator(model)
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert got.shape == (4097, C)
    if kernel == "staged" and C <= 10 and D <= 10:
        assert ev.apply_kernel() == "staged"
    assert np.array_equal(got, want)
    dev = ev.predict_device(torch.from_numpy(np.ascontiguousarray(x.T)).cuda(), obt.Layout.FEATURE_MAJOR).cpu().numpy()
    assert np.array_equal(dev, want)
    paths(leaf_storage=0)
    ev64 = multiclass.MultiOutputEvaluator(model)
    assert np.array_equal(ev64.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)), want)


@pytest.mark.parametrize("D,C,F,B", [(10, 10, 40, 254), (6, 3, 17, 64), (8, 8, 9, 128), (3, 2, 5, 7),
                                     (10, 9, 33, 100), (4, 5, 8, 200), (10, 4, 2, 254), (8, 7, 12, 16)])
def test_multi_output_binary16_half2_records(D, C, F, B):
    """The binary16 family for multi-output models (EvalConfig NAIVE16): each output's
    leaves through the reference's binary16 bank (RNE, +-65504 saturation) and a
    binary32 fold; on the GPU the records pack two binary16 outputs per word (half2) and
    fold two outputs per FADD2.  Bit-exact against the oracle's BINARY16 evaluation,
    both layouts, including saturated leaves."""
    from paper_2211_00391_b200 import multiclass

    spec = synthetic.WorkloadSpec("m", 1, F, B, 57, D, 0.01, n_outputs=C, cfg=5)
    arrays = synthetic.model_arrays(spec, seed=D * 100 + C + 7, affine=True)
    arrays["leaves"][0, 0, :2] = (7.0e4, -9.0e4)   # saturate to +-65504 (model.py:262-268)
    arrays["leaves"][1, C - 1, 3] = np.inf
    model = multiclass.from_arrays(arrays)
    x = _features(obt.ObliviousModel(tuple(obt.FloatFeatureBorders(f, b) for f, b in enumerate(arrays["borders"])),
                                      (), 1.0, 0.0), 4097, seed=D + C + 1)
    fm = oracle.FlatModel(np.stack(arrays["borders"]), np.full(F, B, np.int32), np.full(57, D, np.int32),
                          arrays["split_feature"], arrays["split_ordinal"], arrays["leaves"], model.scale, model.bias)
    want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY16)
    ev = multiclass.MultiOutputEvaluator(model, config=obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16))
    assert ev.leaf_storage == "fp16" and ev.apply_kernel() == "staged"
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert got.shape == (4097, C)
    assert np.array_equal(got, want), int(np.count_nonzero(got != want))
    dev = ev.predict_device(torch.from_numpy(np.ascontiguousarray(x.T)).cuda(), obt.Layout.FEATURE_MAJOR).cpu().numpy()
    assert np.array_equal(dev, want)


def test_multi_output_binary16_limits():
    """The binary16 multi-output family runs on the staged kernel only: more than 10
    outputs or depth above 10 are refused with a message, not run elsewhere."""
    from paper_2211_00391_b200 import multiclass

    for D, C in ((12, 3), (6, 12)):
        spec = synthetic.WorkloadSpec("m", 1, 6, 16, 9, D, 0.01, n_outputs=C, cfg=5)
        model = multiclass.from_arrays(synthetic.model_arrays(spec, seed=3))
        with pytest.raises(_native.NativeError, match="binary16 multi-output"):
            multiclass.MultiOutputEvaluator(model, config=obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16))


def test_multi_output_tree_shard_partials_sum_to_prediction():
    """Tree sharding of a multi-output model: partial sums of the shards (scale 1, bias 0)
    reduce to the full prediction within binary64 reassociation."""
    from paper_2211_00391_b200 import multiclass, sharding

    spec = synthetic.WorkloadSpec("m", 1, 30, 100, 203, 10, 0.01, n_outputs=10, cfg=5)
    model = multiclass.from_arrays(synthetic.model_arrays(spec, seed=5, affine=True))
    x = np.random.default_rng(1).standard_normal((777, 30)).astype(np.float32)
    full = multiclass.MultiOutputEvaluator(model).predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    parts = []
    for r in range(4):
        b, e = sharding.tree_shard(model.n_trees, r, 4)
        parts.append(multiclass.MultiOutputEvaluator(model.subset(b, e)).predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)))
    combined = sum(parts) * model.scale + model.bias
    assert np.max(np.abs(combined - full) / np.maximum(np.abs(full), 1e-300)) < 1e-12


@pytest.mark.parametrize("n", [1, 129, 1000, 4097])
@pytest.mark.parametrize("tpw", ["1", "2"])
def test_no_writes_outside_outputs_and_workspace(paths, n, tpw):
    """compute-sanitizer is unavailable on this pool: guard regions around the score
    vector and the bucket workspace must be untouched after a predict (ragged n, both
    apply kernels), and results must still match the oracle."""
    paths(tpw=int(tpw))
    paths(fan=0)  # the K2 / K2s paths, not the small-batch K2f
    model = _model(24, 60, 75, 6, seed=n)
    x = _features(model, n, seed=n)
    ev = obt.Evaluator(model)
    guard = 64
    out = torch.full((n + guard,), 12345.0, dtype=torch.float64, device="cuda")
    ws_bytes = ev.workspace_bytes(n)
    ws = torch.full((ws_bytes + 4096,), 0xAB, dtype=torch.uint8, device="cuda")
    ev.predict_device(torch.from_numpy(x).cuda(), out=out[:n], workspace=ws[:ws_bytes])
    torch.cuda.synchronize()
    assert torch.all(out[n:] == 12345.0)
    assert torch.all(ws[ws_bytes:] == 0xAB)
    assert np.array_equal(out[:n].cpu().numpy(), oracle.evaluate_scalar(oracle.flatten(model), x))


def test_multi_output_no_writes_outside_output():
    from paper_2211_00391_b200 import multiclass

    spec = synthetic.WorkloadSpec("m", 1, 11, 30, 21, 10, 0.01, n_outputs=10, cfg=5)
    mm = multiclass.from_arrays(synthetic.model_arrays(spec, seed=9))
    n = 777
    x = torch.randn(n, 11, device="cuda")
    big = torch.full((n * 10 + 80,), -7.0, dtype=torch.float64, device="cuda")
    multiclass.MultiOutputEvaluator(mm).predict_device(x, out=big[: n * 10].view(n, 10))
    torch.cuda.synchronize()
    assert torch.all(big[n * 10:] == -7.0)


def test_reference_corpus_on_gpu():
    """The reference's 100-model acceptance corpus (tests/golden/corpus.npz, written by
    running the reference itself): GPU predictions equal the reference's outputs bit for
    bit in both precision families, and GPU buckets / leaf indices equal its panels."""
    from pathlib import Path

    corpus = np.load(Path(__file__).parent / "golden" / "corpus.npz")
    families = ((obt.LeafStrategy.NAIVE, "oracle64"), (obt.LeafStrategy.NAIVE16, "oracle16"))
    off = 0
    for i, (F, B, T, D, seed) in enumerate(corpus["specs"]):
        model = oracle.to_model(oracle.synthetic_model(int(F), int(B), int(T), int(D), int(seed)), obt)
        evs = [(obt.Evaluator(model, obt.EvalConfig(strategy=s)), key) for s, key in families]
        for batch in corpus["batch_sizes"]:
            x = oracle.feature_matrix(int(batch), int(F), int(seed) * 13 + int(batch), nan_fraction=0.02,
                                      inf_fraction=0.01)
            for ev, key in evs:
                got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
                assert np.array_equal(got, corpus[key][off: off + int(batch)]), (i, int(batch), key)
            off += int(batch)
    assert off == corpus["oracle64"].size
    for name in corpus.files:
        if not name.startswith("q"):
            continue
        i = int(name[1:])
        F, B, T, D, seed = (int(v) for v in corpus["specs"][i])
        model = oracle.to_model(oracle.synthetic_model(F, B, T, D, seed), obt)
        x = torch.from_numpy(oracle.feature_matrix(257, F, seed * 13 + 257, nan_fraction=0.02, inf_fraction=0.01))
        assert np.array_equal(stages.quantize(model, x.cuda()).cpu().numpy(), corpus[name])
        assert np.array_equal(stages.as_uint16(stages.leaf_indices(model, x.cuda())), corpus[f"i{i}"].astype(np.uint16))


@pytest.mark.parametrize("tpw", ["2", "4"])
@pytest.mark.parametrize("D", [4, 8])
@pytest.mark.parametrize("F,B,T", [(29, 100, 70), (3, 254, 200)])  # 7-bit / 8-bit compare after remap
def test_depth_split_lanes_bit_exact(paths, tpw, D, F, B, T):
    """K2s: TPW lanes per bucket word (path option tpw forces it) keep the tree-order fold exact."""
    paths(tpw=int(tpw))
    paths(fan=0)  # the K2 / K2s paths, not the small-batch K2f
    model = _model(F, B, T, D, seed=D * 100 + F)
    x = _features(model, 3001, seed=D + F)
    fm = oracle.flatten(model)
    for strategy, prec in ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16)):
        got = obt.Evaluator(model, obt.EvalConfig(strategy=strategy)).predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
        want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
        assert np.array_equal(got, want), (strategy, int(np.count_nonzero(got != want)))


def test_default_mempool_left_alone():
    """Workspace and staging buffers come from the library's own pool: the device's
    default pool (the application's) keeps its release threshold."""
    rt = pytest.importorskip("cuda.bindings.runtime")
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    assert err == rt.cudaError_t.cudaSuccess
    attr = rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold
    err, before = rt.cudaMemPoolGetAttribute(pool, attr)
    model = _model(11, 20, 30, 6, seed=5)
    x = _features(model, 5000, seed=6)
    ev = obt.Evaluator(model)
    ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    ev.predict_device(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    err, after = rt.cudaMemPoolGetAttribute(pool, attr)
    assert int(after) == int(before)


def test_concurrent_predicts_from_threads():
    """Reentrancy: host threads predicting concurrently on their own streams,
    with batch sizes that give different tiles and shared-memory sizes, all bit-exact."""
    import threading

    cases = []
    for i, (F, n) in enumerate([(13, 700), (40, 90000), (13, 33000), (77, 5000)]):
        model = _model(F, 50, 120, 6 if i % 2 else 5, seed=40 + i)
        x = _features(model, n, seed=50 + i)
        cases.append((model, x, oracle.evaluate_scalar(oracle.flatten(model), x)))
    errors = []

    def worker(model, x, want):
        try:
            ev = obt.Evaluator(model)
            xd = torch.from_numpy(x).cuda()
            torch.cuda.current_stream().synchronize()  # the copy ran on this thread's default stream
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(6):
                    got = ev.predict_device(xd)
                    s.synchronize()
                    if not np.array_equal(got.cpu().numpy(), want):
                        errors.append("device path mismatch")
                    if not np.array_equal(ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)), want):
                        errors.append("host path mismatch")
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=c) for c in cases]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:3]


@pytest.mark.parametrize("F", [4, 8, 12, 200])
@pytest.mark.parametrize("n", [1, 127, 1023, 1025, 4099])
def test_tma_quantize_path_ragged_batches(F, n):
    """K1t (TMA-staged rows: object-major, F % 4 == 0, 16-byte aligned) on ragged
    batches -- partial CTAs and zero-filled rows past n -- and the LDG fallback on the
    same data through a misaligned view (forces K1): both bit-exact."""
    model = _model(F, 64, 50, 6, seed=F * 10 + n % 7)
    x = _features(model, n, seed=F + n)
    fm = oracle.flatten(model)
    want = oracle.evaluate_scalar(fm, x)
    ev = obt.Evaluator(model)
    xd = torch.from_numpy(x).cuda()
    assert np.array_equal(ev.predict_device(xd).cpu().numpy(), want)
    pad = torch.empty(n * F + 1, dtype=torch.float32, device="cuda")
    xm = pad[1:].view(n, F)  # 4-byte aligned only: not eligible for the tensor map
    xm.copy_(xd)
    assert np.array_equal(ev.predict_device(xm).cpu().numpy(), want)
    q_ref = oracle.quantize(fm, x)
    assert np.array_equal(stages.quantize(model, xd).cpu().numpy(), q_ref)


def test_misaligned_workspace_and_output_rejected():
    """Caller buffers the kernels cannot use are refused with OBT_E_INVALID, not faulted on."""
    from paper_2211_00391_b200 import _native

    model = _model(8, 16, 10, 4, seed=3)
    x = torch.from_numpy(_features(model, 300, seed=4)).cuda()
    ev = obt.Evaluator(model)
    ws = torch.empty(ev.workspace_bytes(300) + 512, dtype=torch.uint8, device="cuda")
    with pytest.raises(_native.NativeError, match="256-byte aligned"):
        ev.predict_device(x, workspace=ws[1:])
    lib = _native.require_gpu()
    out = torch.empty(301, dtype=torch.float64, device="cuda")
    handle = ev._dev.handle if hasattr(ev, "_dev") else None
    if handle is None:
        pytest.skip("evaluator exposes no device handle")
    rc = lib.obt_predict_dev(handle, x.data_ptr(), 300, 0, out.data_ptr() + 4, None, 0,
                             _native.current_stream_handle())
    assert rc == _native.OBT_E_INVALID and b"8-byte aligned" in lib.obt_last_error()
    ev.predict_device(x, workspace=ws[:ev.workspace_bytes(300)])  # aligned: fine


@pytest.mark.parametrize("D", [6, 8])
@pytest.mark.parametrize("layout", [obt.Layout.OBJECT_MAJOR, obt.Layout.FEATURE_MAJOR])
def test_tail_wave_split_bit_exact(paths, D, layout):
    """Batches past one full wave run the partial last wave as a second region of
    smaller tiles (F = 500: 384-object tiles, 148 per wave): bit-exact against the oracle
    and against the single-region path, in both input layouts."""
    model = _model(500, 64, 30, D, seed=D)
    n = 70001
    x = _features(model, n, seed=D + 1, specials=False)
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    ev = obt.Evaluator(model)
    xin = x if layout is obt.Layout.OBJECT_MAJOR else np.ascontiguousarray(x.T)
    xd = torch.from_numpy(xin).cuda()
    got = ev.predict_device(xd, layout=layout).cpu().numpy()
    assert np.array_equal(got, want)
    paths(tail_split=0)
    assert np.array_equal(ev.predict_device(xd, layout=layout).cpu().numpy(), want)


def test_config_invariance_within_precision_family():
    """Every valid EvalConfig of a precision family gives the same bits (the reference's
    layout/width/block/tail invariance, test_evaluate.py:172-213)."""
    import itertools

    from paper_2211_00391_b200.config import BLOCK_SIZES, TailPolicy, VectorWidth

    model = _mixed_depth_model(19, 40, 70, seed=21)
    x = _features(model, 777, seed=22)
    fm = oracle.flatten(model)
    want = {oracle.BINARY64: oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY64),
            oracle.BINARY16: oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY16)}
    checked = 0
    for strategy, width, block, tail in itertools.product(obt.LeafStrategy, VectorWidth, BLOCK_SIZES, TailPolicy):
        cfg = obt.EvalConfig(block_size=block, width=width, strategy=strategy, tail_policy=tail)
        try:
            cfg.validate()
        except ValueError:
            continue
        prec = oracle.BINARY16 if strategy.precision.value == "binary16" else oracle.BINARY64
        got = obt.Evaluator(model, cfg).predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
        assert np.array_equal(got, want[prec]), cfg.describe()
        checked += 1
    assert checked >= 10


def test_prediction_is_the_composition_of_the_stages():
    """Fused = unit composition (test_evaluate.py:271-300): GPU leaf indices folded on the
    host in tree order with the bank's leaves, then scale/bias, equal the GPU prediction."""
    model = _mixed_depth_model(23, 50, 64, seed=31)
    x = _features(model, 1500, seed=32)
    idx = stages.as_uint16(stages.leaf_indices(model, torch.from_numpy(x).cuda())).astype(np.int64)
    acc = np.zeros(x.shape[0])
    for t, tree in enumerate(model.trees):
        acc = acc + np.asarray(tree.leaf_values, dtype=np.float64)[idx[t]]
    want = acc * model.scale + model.bias
    got = obt.Evaluator(model).predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, want)


def test_fp16_family_within_reference_bound():
    """FP16 leaves vs binary64 leaves on the GPU: |p16 - p64| <= |scale| T max|leaf| 2^-10
    (test_acceptance.py:156, 240-247), and the binary16 family matches its oracle exactly."""
    model = _model(40, 64, 300, 6, seed=41, sigma=0.05)
    x = _features(model, 4000, seed=42)
    fmx = obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)
    p64 = obt.Evaluator(model, obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE)).predict(fmx)
    p16 = obt.Evaluator(model, obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16)).predict(fmx)
    max_leaf = max(float(np.abs(t.leaf_values).max()) for t in model.trees)
    bound = abs(model.scale) * model.n_trees * max_leaf * 2.0 ** -10
    assert float(np.abs(p16 - p64).max()) <= bound
    assert np.array_equal(p16, oracle.evaluate_scalar(oracle.flatten(model), x, oracle.OBJECT_MAJOR, oracle.BINARY16))


def test_predict_captures_into_cuda_graph():
    """predict_device is capturable (stream-ordered allocations, by-value tensor map,
    plans built at warm-up): a CUDA graph replay is bit-exact and tracks new inputs."""
    model = _model(24, 40, 120, 6, seed=61)
    x1 = _features(model, 5000, seed=62)
    x2 = _features(model, 5000, seed=63)
    fm = oracle.flatten(model)
    ev = obt.Evaluator(model)
    xd = torch.from_numpy(x1).cuda()
    out = torch.empty(5000, dtype=torch.float64, device="cuda")
    ws = torch.empty(ev.workspace_bytes(5000), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ev.predict_device(xd, out=out, workspace=ws)  # warm-up: tile plans, attributes
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ev.predict_device(xd, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.evaluate_scalar(fm, x1))
    xd.copy_(torch.from_numpy(x2))
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.evaluate_scalar(fm, x2))


def _border_model(border_sets, T, D, seed):
    """A model over hand-made border sets (one feature each), random splits."""
    rng = np.random.default_rng(seed)
    feats = tuple(obt.FloatFeatureBorders(f, np.asarray(b, np.float32)) for f, b in enumerate(border_sets))
    usable = [f for f, b in enumerate(border_sets) if len(b)]
    trees = []
    for _ in range(T):
        splits = []
        for _ in range(D):
            f = int(rng.choice(usable))
            splits.append(obt.SplitCondition(f, int(rng.integers(0, len(border_sets[f])))))
        trees.append(obt.ObliviousTree(depth=D, splits=tuple(splits), leaf_values=rng.normal(0, 0.1, 1 << D).astype(np.float32)))
    return obt.ObliviousModel(feats, tuple(trees), scale=1.0, bias=0.0)


def _edge_values(border_sets, n, seed):
    """Values at, just above and just below every border, plus NaN, +-inf, +-0, denormals."""
    rng = np.random.default_rng(seed)
    F = len(border_sets)
    x = np.empty((n, F), np.float32)
    for f, b in enumerate(border_sets):
        b = np.asarray(b, np.float32)
        pool = [np.float32(np.nan), np.float32(np.inf), np.float32(-np.inf), np.float32(0.0), np.float32(-0.0),
                np.float32(2.0**-140), np.float32(-(2.0**-140)), np.float32(3.4e38), np.float32(-3.4e38)]
        if b.size:
            pool += list(b) + list(np.nextafter(b, np.float32(np.inf))) + list(np.nextafter(b, np.float32(-np.inf)))
            lo, hi = float(b.min()), float(b.max())
            span = max(hi - lo, 1.0)
            pool += list(rng.uniform(lo - span, hi + span, 64).astype(np.float32))
        x[:, f] = np.asarray(pool, np.float32)[rng.integers(0, len(pool), n)]
    return x


_LUT_SETS = {
    # cfg-like quantile / uniform / integer / lognormal sets, singletons, clustered borders
    # (up to 4 per cell), denormal and signed-zero borders, an empty feature
    "mixed": [
        np.sort(np.random.default_rng(1).normal(0, 1, 64)).astype(np.float32),
        (100 * np.arange(1, 65) / 65).astype(np.float32),
        np.unique(np.floor(1000 * np.arange(1, 129) / 129)).astype(np.float32),
        np.unique(np.exp(np.random.default_rng(2).normal(0, 1, 40))).astype(np.float32),
        np.array([0.5], np.float32),
        np.array([-0.0, 2.0**-140, 1.0], np.float32),
        np.array([0.0, 1e-3, 2e-3, 3e-3, 10.0], np.float32),   # 4 borders share the lowest cell
        np.array([-5.0, -4.999999, -4.999998, 7.0], np.float32),
    ],
    # ranges the affine cell map cannot hold: the Eytzinger search runs instead
    "fallback": [
        np.array([1e6, 1000001.0, 1000002.0], np.float32),  # lo * s ~ 2.5e8 > 2^23
        np.sort(np.random.default_rng(3).normal(0, 1, 16)).astype(np.float32),
    ],
    # five borders in one of 256 cells, at most two in one of 1024: the 1024-cell tables
    "crowded256": [
        np.array([0.0, 0.25, 0.5, 0.75, 0.9, 255.0], np.float32),
        np.sort(np.random.default_rng(4).normal(0, 1, 30)).astype(np.float32),
    ],
    # five borders in one cell even at 1024 cells: more than the cell kernel's compares
    "crowded": [
        np.array([0.0, 1e-6, 2e-6, 3e-6, 4e-6, 100.0], np.float32),
        np.array([1.0, 2.0], np.float32),
    ],
}


@pytest.mark.parametrize("name,expect,cells", [("mixed", "cells", "256"), ("mixed", "cells1024", "1024"),
                                              ("fallback", "eytzinger", ""), ("crowded256", "cells1024", ""),
                                              ("crowded", "eytzinger", "")])
def test_cell_table_quantize_edges(paths, name, expect, cells):
    """K1L (cell-table quantize) against the oracle on values at, next to and far from
    every border, NaN, +-inf, signed zeros and denormals; and equal to the Eytzinger
    search (path option quant_lut=0) bucket for bucket through the predictions and leaf indices."""
    paths(quant_lut=1)  # K1L wherever its tables exist (not only where it is faster)
    if cells:
        paths(lut_cells=int(cells))
    sets = [np.asarray(b, np.float32) for b in _LUT_SETS[name]]
    pad = (-len(sets)) % 4  # F % 4 == 0: the TMA-staged path
    sets += [np.array([0.25 * (i + 1)], np.float32) for i in range(pad)]
    model = _border_model(sets, T=40, D=6, seed=len(sets))
    ev = obt.Evaluator(model)
    dm = ev.tables.device_model(ev.precision, ev.device)
    x = _edge_values(sets, 5000, seed=11)
    fm = oracle.flatten(model)
    want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY64)
    got = ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(got, want), int(np.count_nonzero(got != want))
    assert dm.quantize_kernel()[0] == expect
    # the LDG-loaded kernel (feature-major rows) runs the same cell-table search
    xt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    assert np.array_equal(ev.predict_device(xt, layout=obt.Layout.FEATURE_MAJOR).cpu().numpy(), want)
    paths(quant_lut=0)
    assert np.array_equal(ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy(), want)
    assert np.array_equal(ev.predict_device(xt, layout=obt.Layout.FEATURE_MAJOR).cpu().numpy(), want)


@pytest.mark.parametrize("split", ["1", "0", "auto"])
def test_tail_split_behind_parameter_bank(paths, split):
    """A parameter-bank main region (7-bit compare, one lane per word) skips the tail
    split by default; forced on (tail_split=1) or off, predictions stay bit-exact."""
    if split != "auto":
        paths(tail_split=int(split))
    model = _model(48, 64, 40, 6, seed=77)
    n = 400001  # past one wave of the largest tile at F = 48
    x = _features(model, n, seed=78, specials=False)
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    got = obt.Evaluator(model).predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("D", [1, 3, 6, 8])
@pytest.mark.parametrize("B", [16, 200])
@pytest.mark.parametrize("n", [1, 127, 129, 5000])
def test_fanned_out_small_batch_apply(paths, D, B, n):
    """K2f (small batches: trees fanned out over a CTA's compute warps, the fold in tree
    order by the fold warps) bit-exact against the oracle in both precision families, and
    equal to the K2 / K2s path (fan=0)."""
    model = _model(21, B, 131, D, seed=D * 31 + B)  # 131 trees: a ragged last chunk
    x = _features(model, n, seed=n + D)
    fm = oracle.flatten(model)
    for strategy, prec in ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16)):
        paths(fan=1)
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy))
        got = ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
        want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
        assert np.array_equal(got, want), (strategy, int(np.count_nonzero(got != want)))
        paths(fan=0)
        assert np.array_equal(ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy(), want)


@pytest.mark.parametrize("D", [4, 8])
def test_fanned_out_eight_bit_compare(paths, D):
    """K2f with the 8-bit compare (more than 127 used borders on a feature)."""
    paths(fan=1)
    model = _model(2, 254, 160, D, seed=D)  # 320+ splits on each of 2 features: > 127 used borders
    x = _features(model, 2000, seed=D + 1)
    ev = obt.Evaluator(model)
    got = ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert ev.tables.device_model(ev.precision, ev.device).compare_mode == 8
    assert np.array_equal(got, oracle.evaluate_scalar(oracle.flatten(model), x))


def test_fanned_out_binary64_leaf_tables(paths):
    """K2f with binary64 leaf tables (leaves not exactly binary32)."""
    paths(fan=1)
    rng = np.random.default_rng(5)
    base = _model(13, 40, 97, 5, seed=5)
    trees = tuple(obt.ObliviousTree(depth=t.depth, splits=t.splits, leaf_values=rng.normal(0, 1, 1 << t.depth))
                  for t in base.trees)
    model = obt.ObliviousModel(base.float_features, trees, scale=1.5, bias=0.25)
    x = _features(model, 3000, seed=6)
    ev = obt.Evaluator(model)
    got = ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert ev.leaf_storage == "fp64"
    assert np.array_equal(got, oracle.evaluate_scalar(oracle.flatten(model), x))


def test_chained_parameter_bank_launches(paths):
    """Launch chaining (programmatic dependent launches with per-tile carry flags): a
    2000-tree depth-6 model folds over 3 parameter-bank launches of 2 waves each; the
    chained and the plainly serialised launches equal the oracle bit for bit."""
    model = _model(24, 64, 2000, 6, seed=91)
    n = 600001
    x = _features(model, n, seed=92, specials=False)
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    ev = obt.Evaluator(model)
    xd = torch.from_numpy(x).cuda()
    for pdl in ("1", "0", "1"):
        paths(pdl=int(pdl))
        got = ev.predict_device(xd).cpu().numpy()
        assert np.array_equal(got, want), (pdl, int(np.count_nonzero(got != want)))


# ---------------------------------------------------------------------------
# K2w (warp-specialised apply for wide feature sets), forced with the path option wide=1 on small
# models and chosen by default at config 4's shape.

def _wide_cases():
    for D in (1, 3, 6, 8):
        for B in (16, 200):          # 7-bit and 8-bit compares (200 used borders -> 8-bit)
            yield D, B


@pytest.mark.parametrize("D,B", list(_wide_cases()))
@pytest.mark.parametrize("n", [1, 255, 257, 256 * 148 + 77, 256 * 148 * 3 + 5])
def test_wide_apply_bit_exact(paths, D, B, n):
    paths(wide=1)
    paths(fan=0)
    model = _model(37, B, 53, D, seed=D * 13 + B)
    x = _features(model, n, seed=n % 1000 + D)
    fm = oracle.flatten(model)
    for strategy, prec in ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16)):
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy), device=0)
        got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
        assert np.array_equal(got, oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)), (strategy, D, B, n)


def test_wide_apply_mixed_depth_binary64_tables_and_layouts(paths):
    paths(wide=1)
    paths(fan=0)
    model = _mixed_depth_model(29, 60, 141, seed=5)
    x = _features(model, 40_000, seed=6)
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    ev = obt.Evaluator(model, device=0)
    assert ev.leaf_storage == "fp64"  # uniform(-1, 1) binary64 leaves are not fp32-exact
    assert np.array_equal(ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)), want)
    assert np.array_equal(ev.predict(obt.FeatureMatrix(np.ascontiguousarray(x.T), obt.Layout.FEATURE_MAJOR)), want)
    assert np.array_equal(ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy(), want)


def test_wide_apply_zero_trees_and_empty(paths):
    paths(wide=1)
    base = _model(9, 5, 1, 1, seed=2)
    model = obt.ObliviousModel(base.float_features, (), scale=2.0, bias=-0.75)
    x = _features(model, 1000, seed=3)
    ev = obt.Evaluator(model, device=0)
    assert np.array_equal(ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)), np.full(1000, -0.75))
    assert ev.predict(obt.FeatureMatrix(x[:0], obt.Layout.OBJECT_MAJOR)).shape == (0,)


def test_wide_apply_is_the_default_at_config4_shape():
    """Config 4's model (F = 500, 128 borders, depth 8) runs K2w by default; the first
    60k objects of a config-4 batch equal the oracle bit for bit (60k objects: past the K2f small-batch range)."""
    spec = synthetic.CONFIGS[4]
    model = synthetic.build_model(synthetic.WorkloadSpec(**{**spec.__dict__, "n_trees": 512}))
    x = synthetic.host_features(spec, n_objects=60_000, seed=9)
    ev = obt.Evaluator(model, device=0)
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, oracle.evaluate_scalar(oracle.flatten(model), x))


# ---------------------------------------------------------------------------
# Register/shuffle "permute" leaf selection (PERMUTE16 / PERMUTE64 of
# the reference, accumulate.py:116-159): K2 holds each 128-byte table one word per lane
# and selects leaves with SHFL instead of shared-memory gathers.

@pytest.mark.parametrize("D", [1, 3, 5, 6])
@pytest.mark.parametrize("B", [16, 200])
@pytest.mark.parametrize("source", [0, 1])
def test_permute_leaf_selection_bit_exact(paths, D, B, source):
    paths(leaf_select=1, fan=0, wide=0, tpw=1, desc_source=source)
    model = _model(23, B, 97, D, seed=D * 7 + B)
    x = _features(model, 70_001, seed=D + B)
    fm = oracle.flatten(model)
    for strategy, prec in ((obt.LeafStrategy.NAIVE16, oracle.BINARY16), (obt.LeafStrategy.NAIVE, oracle.BINARY64)):
        if prec == oracle.BINARY64 and D > 5:
            continue  # 64 binary32 leaves are two words per lane: gathers only
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy), device=0)
        got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
        assert np.array_equal(got, oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)), (strategy, D, B)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_predict_chunked_pageable_and_pinned(pinned):
    """Evaluator.predict on host arrays larger than one 128 MB chunk: pageable numpy input
    goes through the library's pinned staging buffers (host threads fill them while the
    previous chunk's DMA runs), pinned input straight to DMA; both equal the oracle."""
    model = _model(64, 32, 40, 6, seed=91)
    x = _features(model, 700_001, seed=92, specials=False)
    if pinned:
        xt = torch.from_numpy(x).pin_memory()
        x = xt.numpy()
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    ev = obt.Evaluator(model, device=0)
    got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
    assert np.array_equal(got, want)
    again = ev.predict(obt.FeatureMatrix(x[:300_001], obt.Layout.OBJECT_MAJOR))  # staging reused
    assert np.array_equal(again, want[:300_001])


# ---------------------------------------------------------------------------
# Single-output models whose F bytes per object do not fit K2's 128-object bucket tile
# (the reference has no feature limit; its own bench preset epsilon8k64 has F = 2,000):
# the record path, K5 with one output, staging only the bucket rows each tree reads.

@pytest.mark.parametrize("F,D,B", [(2000, 6, 64), (2500, 8, 200), (6000, 3, 16)])
def test_large_feature_count_single_output(F, D, B):
    model = _model(F, B, 45, D, seed=F + D)
    x = _features(model, 3001, seed=D)
    fm = oracle.flatten(model)
    for strategy, prec in ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16)):
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy), device=0)
        want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
        assert np.array_equal(ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)), want), (F, D, strategy)
        xt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
        assert np.array_equal(ev.predict_device(xt, layout=obt.Layout.FEATURE_MAJOR).cpu().numpy(), want)


@pytest.mark.parametrize("F,n", [(500, 620_001), (2000, 150_001)])
def test_cell_table_quantize_row_block_groups(paths, F, n):
    """K1L quantizing several consecutive 1024-row blocks per CTA with the chunk's tables
    staged once (F = 500: 4 blocks per CTA over 16 feature chunks; F = 2,000: 5 blocks
    over ~84 chunks), the last group partial: every row's prediction equals the oracle
    bit for bit (a 300-tree model reads most features of every chunk)."""
    paths(quant_lut=1)
    model = _model(F, 128, 300, 6, seed=F)
    x = _features(model, n, seed=F + 1)
    ev = obt.Evaluator(model, device=0)
    assert ev.quantize_kernel()[0].startswith("cells")
    oracle.set_threads(oracle.host_cores())
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    got = ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(got, want), int(np.count_nonzero(got != want))


def test_large_feature_count_binary64_leaves():
    """Leaves that are not binary32-exact keep binary64 records on the record path."""
    base = _model(3000, 32, 30, 6, seed=11)
    rng = np.random.default_rng(12)
    trees = tuple(obt.ObliviousTree(t.depth, t.splits, rng.uniform(-1, 1, t.leaf_values.size)) for t in base.trees)
    model = obt.ObliviousModel(base.float_features, trees, base.scale, base.bias)
    x = _features(model, 2000, seed=13)
    ev = obt.Evaluator(model, device=0)
    assert ev.leaf_storage == "fp64"
    assert np.array_equal(ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)), oracle.evaluate_scalar(oracle.flatten(model), x))


def test_random_model_shapes_fuzz():
    """60 seeded random shapes across every planner branch (F 1..3,000, depth 1..8, 1..254
    borders, 0..150 trees, batches 0..9,000, both precision families, both layouts,
    affine finalize): predictions equal the oracle bit for bit."""
    rng = np.random.default_rng(20261021)
    for case in range(60):
        F = int(rng.choice([1, 3, 4, 17, 50, 200, 501, 1203, 1800, 3000]))
        D = int(rng.integers(1, 9))
        B = int(rng.choice([1, 2, 7, 16, 64, 127, 128, 200, 254]))
        T = int(rng.choice([0, 1, 5, 33, 150]))
        n = int(rng.choice([0, 1, 129, 1000, 9000]))
        model = _model(F, B, T, D, seed=case) if T else obt.ObliviousModel(_model(F, B, 1, D, seed=case).float_features,
                                                                              (), 1.5, -0.25)
        x = _features(model, n, seed=case + 1000)
        fm = oracle.flatten(model)
        strategy, prec = ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16))[case % 2]
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy), device=0)
        want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
        layout = obt.Layout.OBJECT_MAJOR if case % 3 else obt.Layout.FEATURE_MAJOR
        xin = x if layout is obt.Layout.OBJECT_MAJOR else np.ascontiguousarray(x.T)
        got = ev.predict(obt.FeatureMatrix(xin, layout))
        assert got.shape == (n,)
        assert np.array_equal(got, want), (case, F, D, B, T, n, strategy, layout)


def test_random_shapes_and_forced_paths_fuzz(paths):
    """Seeded random shapes with a random forced planner choice each (descriptor source,
    lanes per word, K2w / K2f on or off, tail split, quantize search, permute selection):
    every combination the planner accepts equals the oracle."""
    rng = np.random.default_rng(77)
    options = [("desc_source", (0, 1)), ("tpw", (1, 2, 4)), ("wide", (0, 1)), ("fan", (0, 1)),
               ("tail_split", (0, 1)), ("quant_lut", (0, 1)), ("leaf_select", (1,)), ("pdl", (0,))]
    for case in range(40):
        F = int(rng.choice([4, 12, 50, 200, 500, 800]))
        D = int(rng.choice([2, 4, 6, 8]))
        B = int(rng.choice([7, 64, 128, 200]))
        T = int(rng.choice([20, 97, 700]))
        n = int(rng.choice([1, 300, 5000, 70_000]))
        name, values = options[int(rng.integers(len(options)))]
        value = int(rng.choice(values))
        paths(**{name: value})
        model = _model(F, B, T, D, seed=case + 500)
        x = _features(model, n, seed=case + 600)
        strategy, prec = ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16))[case % 2]
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy), device=0)
        want = oracle.evaluate_scalar(oracle.flatten(model), x, oracle.OBJECT_MAJOR, prec)
        got = ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(got, want), (case, F, D, B, T, n, name, value, strategy)
        paths(**{name: -1})


def test_random_multi_output_fuzz(paths):
    """Seeded random multi-output shapes (C 2..16, depth 1..12, F 1..3,000, both families
    where they apply, K4 / K5), against the multi-output restatement."""
    from paper_2211_00391_b200 import multiclass

    rng = np.random.default_rng(4242)
    for case in range(24):
        C = int(rng.choice([2, 3, 7, 10, 16]))
        D = int(rng.choice([1, 4, 7, 10, 12]))
        F = int(rng.choice([1, 9, 300, 3000]))
        B = int(rng.choice([3, 64, 254]))
        n = int(rng.choice([1, 513, 4097]))
        half = bool(case % 3 == 0) and C <= 10 and D <= 10
        paths(multi_staged=int(rng.integers(0, 2)) if not half else -1)
        spec = synthetic.WorkloadSpec("m", 1, F, B, 37, D, 0.01, n_outputs=C, cfg=5)
        arrays = synthetic.model_arrays(spec, seed=case + 900, affine=True)
        model = multiclass.from_arrays(arrays)
        x = _features(obt.ObliviousModel(tuple(obt.FloatFeatureBorders(f, b) for f, b in enumerate(arrays["borders"])),
                                          (), 1.0, 0.0), n, seed=case + 901)
        fm = oracle.FlatModel(np.stack(arrays["borders"]), np.full(F, B, np.int32), np.full(37, D, np.int32),
                              arrays["split_feature"], arrays["split_ordinal"], arrays["leaves"], model.scale, model.bias)
        cfg = obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16 if half else obt.LeafStrategy.NAIVE)
        want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY16 if half else oracle.BINARY64)
        ev = multiclass.MultiOutputEvaluator(model, config=cfg)
        got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
        assert np.array_equal(got, want.reshape(got.shape)), (case, C, D, F, B, n, half, ev.apply_kernel())


def test_quantize_stage_release_is_ordered_before_the_refill(paths):
    """Regression: K1L / K1t released a row stage with a plain mbarrier arrive right behind
    the loads that read it; under a busy shared-memory pipe the arrive overtook loads still
    queued and the tensor copy refilled the stage under them (F = 2,000: one warp's 128
    objects of one 8-feature step quantized from the next step's rows in ~20% of predicts).
    Repeated predicts with other work in between: the tiled bucket matrix K1L leaves in the
    workspace must equal K1t's every time, and the predictions the oracle's."""
    F, n = 2000, 150_001
    model = _model(F, 128, 300, 6, seed=F)
    x = _features(model, n, seed=F + 1)
    ev = obt.Evaluator(model, device=0)
    xd = torch.from_numpy(x).cuda()
    nbytes = ev.workspace_bytes(n)
    qbytes = -(-n // 2048) * 2048 * F  # the K5 record path's 2048-object bucket tiles
    assert qbytes <= nbytes
    paths(quant_lut=0)
    ws_ref = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    want = ev.predict_device(xd, workspace=ws_ref).clone()
    oracle.set_threads(oracle.host_cores())
    assert np.array_equal(want.cpu().numpy(), oracle.evaluate_scalar(oracle.flatten(model), x))
    paths(quant_lut=1)
    assert ev.quantize_kernel()[0].startswith("cells")
    for it in range(40):
        junk = torch.empty(64 << 20, dtype=torch.uint8, device="cuda").random_()  # disturb timing, evict L2
        ws = torch.full((nbytes,), 0xEE, dtype=torch.uint8, device="cuda")
        got = ev.predict_device(xd, workspace=ws)
        assert torch.equal(ws[:qbytes], ws_ref[:qbytes]), (it, int((ws[:qbytes] != ws_ref[:qbytes]).sum()))
        assert torch.equal(got, want), it
        del junk


@pytest.mark.parametrize("case", ["k2w", "k2w_fp16", "k2_chained", "k2s", "k5", "k5_fp16", "k5_one_output"])
def test_repeated_predicts_are_bit_identical(paths, case):
    """Every ring in these kernels is refilled by the copy engine behind the consumers'
    release; a release that overtakes its loads shows up as a run that differs.  Repeated
    predicts with other device work in between must reproduce the first run bit for bit
    (tests/stress/ runs the same check longer and at the full BASELINE sizes)."""
    from paper_2211_00391_b200 import multiclass

    W = synthetic.WorkloadSpec
    half = case.endswith("fp16")
    n = 200_000
    if case.startswith("k2w"):
        spec = W("t", n, 500, 128, 800, 8, 0.02, cfg=4)
    elif case == "k2_chained":
        spec = W("t", n, 200, 64, 2000, 6, 0.05, cfg=2)
    elif case == "k2s":
        spec, n = W("t", 100_000, 500, 128, 400, 8, 0.02, cfg=4), 100_000
        paths(wide=0)
    elif case == "k5_one_output":
        spec = W("t", n, 2000, 64, 400, 6, 0.05, cfg=6)
    else:
        spec, n = W("t", 100_000, 1000, 254, 100, 10, 0.01, n_outputs=10, cfg=5), 100_000
    if spec.n_outputs > 1:
        model = multiclass.from_arrays(synthetic.model_arrays(spec))
        cfg = obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16) if half else None
        ev = multiclass.MultiOutputEvaluator(model, device=0, config=cfg)
    else:
        model = synthetic.build_model(spec)
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16 if half else obt.LeafStrategy.NAIVE),
                           device=0)
    x = synthetic.device_features(spec, n_objects=n, device="cuda")
    first = ev.predict_device(x).clone()
    for it in range(12):
        junk = torch.empty(64 << 20, dtype=torch.uint8, device="cuda").random_()
        assert torch.equal(ev.predict_device(x), first), (case, it)
        del junk
