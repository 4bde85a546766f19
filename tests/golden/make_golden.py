#!/usr/bin/env python
"""Generate the golden fixtures under tests/golden by running the REFERENCE package.

Runs only where the reference is importable (this build container:
PYTHONPATH=/root/reference/pkg/src).  The GPU box never runs this script; it only
reads the committed fixtures.  Every fixture is produced by calling the reference's
own public functions (obtree.*), so the oracle restatement in oracle/ and the product
package are pinned to the reference's behaviour, not to a re-derivation of it.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import obtree  # noqa: E402  (the reference package)
from obtree import (  # noqa: E402
    EvalConfig,
    FeatureMatrix,
    FloatFeatureBorders,
    Layout,
    LeafIndexVector,
    LeafPrecision,
    LeafStrategy,
    ObliviousModel,
    ObliviousTree,
    QuantizedBlock,
    SplitCondition,
    SyntheticSpec,
    VectorWidth,
    Xoshiro256StarStar,
    build_leaf_bank,
    compute_leaf_indices,
    deserialize_model,
    deviation_metrics,
    evaluate,
    evaluate_scalar,
    generate_feature_matrix,
    generate_synthetic_model,
    quantize_block,
    quantize_value,
    serialize_model,
    validate_model,
)
from obtree.evaluate import Evaluator, ModelTables  # noqa: E402

BATCH_SIZES = (1, 7, 31, 32, 33, 100, 128, 257)


def digest_model(model) -> str:
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


def digest_array(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def one_feature(borders):
    return (FloatFeatureBorders(0, np.array(borders, dtype=np.float32)),)


def known_answers() -> dict:
    out = {}
    # stage-1 value rules (the reference's quantize_value on its documented cases)
    cases = [
        (0.7, [0.5]), (2.0, [1.0, 2.0, 3.0]), (float("nan"), [-10.0, 0.0, 10.0]),
        (float("inf"), [0.0, 1.0]), (float("-inf"), [0.0, 1.0]), (5.0, []),
        (0.0, [-0.0]), (-0.0, [0.0]), (1e-45, [0.0]), (-1e-45, [0.0]), (3.0, [1.0, 2.0, 3.0]),
    ]
    out["quantize_value"] = [
        {"value": repr(v), "borders": b, "bucket": int(quantize_value(v, np.array(b, dtype=np.float32)))}
        for v, b in cases
    ]
    # sign split on a zero border, through quantize_block
    m = FeatureMatrix(np.array([[-1.0], [1.0]], dtype=np.float32), Layout.OBJECT_MAJOR)
    blk = QuantizedBlock(1, 64)
    quantize_block(m, (0, 2), [np.array([0.0], dtype=np.float32)], VectorWidth.W512, blk)
    out["sign_split_buckets"] = [int(v) for v in blk.quantiles[0, :2]]
    # all +inf values -> bucket = B
    vals = np.full((5, 1), np.inf, dtype=np.float32)
    blk = QuantizedBlock(1, 64)
    quantize_block(FeatureMatrix(vals, Layout.OBJECT_MAJOR), (0, 5), [np.array([0.0, 1.0, 2.0], np.float32)],
                   VectorWidth.W512, blk)
    out["all_inf_buckets"] = [int(v) for v in blk.quantiles[0, :5]]
    # depth-3 index fixture: conditions (1, 0, 1) -> leaf 5
    feats = tuple(FloatFeatureBorders(i, np.array([0.5], dtype=np.float32)) for i in range(3))
    tree = ObliviousTree(3, (SplitCondition(0, 0), SplitCondition(1, 0), SplitCondition(2, 0)), np.arange(10.0, 18.0))
    model = ObliviousModel(feats, (tree,), scale=2.0, bias=1.0)
    x = np.array([[1.0, 0.0, 1.0]], dtype=np.float32)
    blk = QuantizedBlock(3, 64)
    quantize_block(FeatureMatrix(x, Layout.OBJECT_MAJOR), (0, 1), model.float_features, VectorWidth.W512, blk)
    idx = LeafIndexVector(64)
    compute_leaf_indices(blk, tree, VectorWidth.W512, idx)
    out["depth3"] = {
        "x": x.tolist(), "leaf_index": int(idx.indices[0]),
        "prediction": float(evaluate(model, FeatureMatrix(x, Layout.OBJECT_MAJOR))[0]),
        "oracle": float(evaluate_scalar(model, FeatureMatrix(x, Layout.OBJECT_MAJOR))[0]),
    }
    # zero trees -> bias; one constant tree -> affine
    zero = ObliviousModel(one_feature([0.5]), (), scale=3.0, bias=-1.25)
    xm = generate_feature_matrix(17, 1, seed=1)
    out["zero_trees"] = {"bias": -1.25, "predictions": evaluate(zero, xm).tolist(), "x": xm.values.tolist()}
    const = ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(0, 0),), np.array([2.0, 2.0])),),
                           scale=0.5, bias=1.0)
    xm = generate_feature_matrix(9, 1, seed=2)
    out["affine"] = {"predictions": evaluate(const, xm).tolist(), "x": xm.values.tolist()}
    # binary16 bank: saturation and exact values
    sat = ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(0, 0),), np.array([70000.0, -70000.0])),),
                         1.0, 0.0)
    bank = build_leaf_bank(sat, LeafPrecision.BINARY16)
    out["half_saturation"] = {"bits": [int(v) for v in bank.table(0)[:2].view(np.uint16)],
                              "count": int(bank.saturation_count)}
    # infinite leaves are saturated and counted too (model.py:262-268 tests isinf on the
    # cast values); the NAIVE16 pipeline then sums finite +/-65504 instead of +/-inf
    inf_model = ObliviousModel(one_feature([0.5]),
                               (ObliviousTree(2, (SplitCondition(0, 0), SplitCondition(0, 0)),
                                              np.array([np.inf, -np.inf, 70000.0, 1.0])),
                                ObliviousTree(1, (SplitCondition(0, 0),), np.array([-np.inf, 3.0]))), 1.0, 0.0)
    bank = build_leaf_bank(inf_model, LeafPrecision.BINARY16)
    xm = FeatureMatrix(np.array([[0.25], [0.75], [np.nan], [0.5]], np.float32), Layout.OBJECT_MAJOR)
    out["half_saturation_inf"] = {
        "bits": [int(v) for v in bank.table(0)[:4].view(np.uint16)] + [int(v) for v in bank.table(1)[:2].view(np.uint16)],
        "count": int(bank.saturation_count), "x": [0.25, 0.75, None, 0.5],
        "predictions_naive16": evaluate(inf_model, xm, EvalConfig(strategy=LeafStrategy.NAIVE16)).tolist(),
        "predictions_scalar16": evaluate_scalar(inf_model, xm, LeafPrecision.BINARY16).tolist()}
    # xoshiro streams (seed expansion + update rule)
    streams = {}
    for seed in (0, 1, 99, 90125, 2**64 - 1):
        r = Xoshiro256StarStar(seed)
        streams[str(seed)] = [str(r.next_u64()) for _ in range(8)]
    r = Xoshiro256StarStar(0)
    r._s = [1, 2, 3, 4]
    streams["state_1234"] = [str(r.next_u64()), str(r.next_u64())]
    out["xoshiro"] = streams
    # deviation metrics fixture
    d = deviation_metrics(np.array([0.0, 0.0]), np.array([3.0, 4.0]))
    out["deviation_metrics"] = {"a": [0.0, 0.0], "b": [3.0, 4.0], "max_abs": d.max_abs, "mean_abs": d.mean_abs,
                                "median_abs": d.median_abs, "rms": d.rms}
    return out


def criterion1_cases():
    """10,000 (value, borders) cases built exactly like the reference's acceptance
    criterion 1, answered by the reference's quantize_value."""
    rng = Xoshiro256StarStar(40001)
    pools = []
    for p in range(50):
        count = 254 if p < 3 else 1 + rng.below(64)
        seen = set()
        while len(seen) < count:
            seen.add(float(np.float32(rng.uniform(-2.0, 2.0))))
        pools.append(sorted(seen))
    specials = (math.nan, math.inf, -math.inf)
    pool_idx, values, expected = [], [], []
    for i in range(10_000):
        k = rng.below(len(pools))
        borders = pools[k]
        roll = rng.below(10)
        if roll == 0:
            value = specials[i % 3]
        elif roll == 1:
            value = borders[rng.below(len(borders))]
        else:
            value = float(np.float32(rng.uniform(-3.0, 3.0)))
        pool_idx.append(k)
        values.append(value)
        expected.append(quantize_value(value, borders))
    padded = np.full((len(pools), 254), np.inf, dtype=np.float32)
    counts = np.array([len(p) for p in pools], dtype=np.int32)
    for i, p in enumerate(pools):
        padded[i, : len(p)] = p
    return {"pools": padded, "pool_counts": counts, "pool_idx": np.array(pool_idx, np.int32),
            "values": np.array(values, np.float64), "expected": np.array(expected, np.int32)}


def half_bits():
    """binary64 -> binary16 bank conversion (numpy, the reference's arithmetic)."""
    rng = np.random.default_rng(7)
    exps = rng.uniform(-30, 18, size=4000)
    vals = np.sign(rng.standard_normal(4000)) * 2.0**exps
    special = np.array([0.0, -0.0, 1.0, -2.0, 65504.0, 2.0**-24, 2.0**-25, 1024.5, 65519.0, 65520.0,
                        2.0**-14, 2.0**-15 * 3, 5.960464477539063e-08, 1e-300, -1e300, 0.1, 0.2], np.float64)
    vals = np.concatenate([special, vals])
    with np.errstate(over="ignore"):
        raw = vals.astype(np.float16).view(np.uint16)
    model_leaves = vals[np.isfinite(vals)]
    sat_bits = []
    for v in model_leaves[:512]:
        m = ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(0, 0),), np.array([v, v])),), 1.0, 0.0)
        sat_bits.append(int(build_leaf_bank(m, LeafPrecision.BINARY16).table(0)[0].view(np.uint16)))
    return {"values": vals, "raw_bits": raw, "bank_values": model_leaves[:512], "bank_bits": np.array(sat_bits, np.uint16)}


def corpus():
    """The reference acceptance corpus (test_acceptance.py corpus_spec): 100 models x 8
    batch sizes with NaN 2% / inf 1% sprinkles, answered by evaluate_scalar in both
    precision families; the reference Evaluator's default NAIVE and NAIVE16 runs are
    checked equal to them here (the reference's own oracle == pipeline property)."""
    shape_rng = Xoshiro256StarStar(90125)
    specs, model_digests, matrix_digests, o64, o16 = [], [], [], [], []
    quant, idx = {}, {}
    for index in range(100):
        spec = SyntheticSpec(
            n_features=1 + shape_rng.below(50),
            borders_per_feature=1 + shape_rng.below(64),
            n_trees=1 + shape_rng.below(200),
            depth=1 + shape_rng.below(8),
            seed=31_000 + index,
        )
        model = generate_synthetic_model(spec)
        tables = ModelTables(model)
        ev64 = Evaluator(tables, EvalConfig())
        ev16 = Evaluator(tables, EvalConfig(block_size=512, strategy=LeafStrategy.NAIVE16))
        specs.append([spec.n_features, spec.borders_per_feature, spec.n_trees, spec.depth, spec.seed])
        model_digests.append(digest_model(model))
        for batch in BATCH_SIZES:
            om = generate_feature_matrix(batch, model.n_features, seed=spec.seed * 13 + batch,
                                         nan_fraction=0.02, inf_fraction=0.01)
            a = evaluate_scalar(model, om)
            b = evaluate_scalar(model, om, LeafPrecision.BINARY16)
            assert np.array_equal(ev64.predict(om), a)
            assert np.array_equal(ev16.predict(om), b)
            matrix_digests.append(digest_array(om.values))
            o64.append(a)
            o16.append(b)
            if index < 12 and batch == 257:
                blk = QuantizedBlock(model.n_features, 512)
                quantize_block(om, (0, batch), model.float_features, VectorWidth.W512, blk)
                quant[f"q{index}"] = blk.quantiles[:, :batch].copy()
                rows = []
                for tree in model.trees:
                    liv = LeafIndexVector(512)
                    compute_leaf_indices(blk, tree, VectorWidth.W512, liv)
                    rows.append(liv.indices[:batch].copy())
                idx[f"i{index}"] = np.array(rows, dtype=np.uint8)
    return {"specs": np.array(specs, np.int64), "model_digests": np.array(model_digests),
            "matrix_digests": np.array(matrix_digests), "oracle64": np.concatenate(o64),
            "oracle16": np.concatenate(o16), "batch_sizes": np.array(BATCH_SIZES), **quant, **idx}


def baseline_cfg1():
    """BASELINE config 1 (this repo's seeded generator) answered by the reference."""
    from paper_2211_00391_b200 import synthetic

    spec = synthetic.CONFIGS[1]
    ours = synthetic.build_model(spec)
    ref_model = ObliviousModel(
        tuple(FloatFeatureBorders(f.feature_index, f.borders) for f in ours.float_features),
        tuple(ObliviousTree(t.depth, tuple(SplitCondition(s.feature_index, s.border_ordinal) for s in t.splits),
                            t.leaf_values) for t in ours.trees),
        ours.scale, ours.bias)
    x = synthetic.host_features(spec)
    fm = FeatureMatrix(x, Layout.OBJECT_MAJOR)
    a = evaluate(ref_model, fm)
    b = evaluate(ref_model, fm, EvalConfig(block_size=512, strategy=LeafStrategy.NAIVE16))
    assert np.array_equal(a, evaluate_scalar(ref_model, fm))
    assert np.array_equal(b, evaluate_scalar(ref_model, fm, LeafPrecision.BINARY16))
    return {"model_digest": np.array(digest_model(ref_model)), "x_digest": np.array(digest_array(x)),
            "pred64": a, "pred16": b}


def error_texts():
    """Validation and document errors exactly as the reference words them."""
    out = {"validate": [], "format": []}
    bad_models = {
        "no_features": ObliviousModel((), (), 1.0, 0.0),
        "index_mismatch": ObliviousModel((FloatFeatureBorders(3, np.array([0.5], np.float32)),), (), 1.0, 0.0),
        "nan_border": ObliviousModel(one_feature([0.5, float("nan")]), (), 1.0, 0.0),
        "descending": ObliviousModel(one_feature([1.0, 1.0]), (), 1.0, 0.0),
        "too_many_borders": ObliviousModel(one_feature(list(np.arange(255.0))), (), 1.0, 0.0),
        "depth_0": ObliviousModel(one_feature([0.5]), (ObliviousTree(0, (), np.array([1.0])),), 1.0, 0.0),
        "depth_9": ObliviousModel(one_feature([0.5]), (ObliviousTree(9, (), np.zeros(512)),), 1.0, 0.0),
        "split_count": ObliviousModel(one_feature([0.5]), (ObliviousTree(2, (SplitCondition(0, 0),), np.zeros(4)),), 1.0, 0.0),
        "leaf_count": ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(0, 0),), np.zeros(3)),), 1.0, 0.0),
        "nan_leaf": ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(0, 0),), np.array([0.0, np.nan])),), 1.0, 0.0),
        "feature_range": ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(4, 0),), np.zeros(2)),), 1.0, 0.0),
        "ordinal_range": ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(0, 3),), np.zeros(2)),), 1.0, 0.0),
    }
    for name, m in bad_models.items():
        out["validate"].append({"name": name, "errors": validate_model(m)})
    good = ObliviousModel(one_feature([0.5]), (ObliviousTree(1, (SplitCondition(0, 0),), np.array([-1.0, 2.0])),), 1.0, 0.0)
    doc = json.loads(serialize_model(good))
    variants = {"valid": json.dumps(doc), "not_json": "{\"float_features\": [", "not_object": "[1, 2]"}
    for key in ("float_features", "trees", "scale_hex", "bias_hex"):
        d = json.loads(json.dumps(doc))
        del d[key]
        variants[f"missing_{key}"] = json.dumps(d)
    d = json.loads(json.dumps(doc)); d["scale_hex"] = "3ff0"; variants["short_hex"] = json.dumps(d)
    d = json.loads(json.dumps(doc)); d["bias_hex"] = "zzzzzzzzzzzzzzzz"; variants["bad_hex"] = json.dumps(d)
    d = json.loads(json.dumps(doc)); d["trees"][0]["depth"] = True; variants["bool_depth"] = json.dumps(d)
    d = json.loads(json.dumps(doc)); d["trees"][0]["splits"][0]["border"] = 5; variants["invalid_model"] = json.dumps(d)
    d = json.loads(json.dumps(doc)); d["float_features"][0]["borders_hex"] = "3f000000"; variants["not_list"] = json.dumps(d)
    for name, text in variants.items():
        try:
            m = deserialize_model(text)
            out["format"].append({"name": name, "text": text, "ok": True, "digest": digest_model(m)})
        except ValueError as exc:
            out["format"].append({"name": name, "text": text, "ok": False, "type": type(exc).__name__,
                                  "message": str(exc)})
    return out


def main():
    (HERE / "known_answers.json").write_text(json.dumps(known_answers(), indent=1))
    np.savez_compressed(HERE / "criterion1.npz", **criterion1_cases())
    np.savez_compressed(HERE / "half_bits.npz", **half_bits())
    np.savez_compressed(HERE / "corpus.npz", **corpus())
    np.savez_compressed(HERE / "cfg1.npz", **baseline_cfg1())
    (HERE / "errors.json").write_text(json.dumps(error_texts(), indent=1))
    print("reference", obtree.__version__, "fixtures written to", HERE)


if __name__ == "__main__":
    main()
