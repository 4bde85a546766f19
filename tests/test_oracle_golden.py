"""Pin the CPU oracle (oracle/, a C restatement of the reference) to the reference.

Every expected value here was produced by running the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce them bit for bit.  CPU
only: no GPU is touched.
"""

from __future__ import annotations

import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import synthetic

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def known():
    return json.loads((GOLDEN / "known_answers.json").read_text())


def _digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_quantize_value_rules(known):
    for case in known["quantize_value"]:
        v = float(case["value"]) if case["value"] not in ("nan", "inf", "-inf") else float(case["value"])
        assert oracle.quantize_value(v, case["borders"]) == case["bucket"], case


def test_quantize_criterion1_10k_cases():
    g = np.load(GOLDEN / "criterion1.npz")
    pools, counts = g["pools"], g["pool_counts"]
    for k, v, e in zip(g["pool_idx"], g["values"], g["expected"]):
        assert oracle.quantize_value(float(np.float32(v)), pools[k, : counts[k]]) == e
    # the exhaustive matrix form agrees with the early-exit scalar form
    fm = oracle.FlatModel(pools, counts, np.zeros(0, np.int32), np.zeros((0, 0), np.int32),
                          np.zeros((0, 0), np.int32), np.zeros((0, 1, 1)), 1.0, 0.0)
    x = np.zeros((g["values"].size, pools.shape[0]), dtype=np.float32)
    x[np.arange(x.shape[0]), g["pool_idx"]] = g["values"].astype(np.float32)
    q = oracle.quantize(fm, x)
    assert np.array_equal(q[g["pool_idx"], np.arange(x.shape[0])], g["expected"])


def test_sign_split_and_all_inf(known):
    fm = oracle.FlatModel(np.array([[0.0]], np.float32), np.array([1], np.int32), np.zeros(0, np.int32),
                          np.zeros((0, 0), np.int32), np.zeros((0, 0), np.int32), np.zeros((0, 1, 1)), 1.0, 0.0)
    assert list(oracle.quantize(fm, np.array([[-1.0], [1.0]], np.float32))[0]) == known["sign_split_buckets"]
    fm3 = oracle.FlatModel(np.array([[0.0, 1.0, 2.0]], np.float32), np.array([3], np.int32), np.zeros(0, np.int32),
                           np.zeros((0, 0), np.int32), np.zeros((0, 0), np.int32), np.zeros((0, 1, 1)), 1.0, 0.0)
    assert list(oracle.quantize(fm3, np.full((5, 1), np.inf, np.float32))[0]) == known["all_inf_buckets"]


def test_half_conversion_matches_numpy_and_bank():
    g = np.load(GOLDEN / "half_bits.npz")
    for v, bits in zip(g["values"], g["raw_bits"]):
        assert oracle.half_bits(float(v)) == int(bits), v
    got, _ = oracle.half_bank(g["bank_values"])
    assert np.array_equal(got, g["bank_bits"])


def test_half_saturation(known):
    bits, count = oracle.half_bank(np.array([70000.0, -70000.0]))
    assert [int(b) for b in bits] == known["half_saturation"]["bits"]
    assert count == known["half_saturation"]["count"]


def test_half_saturation_of_infinite_leaves(known):
    """model.py:262-268: every +/-inf cast result is clamped and counted, infinite
    leaves included; the binary16 oracle then sums the finite clamps."""
    g = known["half_saturation_inf"]
    bits0, c0 = oracle.half_bank(np.array([np.inf, -np.inf, 70000.0, 1.0]))
    bits1, c1 = oracle.half_bank(np.array([-np.inf, 3.0]))
    assert [int(b) for b in bits0] + [int(b) for b in bits1] == g["bits"]
    assert c0 + c1 == g["count"]


def test_xoshiro_streams(known):
    for seed, expect in known["xoshiro"].items():
        if seed == "state_1234":
            continue
        r = oracle.Xoshiro(int(seed))
        assert [str(r.next_u64()) for _ in range(8)] == expect
    # known state (1, 2, 3, 4): outputs 11520 then 0
    r = oracle.Xoshiro(0)
    for i, v in enumerate((1, 2, 3, 4)):
        r._state[i] = v
    assert [str(r.next_u64()), str(r.next_u64())] == known["xoshiro"]["state_1234"]


def test_depth3_zero_trees_affine(known):
    d3 = known["depth3"]
    feats = tuple(obt.FloatFeatureBorders(i, np.array([0.5], np.float32)) for i in range(3))
    tree = obt.ObliviousTree(3, (obt.SplitCondition(0, 0), obt.SplitCondition(1, 0), obt.SplitCondition(2, 0)),
                             np.arange(10.0, 18.0))
    model = obt.ObliviousModel(feats, (tree,), 2.0, 1.0)
    fm = oracle.flatten(model)
    x = np.array(d3["x"], np.float32)
    assert oracle.leaf_indices(fm, oracle.quantize(fm, x))[0, 0] == d3["leaf_index"]
    assert oracle.evaluate_scalar(fm, x)[0] == d3["prediction"] == d3["oracle"]
    z = known["zero_trees"]
    zm = obt.ObliviousModel((obt.FloatFeatureBorders(0, np.array([0.5], np.float32)),), (), 3.0, -1.25)
    assert np.array_equal(oracle.evaluate_scalar(oracle.flatten(zm), np.array(z["x"], np.float32)), z["predictions"])
    a = known["affine"]
    am = obt.ObliviousModel((obt.FloatFeatureBorders(0, np.array([0.5], np.float32)),),
                            (obt.ObliviousTree(1, (obt.SplitCondition(0, 0),), np.array([2.0, 2.0])),), 0.5, 1.0)
    assert np.array_equal(oracle.evaluate_scalar(oracle.flatten(am), np.array(a["x"], np.float32)), a["predictions"])


@pytest.fixture(scope="module")
def corpus():
    return np.load(GOLDEN / "corpus.npz")


def test_corpus_regenerated_bit_identically_and_oracle_matches(corpus):
    """The reference's 100-model acceptance corpus: models and matrices regenerate
    bit-identically from the C restatement of synthetic.py, and evaluate_scalar of
    the restatement equals the reference's outputs in both precision families."""
    off = 0
    k = 0
    for i, (F, B, T, D, seed) in enumerate(corpus["specs"]):
        fm = oracle.synthetic_model(int(F), int(B), int(T), int(D), int(seed))
        assert oracle.model_digest(oracle.to_model(fm, obt)) == str(corpus["model_digests"][i])
        for batch in corpus["batch_sizes"]:
            x = oracle.feature_matrix(int(batch), int(F), int(seed) * 13 + int(batch), nan_fraction=0.02,
                                      inf_fraction=0.01)
            assert _digest(x) == str(corpus["matrix_digests"][k])
            a = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY64)
            b = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY16)
            assert np.array_equal(a, corpus["oracle64"][off: off + batch])
            assert np.array_equal(b, corpus["oracle16"][off: off + batch])
            # feature-major input gives the same bits
            assert np.array_equal(oracle.evaluate_scalar(fm, np.ascontiguousarray(x.T), oracle.FEATURE_MAJOR), a)
            off += int(batch)
            k += 1
    assert off == corpus["oracle64"].size


def test_corpus_buckets_and_leaf_indices(corpus):
    for name in corpus.files:
        if not name.startswith("q"):
            continue
        i = int(name[1:])
        F, B, T, D, seed = (int(v) for v in corpus["specs"][i])
        fm = oracle.synthetic_model(F, B, T, D, seed)
        x = oracle.feature_matrix(257, F, seed * 13 + 257, nan_fraction=0.02, inf_fraction=0.01)
        q = oracle.quantize(fm, x)
        assert np.array_equal(q, corpus[name])
        assert np.array_equal(oracle.leaf_indices(fm, q), corpus[f"i{i}"].astype(np.uint16))


def test_baseline_cfg1_against_reference_outputs():
    g = np.load(GOLDEN / "cfg1.npz")
    spec = synthetic.CONFIGS[1]
    model = synthetic.build_model(spec)
    x = synthetic.host_features(spec)
    assert oracle.model_digest(model) == str(g["model_digest"])
    assert _digest(x) == str(g["x_digest"])
    fm = oracle.flatten(model)
    assert np.array_equal(oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY64), g["pred64"])
    assert np.array_equal(oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY16), g["pred16"])


def test_deviation_metrics_fixture(known):
    d = known["deviation_metrics"]
    m = obt.deviation_metrics(np.array(d["a"]), np.array(d["b"]))
    assert (m.max_abs, m.mean_abs, m.median_abs) == (d["max_abs"], d["mean_abs"], d["median_abs"])
    assert abs(m.rms - d["rms"]) < 1e-15 and abs(m.rms - math.sqrt(12.5)) < 1e-15


def test_multi_output_restatement_matches_single_output_slices():
    """The depth>8 / multi-output restatement used for config 5 equals the C single-output
    evaluation on each output's slice (SURVEY.md 8c cross-check)."""
    rng = np.random.default_rng(3)
    F, B, T, D, C = 6, 9, 17, 5, 3
    base = oracle.synthetic_model(F, B, T, D, 123)
    leaves = rng.standard_normal((T, C, 1 << D))
    multi = oracle.FlatModel(base.borders, base.border_counts, base.depths, base.split_feature, base.split_ordinal,
                             leaves, 1.5, -0.25)
    x = oracle.feature_matrix(300, F, 9)
    got = oracle.evaluate_scalar(multi, x)
    for c in range(C):
        single = oracle.FlatModel(base.borders, base.border_counts, base.depths, base.split_feature,
                                  base.split_ordinal, leaves[:, c: c + 1, :].copy(), 1.5, -0.25)
        assert np.array_equal(got[:, c], oracle.evaluate_scalar(single, x))


def test_oracle_thread_count_overrides_environment():
    """The CPU baseline must use every host core even under torchrun (OMP_NUM_THREADS=1)."""
    before = oracle.max_threads()
    try:
        oracle.set_threads(2)
        assert oracle.max_threads() == 2
        oracle.set_threads(oracle.host_cores())
        assert oracle.max_threads() == oracle.host_cores()
    finally:
        oracle.set_threads(before)
