"""The drop-in surface on the host (no GPU): model types, validation texts, documents,
configuration errors, the binary16 bank and the C-ABI packing -- each held to what
the reference itself produced (tests/golden/errors.json, known_answers.json)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200.evaluate import ModelTables

GOLDEN = Path(__file__).resolve().parent / "golden"


def one_feature(borders):
    return (obt.FloatFeatureBorders(0, np.array(borders, dtype=np.float32)),)


BAD_MODELS = {
    "no_features": lambda: obt.ObliviousModel((), (), 1.0, 0.0),
    "index_mismatch": lambda: obt.ObliviousModel((obt.FloatFeatureBorders(3, np.array([0.5], np.float32)),), (), 1.0, 0.0),
    "nan_border": lambda: obt.ObliviousModel(one_feature([0.5, float("nan")]), (), 1.0, 0.0),
    "descending": lambda: obt.ObliviousModel(one_feature([1.0, 1.0]), (), 1.0, 0.0),
    "too_many_borders": lambda: obt.ObliviousModel(one_feature(list(np.arange(255.0))), (), 1.0, 0.0),
    "depth_0": lambda: obt.ObliviousModel(one_feature([0.5]), (obt.ObliviousTree(0, (), np.array([1.0])),), 1.0, 0.0),
    "depth_9": lambda: obt.ObliviousModel(one_feature([0.5]), (obt.ObliviousTree(9, (), np.zeros(512)),), 1.0, 0.0),
    "split_count": lambda: obt.ObliviousModel(
        one_feature([0.5]), (obt.ObliviousTree(2, (obt.SplitCondition(0, 0),), np.zeros(4)),), 1.0, 0.0),
    "leaf_count": lambda: obt.ObliviousModel(
        one_feature([0.5]), (obt.ObliviousTree(1, (obt.SplitCondition(0, 0),), np.zeros(3)),), 1.0, 0.0),
    "nan_leaf": lambda: obt.ObliviousModel(
        one_feature([0.5]), (obt.ObliviousTree(1, (obt.SplitCondition(0, 0),), np.array([0.0, np.nan])),), 1.0, 0.0),
    "feature_range": lambda: obt.ObliviousModel(
        one_feature([0.5]), (obt.ObliviousTree(1, (obt.SplitCondition(4, 0),), np.zeros(2)),), 1.0, 0.0),
    "ordinal_range": lambda: obt.ObliviousModel(
        one_feature([0.5]), (obt.ObliviousTree(1, (obt.SplitCondition(0, 3),), np.zeros(2)),), 1.0, 0.0),
}


@pytest.fixture(scope="module")
def errors():
    return json.loads((GOLDEN / "errors.json").read_text())


def test_validation_texts_match_reference(errors):
    for case in errors["validate"]:
        assert obt.validate_model(BAD_MODELS[case["name"]]()) == case["errors"], case["name"]


def test_require_valid_raises_value_error():
    with pytest.raises(ValueError, match="invalid model: "):
        obt.require_valid(BAD_MODELS["descending"]())
    with pytest.raises(ValueError, match="invalid model"):
        ModelTables(BAD_MODELS["nan_leaf"]())


def test_document_errors_match_reference(errors):
    for case in errors["format"]:
        if case["ok"]:
            m = obt.deserialize_model(case["text"])
            assert oracle.model_digest(m) == case["digest"]
            continue
        with pytest.raises(obt.ModelFormatError) as info:
            obt.deserialize_model(case["text"])
        assert type(info.value).__name__ == case["type"] == "ModelFormatError"
        assert str(info.value) == case["message"], case["name"]
        assert isinstance(info.value, ValueError)


def test_round_trip_bit_exact(tmp_path):
    for seed in range(40):
        fm = oracle.synthetic_model(1 + seed % 7, 1 + seed % 11, seed % 9, 1 + seed % 8, 5000 + seed)
        model = oracle.to_model(fm, obt)
        text = obt.serialize_model(model)
        assert obt.deserialize_model(text) == model
    special = obt.ObliviousModel(one_feature([-0.0, 1e-45, 3.4e38]),
                                 (obt.ObliviousTree(1, (obt.SplitCondition(0, 2),), np.array([-0.0, 5e-324])),),
                                 scale=float.fromhex("0x1.0000000000001p+0"), bias=-0.0)
    path = tmp_path / "m.json"
    obt.save_model(special, str(path))
    back = obt.load_model(str(path))
    assert back == special
    assert np.signbit(back.trees[0].leaf_values[0]) and np.signbit(back.bias)


def test_eval_config_validation():
    obt.EvalConfig().validate()
    with pytest.raises(ValueError, match="block size"):
        obt.EvalConfig(block_size=100).validate()
    with pytest.raises(ValueError, match="incompatible"):
        obt.EvalConfig(strategy=obt.LeafStrategy.PERMUTE64, width=obt.VectorWidth.W256).validate()
    obt.EvalConfig(block_size=64, width=obt.VectorWidth.W512).validate()  # group 64 fits a 64 block
    assert obt.LeafStrategy.NAIVE16.precision is obt.LeafPrecision.BINARY16
    assert obt.LeafStrategy.GATHER.precision is obt.LeafPrecision.BINARY64


def test_feature_matrix_layouts():
    x = np.arange(12, dtype=np.float32).reshape(4, 3)
    om = obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)
    fm = om.transposed()
    assert (om.n_objects, om.n_features) == (4, 3) == (fm.n_objects, fm.n_features)
    assert np.array_equal(om.feature_values(1, 0, 4), fm.feature_values(1, 0, 4))
    with pytest.raises(ValueError, match="2-D"):
        obt.FeatureMatrix(np.zeros(3, np.float32), obt.Layout.OBJECT_MAJOR)


def test_binary16_bank_matches_reference_bits(known=None):
    g = np.load(GOLDEN / "half_bits.npz")
    for v, bits in zip(g["bank_values"][:64], g["bank_bits"][:64]):
        m = obt.ObliviousModel(one_feature([0.5]), (obt.ObliviousTree(1, (obt.SplitCondition(0, 0),), np.array([v, v])),),
                               1.0, 0.0)
        bank = obt.build_leaf_bank(m, obt.LeafPrecision.BINARY16)
        assert int(bank.table(0)[0].view(np.uint16)) == int(bits)
    sat = obt.ObliviousModel(one_feature([0.5]), (obt.ObliviousTree(1, (obt.SplitCondition(0, 0),),
                                                                     np.array([70000.0, -70000.0])),), 1.0, 0.0)
    bank = obt.build_leaf_bank(sat, obt.LeafPrecision.BINARY16)
    assert bank.saturation_count == 2 and bank.table(0).size == 32 and bank.values.flags.writeable is False


def test_binary16_bank_saturates_infinite_leaves():
    import json

    g = json.loads((GOLDEN / "known_answers.json").read_text())["half_saturation_inf"]
    m = _inf_leaf_model()
    bank = obt.build_leaf_bank(m, obt.LeafPrecision.BINARY16)
    got = [int(v) for v in bank.table(0)[:4].view(np.uint16)] + [int(v) for v in bank.table(1)[:2].view(np.uint16)]
    assert got == g["bits"] and bank.saturation_count == g["count"]


def _inf_leaf_model():
    return obt.ObliviousModel(
        one_feature([0.5]),
        (obt.ObliviousTree(2, (obt.SplitCondition(0, 0), obt.SplitCondition(0, 0)),
                           np.array([np.inf, -np.inf, 70000.0, 1.0])),
         obt.ObliviousTree(1, (obt.SplitCondition(0, 0),), np.array([-np.inf, 3.0]))), 1.0, 0.0)


def test_model_tables_packing_for_the_c_abi():
    trees = (
        obt.ObliviousTree(2, (obt.SplitCondition(0, 1), obt.SplitCondition(1, 0)), np.array([1.0, 2.0, 3.0, 4.0])),
        obt.ObliviousTree(1, (obt.SplitCondition(1, 2),), np.array([-1.0, 0.5])),
    )
    feats = (obt.FloatFeatureBorders(0, np.array([0.0, 1.0], np.float32)),
             obt.FloatFeatureBorders(1, np.array([-1.0, 0.0, 2.0], np.float32)))
    t = ModelTables(obt.ObliviousModel(feats, trees, 1.0, 0.0))
    p = t.packed()
    assert t.max_depth == 2
    assert p["split_ordinal"].tolist() == [[1, 0], [2, 255]]  # 255 = sentinel (reference evaluate.py:32)
    assert p["split_feature"].tolist() == [[0, 1], [1, 0]]
    assert p["border_counts"].tolist() == [2, 3]
    assert np.isinf(p["borders"][0, 2])
    assert p["leaves"].tolist() == [[1.0, 2.0, 3.0, 4.0], [-1.0, 0.5, 0.0, 0.0]]
    assert p["leaves_f16"].dtype == np.uint16


def test_deviation_and_flip_metrics():
    m = obt.deviation_metrics(np.array([1.0]), np.array([1.5]))
    assert (m.max_abs, m.mean_abs, m.median_abs, m.rms) == (0.5, 0.5, 0.5, 0.5)
    assert obt.classification_flip_count(np.array([0.1]), np.array([-0.1]), 0.0) == 1
    with pytest.raises(ValueError):
        obt.deviation_metrics(np.zeros(0), np.zeros(0))


def test_evaluator_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    model = obt.ObliviousModel(one_feature([0.5]), (), 1.0, 0.0)
    with pytest.raises(obt.NativeUnavailable):
        obt.Evaluator(model)
    with pytest.raises(ValueError, match="block size"):  # config errors come first, like the reference
        obt.Evaluator(model, obt.EvalConfig(block_size=3))
