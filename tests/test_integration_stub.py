"""INTEGRATION.md Route 2: the ctypes stub a maintainer would add to the reference
package, executed verbatim against the built library.

Run twice: against the REAL reference package when it is installed in baseline/_ref
(pip install --target baseline/_ref, git-ignored, travels to the GPU box with the
repo) -- its own ModelTables, ObliviousModel, FeatureMatrix and EvalConfig feed the
stub -- and against this package's restatement of `obtree.evaluate.ModelTables` (same
attributes, evaluate.py:138-166), which needs nothing but this repo."""

from __future__ import annotations

import re
import sys
import types
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2211_00391_b200 as obt
import importlib

from paper_2211_00391_b200 import _native, synthetic

evaluate_module = importlib.import_module("paper_2211_00391_b200.evaluate")

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


REF_PKG = ROOT / "baseline" / "_ref"


def _real_obtree():
    if not (REF_PKG / "obtree").exists():
        pytest.skip("reference package not installed in baseline/_ref")
    if str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))
    import obtree

    return obtree


def _stub_namespace_real():
    """The stub's code, importing the real reference package."""
    _real_obtree()
    text = (ROOT / "INTEGRATION.md").read_text()
    route2 = text[text.index("## Route 2"):]
    code = re.search(r"```python\n(.*?)```", route2, re.S).group(1)
    lib = str(_native.library_path())
    code = code.replace('ctypes.CDLL("libobtree_b200.so")', f"ctypes.CDLL({lib!r})")
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md:route2", "exec"), ns)
    return ns


def test_integration_stub_with_the_real_reference_package():
    """The maintainer's view: reference model objects and matrices in, GPU scores out,
    equal to the reference's own Evaluator (NAIVE and NAIVE16) bit for bit."""
    _native.require_gpu()
    obtree = _real_obtree()
    import bench

    ns = _stub_namespace_real()
    spec = synthetic.WorkloadSpec("stub", 2000, 19, 40, 60, 7, 0.1, cfg=1)
    model = bench.reference_model(synthetic.build_model(spec, seed=21, affine=True))
    assert type(model).__module__.startswith("obtree")
    x = synthetic.sprinkle_specials(synthetic.host_features(spec, seed=22),
                                    [ff.borders for ff in model.float_features], seed=23)
    for layout in (obtree.Layout.OBJECT_MAJOR, obtree.Layout.FEATURE_MAJOR):
        m = obtree.FeatureMatrix(x if layout is obtree.Layout.OBJECT_MAJOR else np.ascontiguousarray(x.T), layout)
        for strategy in (obtree.LeafStrategy.NAIVE, obtree.LeafStrategy.NAIVE16):
            cfg = obtree.EvalConfig(strategy=strategy)
            got = ns["GpuEvaluator"](importlib.import_module("obtree.evaluate").ModelTables(model), cfg).predict(m)
            want = obtree.Evaluator(model, cfg).predict(m)
            assert np.array_equal(got, want), (layout, strategy)


def _stub_namespace():
    text = (ROOT / "INTEGRATION.md").read_text()
    route2 = text[text.index("## Route 2"):]
    code = re.search(r"```python\n(.*?)```", route2, re.S).group(1)
    lib = str(_native.library_path())
    code = code.replace('ctypes.CDLL("libobtree_b200.so")', f"ctypes.CDLL({lib!r})")
    fake = types.ModuleType("obtree")
    fake_eval = types.ModuleType("obtree.evaluate")
    fake_eval.ModelTables = evaluate_module.ModelTables
    fake.evaluate = fake_eval
    saved = {k: sys.modules.get(k) for k in ("obtree", "obtree.evaluate")}
    sys.modules["obtree"], sys.modules["obtree.evaluate"] = fake, fake_eval
    try:
        ns: dict = {}
        exec(compile(code, "INTEGRATION.md:route2", "exec"), ns)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
    return ns


@pytest.mark.parametrize("layout", [obt.Layout.OBJECT_MAJOR, obt.Layout.FEATURE_MAJOR])
def test_integration_stub_predicts_bit_exact(layout):
    _native.require_gpu()
    ns = _stub_namespace()
    spec = synthetic.WorkloadSpec("stub", 3000, 21, 40, 80, 6, 0.1, cfg=1)
    model = synthetic.build_model(spec, seed=11, affine=True)
    x = synthetic.sprinkle_specials(synthetic.host_features(spec, seed=12),
                                    [ff.borders for ff in model.float_features], seed=13)
    fm = oracle.flatten(model)
    xin = x if layout is obt.Layout.OBJECT_MAJOR else np.ascontiguousarray(x.T)
    for strategy, prec in ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16)):
        ev = ns["GpuEvaluator"](model, obt.EvalConfig(strategy=strategy))
        got = ev.predict(obt.FeatureMatrix(xin, layout))
        assert np.array_equal(got, oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec))
    with pytest.raises(ValueError, match="matrix has 20 features, model expects 21"):
        ns["GpuEvaluator"](model).predict(obt.FeatureMatrix(x[:, :20].copy(), obt.Layout.OBJECT_MAJOR))
