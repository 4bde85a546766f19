"""Single-output models whose F bytes per object do not fit K2's bucket tile (the paper's
epsilon model has F = 2,000): the record path (K5 with one output) against the oracle."""
import sys
import numpy as np
sys.path.insert(0, '.')
import oracle, paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import synthetic
for F, D, T in ((1500, 6, 300), (2000, 6, 300), (2000, 8, 200), (4000, 5, 100), (10000, 8, 50)):
    spec = synthetic.WorkloadSpec("eps", 5000, F, 64, T, D, 0.05, cfg=1)
    model = synthetic.build_model(spec, seed=3, affine=True)
    x = synthetic.sprinkle_specials(synthetic.host_features(spec, seed=4), [f.borders for f in model.float_features], seed=5)
    fm = oracle.flatten(model)
    for strat, prec in ((obt.LeafStrategy.NAIVE, oracle.BINARY64), (obt.LeafStrategy.NAIVE16, oracle.BINARY16)):
        try:
            ev = obt.Evaluator(model, obt.EvalConfig(strategy=strat), device=0)
            got = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
            want = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
            print(F, D, strat.value, "ok", np.array_equal(got, want), flush=True)
        except Exception as e:
            print(F, D, strat.value, "FAIL", type(e).__name__, str(e)[:200], flush=True)
