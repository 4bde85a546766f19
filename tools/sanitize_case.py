"""Small end-to-end case for compute-sanitizer: every kernel family once (quantize
full/used tables, K2 apply, K2s depth-split, K4 multi-output, leaf-index dump)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import _native  # noqa: E402
from paper_2211_00391_b200 import multiclass, stages, synthetic  # noqa: E402

spec = synthetic.WorkloadSpec("s", 3000, 40, 64, 96, 6, 0.05, cfg=2)
model = synthetic.build_model(spec, seed=1, affine=True)
x = synthetic.host_features(spec, seed=2)
xd = torch.from_numpy(x).cuda()
ev = obt.Evaluator(model)
a = ev.predict(obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR))
b = ev.predict_device(xd).cpu().numpy()
assert np.array_equal(a, b)
stages.quantize(model, xd)
stages.leaf_indices(model, xd)
_native.set_path_option("tpw", 2)
ev2 = obt.Evaluator(obt.ModelTables(model))
assert np.array_equal(ev2.predict_device(xd).cpu().numpy(), a)
ev16 = obt.Evaluator(model, obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16))
ev16.predict_device(xd)
mspec = synthetic.WorkloadSpec("m", 2000, 30, 100, 40, 10, 0.01, n_outputs=10, cfg=5)
mm = multiclass.from_arrays(synthetic.model_arrays(mspec, seed=3))
multiclass.MultiOutputEvaluator(mm).predict_device(torch.randn(2000, 30, device="cuda"))
torch.cuda.synchronize()
print("sanitize case ok")
