timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu42.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu42.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu42.log | head
for v in 1 0; do
OBT_LDG_LUT=$v python - <<'P'
import os, sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import synthetic
spec = synthetic.WorkloadSpec("cfg2fm", 1_000_000, 200, 64, 2000, 6, 0.05, cfg=2)
model = synthetic.build_model(spec, seed=2001)
x = synthetic.host_features(spec, seed=2002)
ev = obt.Evaluator(model)
xt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
for _ in range(3): ev.predict_device(xt, layout=obt.Layout.FEATURE_MAJOR)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(20): ev.predict_device(xt, layout=obt.Layout.FEATURE_MAJOR)
e.record(); torch.cuda.synchronize()
print("feature-major cfg2 LDG_LUT=%s: %.4f ms/predict" % (os.environ["OBT_LDG_LUT"], s.elapsed_time(e) / 20))
P
done
