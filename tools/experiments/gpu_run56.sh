python - <<'P'
import sys, time, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import synthetic, _native
spec = synthetic.WorkloadSpec("cfg1", 10000, 50, 16, 500, 6, 0.1, cfg=1)
model = synthetic.build_model(spec, seed=1001)
x = synthetic.host_features(spec, seed=1002)
xp = torch.from_numpy(x).pin_memory().numpy()
out = torch.empty(10000, dtype=torch.float64).pin_memory().numpy()
ev = obt.Evaluator(model)
fm = obt.FeatureMatrix(xp, obt.Layout.OBJECT_MAJOR)
for _ in range(50): ev.predict(fm, out=out)
torch.cuda.synchronize()
t = time.perf_counter(); R = 500
for _ in range(R): ev.predict(fm, out=out)
print("Evaluator.predict pinned: %.1f us" % ((time.perf_counter() - t) / R * 1e6))
lib = _native.load_library(); h = ev._dev.handle
st = _native.current_stream_handle()
t = time.perf_counter()
for _ in range(R): lib.obt_predict_host(h, xp.ctypes.data, 10000, 0, out.ctypes.data, st)
print("obt_predict_host raw: %.1f us" % ((time.perf_counter() - t) / R * 1e6))
xd = torch.from_numpy(x).cuda(); od = torch.empty(10000, dtype=torch.float64, device='cuda')
t = time.perf_counter()
for _ in range(R):
    od.copy_(torch.from_numpy(xp).cuda(non_blocking=True)[:, 0].double()) if False else None
    ev.predict_device(xd, out=od); torch.cuda.synchronize()
print("predict_device + sync: %.1f us" % ((time.perf_counter() - t) / R * 1e6))
a = torch.empty_like(xd)
t = time.perf_counter()
for _ in range(R):
    a.copy_(torch.from_numpy(xp), non_blocking=True); torch.cuda.synchronize()
print("H2D 2 MB pinned + sync: %.1f us" % ((time.perf_counter() - t) / R * 1e6))
P
