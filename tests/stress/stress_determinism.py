"""Repeat predicts of several shapes (every apply kernel family) with other work in between
and compare every run's full output and bucket workspace with the first run's bit for bit:
a race shows up as a run that differs.  The first run is checked against the oracle on a
row sample."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import _native, multiclass, synthetic

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from bench import flat_model, sample_rows  # noqa: E402


def run(name, spec, iters, opts=None, half=False, n=None):
    opts = opts or {}
    for k, v in opts.items():
        _native.set_path_option(k, v)
    try:
        if spec.n_outputs > 1:
            model = multiclass.from_arrays(synthetic.model_arrays(spec))
            cfg = obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16) if half else None
            ev = multiclass.MultiOutputEvaluator(model, device=0, config=cfg)
        else:
            model = synthetic.build_model(spec)
            cfg = obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16 if half else obt.LeafStrategy.NAIVE)
            ev = obt.Evaluator(model, cfg, device=0)
        n = n or spec.n_objects
        x = synthetic.device_features(spec, n_objects=n, device="cuda")
        nbytes = ev.workspace_bytes(n)
        ws0 = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        first = ev.predict_device(x, workspace=ws0).clone()
        torch.cuda.synchronize()
        rows = sample_rows(n, 8192)
        oracle.set_threads(oracle.host_cores())
        want = oracle.evaluate_scalar(flat_model(model), x[torch.from_numpy(rows).cuda()].cpu().numpy(),
                                      oracle.OBJECT_MAJOR, oracle.BINARY16 if half else oracle.BINARY64)
        got = first[torch.from_numpy(rows).cuda()].cpu().numpy()
        exact = np.array_equal(got.reshape(want.shape), want)
        bad = 0
        for it in range(iters):
            junk = torch.empty(96 << 20, dtype=torch.uint8, device="cuda").random_()
            ws = torch.full((nbytes,), 0xEE, dtype=torch.uint8, device="cuda")
            out = ev.predict_device(x, workspace=ws)
            torch.cuda.synchronize()
            nd = int((out != first).sum().item())
            if nd:
                bad += 1
                idx = torch.nonzero((out != first).reshape(n, -1).any(dim=1)).flatten().cpu().numpy()
                print(f"  {name} iter {it}: {nd} outputs differ, objects {idx.min()}..{idx.max()} "
                      f"({idx.size} objects; 256-tiles {sorted(set((idx // 256).tolist()))[:8]})", flush=True)
            del junk, ws, out
        print(f"{name}: oracle-exact sample {exact}; {bad} differing runs of {iters}", flush=True)
    finally:
        for k in opts:
            _native.set_path_option(k, -1)


def main():
    W = synthetic.WorkloadSpec
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    run("K2w cfg4-shape 1M", synthetic.CONFIGS[4], iters, n=1_000_000)
    run("K2w cfg4-shape fp16 1M", W(**{**synthetic.CONFIGS[4].__dict__, "half_leaves": True}), iters, half=True, n=1_000_000)
    run("K2 cfg2 (bank, chained)", synthetic.CONFIGS[2], iters)
    run("K2 cfg2 unchained", synthetic.CONFIGS[2], iters, {"pdl": 0})
    run("K2 cfg2 ring descriptors + tail split", synthetic.CONFIGS[2], iters, {"desc_source": 0, "tail_split": 1})
    run("K2 cfg3 fp16", synthetic.CONFIGS[3], iters, half=True)
    run("K2s cfg4-shape 300k (wide off)", synthetic.CONFIGS[4], iters, {"wide": 0}, n=300_000)
    run("K2f cfg1", synthetic.CONFIGS[1], iters * 3)
    run("K5 cfg5-shape 400 trees 300k", W(**{**synthetic.CONFIGS[5].__dict__, "n_trees": 400}), iters, n=300_000)
    run("K5 fp16 cfg5-shape 400 trees 300k", W(**{**synthetic.CONFIGS[5].__dict__, "n_trees": 400, "half_leaves": True}),
        iters, half=True, n=300_000)
    run("K4 cfg5-shape 100 trees 100k", W(**{**synthetic.CONFIGS[5].__dict__, "n_trees": 100}), max(4, iters // 4),
        {"multi_staged": 0}, n=100_000)
    run("K5 one output, epsilon shape 200k", synthetic.CONFIGS[6], iters, n=200_000)


if __name__ == "__main__":
    main()
