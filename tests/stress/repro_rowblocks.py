"""Repeat the K1L row-block-group predict (F = 2000, the K5 record path with one output)
and report where mismatches against the oracle fall (an intermittent failure was seen once)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
import numpy as np
import torch

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import _native, synthetic


def model_of(F, B, T, D, seed):
    return synthetic.build_model(synthetic.WorkloadSpec("t", 1, F, B, T, D, 0.1, cfg=1), seed=seed, affine=True)


def features(model, n, seed):
    x = synthetic.host_features(synthetic.WorkloadSpec("t", n, model.n_features, 1, 1, 1, 0.1, cfg=1), seed=seed)
    return synthetic.sprinkle_specials(x, [ff.borders for ff in model.float_features], seed=seed + 1)


def main():
    F, n, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    opts = dict(kv.split("=") for kv in sys.argv[4:])
    for k, v in opts.items():
        _native.set_path_option(k, int(v))
    model = model_of(F, 128, 300, 6, seed=F)
    x = features(model, n, seed=F + 1)
    ev = obt.Evaluator(model, device=0)
    oracle.set_threads(oracle.host_cores())
    want = oracle.evaluate_scalar(oracle.flatten(model), x)
    xd = torch.from_numpy(x).cuda()
    bad_runs = 0
    for it in range(iters):
        # disturb timing between runs: other work on the device, cache flush
        junk = torch.empty(64 << 20, dtype=torch.uint8, device="cuda").random_()
        got = ev.predict_device(xd).cpu().numpy()
        bad = np.flatnonzero(got != want)
        if bad.size:
            bad_runs += 1
            print(f"iter {it}: {bad.size} mismatches, objects {bad.min()}..{bad.max()}, "
                  f"1024-blocks {sorted(set((bad // 1024).tolist()))[:12]}, "
                  f"in-block offsets {sorted(set((bad % 1024).tolist()))[:16]}", flush=True)
        del junk
    print(f"F={F} n={n} opts={opts} quantize={ev.quantize_kernel()}: {bad_runs} bad of {iters}", flush=True)


if __name__ == "__main__":
    main()
