"""Compare the tiled bucket matrix K1L leaves in the workspace with K1t's (same used-border
buckets, same layout) over repeated runs; report which (tile, feature, position) differ."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import _native, synthetic
from repro_rowblocks import features, model_of


def main():
    F, n, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    model = model_of(F, 128, 300, 6, seed=F)
    x = features(model, n, seed=F + 1)
    ev = obt.Evaluator(model, device=0)
    xd = torch.from_numpy(x).cuda()
    nbytes = ev.workspace_bytes(n)
    tile = 2048 if F > 1600 else 256
    n_tiles = -(-n // tile)
    qbytes = n_tiles * tile * F
    print("workspace", nbytes, "bucket bytes", qbytes, flush=True)
    ws_ref = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    _native.set_path_option("quant_lut", 0)
    ref_out = ev.predict_device(xd, workspace=ws_ref).clone()
    torch.cuda.synchronize()
    _native.set_path_option("quant_lut", 1)
    print("quantize", ev.quantize_kernel(), flush=True)
    bad_runs = 0
    for it in range(iters):
        junk = torch.empty(64 << 20, dtype=torch.uint8, device="cuda").random_()
        ws = torch.full((nbytes,), 0xEE, dtype=torch.uint8, device="cuda")
        out = ev.predict_device(xd, workspace=ws)
        torch.cuda.synchronize()
        diff = torch.nonzero(ws[:qbytes] != ws_ref[:qbytes]).flatten().cpu().numpy()
        obad = int((out != ref_out).sum().item())
        if diff.size or obad:
            bad_runs += 1
            t = diff // (F * tile)
            f = (diff % (F * tile)) // tile
            pos = diff % tile
            got = ws[torch.from_numpy(diff[:8]).cuda()].cpu().numpy()
            want = ws_ref[torch.from_numpy(diff[:8]).cuda()].cpu().numpy()
            print(f"iter {it}: {diff.size} bucket bytes differ ({obad} predictions); tiles {sorted(set(t.tolist()))[:6]}, "
                  f"features {sorted(set(f.tolist()))[:24]}, positions {pos.min() if diff.size else -1}..{pos.max() if diff.size else -1}; "
                  f"got {got.tolist()} want {want.tolist()}", flush=True)
        del junk
    print(f"{bad_runs} bad of {iters}", flush=True)


if __name__ == "__main__":
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    main()
