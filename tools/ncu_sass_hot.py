#!/usr/bin/env python
"""SASS listing of an ncu report with per-instruction executions, shared wavefronts and
stall samples (all / not-issued), for reading where a kernel waits.

    python tools/ncu_sass_hot.py rep.ncu-rep [min_samples]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
for n, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    f = lambda k: float(r[ix[k]] or 0)  # noqa: E731
    s = f("Warp Stall Sampling (All Samples)")
    if s < thr and f("L1 Wavefronts Shared") == 0:
        continue
    top = sorted(((f(c), c[6:]) for c in stall_cols), reverse=True)[:2]
    tops = " ".join(f"{c}:{v:.0f}" for v, c in top if v > 0)
    print(f"{n:5d} {r[ix['Source']].strip()[:60]:60s} ex={f('Instructions Executed'):.3g} "
          f"wf={f('L1 Wavefronts Shared'):.3g} st={s:.0f} {tops}")
