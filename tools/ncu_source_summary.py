#!/usr/bin/env python
"""Per-opcode totals from an ncu source page (SASS): executed instructions, shared
wavefronts and stall samples -- where a kernel's time goes, instruction class by class."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = {}
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    parts = src.split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    key = op if op.startswith(("LDS", "LDC", "LDCU")) else op.split(".")[0]
    f = lambda k: float(r[ix[k]] or 0) if k in ix else 0.0  # noqa: E731
    t = tot.setdefault(key, [0.0, 0.0, 0.0, 0.0])
    t[0] += f("Instructions Executed")
    t[1] += f("L1 Wavefronts Shared")
    t[2] += f("Warp Stall Sampling (All Samples)")
    t[3] += f("Warp Stall Sampling (Not-issued Samples)")
ti = sum(v[0] for v in tot.values()) or 1
ts = sum(v[2] for v in tot.values()) or 1
tw = sum(v[1] for v in tot.values()) or 1
print(f"{'op':14s} {'inst%':>6s} {'wf%':>6s} {'stall%':>7s} {'wf/inst':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][2])[:18]:
    print(f"{k:14s} {100*v[0]/ti:6.1f} {100*v[1]/tw:6.1f} {100*v[2]/ts:7.1f} {v[1]/max(v[0],1):7.2f}")
