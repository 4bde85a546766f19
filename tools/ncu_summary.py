#!/usr/bin/env python
"""Summarise an ncu --set full report: per kernel, the metrics the design is judged on.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json] [--label cfg2]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "pipe_fp64_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active": "pipe_uniform_pct",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "launch__registers_per_thread": "registers",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wf_pct",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed": "lsu_wf_pct",
    "smsp__inst_executed_op_shared_ld.sum": "lds_inst",
    "sm__mio_inst_issued.avg.pct_of_peak_sustained_active": "mio_issue_pct",
    "sm__mio2rf_writeback_active.avg.pct_of_peak_sustained_active": "mio2rf_pct",
    "smsp__inst_executed_op_shfl.sum": "shfl_inst",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}


def to_float(x: str):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def summarise(path: str) -> list:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        raise SystemExit(f"no data in {path}")
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for i, h in enumerate(hdr):
            if h in KEYS:
                v = to_float(vals[i])
                u = units[i]
                if v is not None and u in ("Mbyte", "Kbyte", "Gbyte", "byte"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                if v is not None and u in ("usecond", "msecond", "nsecond"):
                    v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}[u]
                rec[KEYS[h]] = v
        stalls = sorted(
            ((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), to_float(vals[i]))
             for i, h in enumerate(hdr)
             if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")),
            key=lambda kv: -(kv[1] or 0),
        )
        rec["top_stalls_per_issue"] = [(k, round(v, 3)) for k, v in stalls[:6] if v]
        if rec.get("dram_read") is not None and rec.get("dram_write") is not None:
            rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
        out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    recs = summarise(a.report)
    for r in recs:
        print(json.dumps(r))
    if a.json:
        data = {}
        try:
            data = json.load(open(a.json))
        except Exception:
            pass
        data[a.label or a.report] = recs
        json.dump(data, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
