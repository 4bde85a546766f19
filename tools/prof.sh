#!/bin/bash
# usage: [SKIP=n] [NCU_DIR=dir] tools/prof.sh <label> <kernel-regex> [bench args...]
# Runs the bench command plainly (must exit 0), then once under ncu --set full for
# one launch of the matching kernel (after skipping SKIP matching launches, default 3);
# prints the summary JSON and writes <label>_by_opcode.txt next to the report.  Reports
# go to NCU_DIR (default gpurun_out; large captures belong outside gpurun_out, which
# only travels back below 64 MiB).
label=$1; shift; regex=$1; shift
skip=${SKIP:-3}
dir=${NCU_DIR:-gpurun_out}
mkdir -p "$dir"
cmd="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $*"
$cmd > gpurun_out/plain_$label.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$label.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$regex -s $skip -c 1 -o "$dir/$label" -f $cmd > gpurun_out/ncu_$label.log 2>&1
python tools/ncu_summary.py "$dir/$label.ncu-rep"
python tools/ncu_source_summary.py "$dir/$label.ncu-rep" > gpurun_out/${label}_by_opcode.txt 2>&1
