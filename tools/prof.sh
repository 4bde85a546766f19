#!/bin/bash
# usage: [SKIP=n] tools/prof.sh <label> <kernel-regex> [bench args...]
# Runs the bench command plainly (must exit 0), then once under ncu --set full for
# one launch of the matching kernel (after skipping SKIP matching launches, default 3);
# summary appended to gpurun_out/ncu_<label>.json
label=$1; shift; regex=$1; shift
skip=${SKIP:-3}
cmd="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $*"
$cmd > gpurun_out/plain_$label.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$label.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$regex -s $skip -c 1 -o gpurun_out/$label -f $cmd > gpurun_out/ncu_$label.log 2>&1
python tools/ncu_summary.py gpurun_out/$label.ncu-rep
