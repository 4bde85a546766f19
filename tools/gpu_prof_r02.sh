# Round-2 profiles: launch lists (cold-cache, serialised) of the default bench command and
# ncu --set full captures of the dominant kernels, each after its plain run exits 0.
mkdir -p gpurun_out/r2prof
export NCU_DIR=/tmp/ncu_reps
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2prof/plain_cfg4.json 2>&1; echo "plain cfg4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2prof/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2prof/ncu_launches_cfg4.log 2>&1; echo "launches cfg4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2prof/launches_cfg2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2prof/ncu_launches_cfg2.log 2>&1; echo "launches cfg2 rc=$?"
SKIP=0 timeout 900 bash tools/prof.sh w4 'apply_wide' --config 4 > gpurun_out/r2prof/prof_w4.txt 2>&1; head -c 300 gpurun_out/r2prof/prof_w4.txt
SKIP=1 timeout 900 bash tools/prof.sh q4 'quantize_lut' --config 4 > gpurun_out/r2prof/prof_q4.txt 2>&1; head -c 300 gpurun_out/r2prof/prof_q4.txt
for r in w4 q4; do cp gpurun_out/${r}_by_opcode.txt gpurun_out/r2prof/; python tools/ncu_summary.py $NCU_DIR/$r.ncu-rep --json gpurun_out/r2prof/ncu_$r.json > /dev/null 2>&1; done
cp $NCU_DIR/w4.ncu-rep gpurun_out/r2prof/ 2>/dev/null
ls -la gpurun_out/r2prof
