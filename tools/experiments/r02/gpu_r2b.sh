# cfg4: K2w vs K2s A/B, and ncu of each (one launch)
mkdir -p gpurun_out/r2b
export NCU_DIR=/tmp/ncu_reps
for w in 0 1; do
OBT_WIDE=$w timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2b/cfg4_wide$w.json 2>gpurun_out/r2b/cfg4_wide$w.err; echo "wide=$w rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2b/cfg4_wide$w.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernels'], d['verify']['bit_exact'])"
done
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2b/cfg2.json 2>gpurun_out/r2b/cfg2.err; echo "cfg2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2b/cfg2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernels'], d['verify']['bit_exact'])"
OBT_WIDE=1 SKIP=0 timeout 900 bash tools/prof.sh w4 'apply_wide' --config 4 > gpurun_out/r2b/prof_w4.txt 2>&1; head -c 3000 gpurun_out/r2b/prof_w4.txt
cp gpurun_out/w4_by_opcode.txt gpurun_out/r2b/ 2>/dev/null
OBT_WIDE=0 SKIP=0 timeout 900 bash tools/prof.sh s4 'apply_split' --config 4 > gpurun_out/r2b/prof_s4.txt 2>&1; head -c 3000 gpurun_out/r2b/prof_s4.txt
cp gpurun_out/s4_by_opcode.txt gpurun_out/r2b/ 2>/dev/null
cp /tmp/ncu_reps/w4.ncu-rep /tmp/ncu_reps/s4.ncu-rep gpurun_out/r2b/ 2>/dev/null; ls -la gpurun_out/r2b
