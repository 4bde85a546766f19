# K2w parameter-bank descriptors (multi-launch fold) vs the descriptor ring
mkdir -p gpurun_out/r2n
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or full_model or past_4gib" > gpurun_out/r2n/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2n/pytest.log
for ds in 1 0; do
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --path desc_source=$ds > gpurun_out/r2n/cfg4_ds$ds.json 2>gpurun_out/r2n/cfg4_ds$ds.err; echo "ds=$ds rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2n/cfg4_ds$ds.json').read().strip().splitlines()[-1]);print($ds, d['ms_per_step'], d['kernels']['apply_ms'], d['gpu_launches'], d['verify']['bit_exact'])"
done
export NCU_DIR=/tmp/ncu_reps
SKIP=0 timeout 900 bash tools/prof.sh w4p 'apply_wide' --config 4 > gpurun_out/r2n/prof_w4p.txt 2>&1; head -c 1500 gpurun_out/r2n/prof_w4p.txt
cp /tmp/ncu_reps/w4p.ncu-rep gpurun_out/r2n/ 2>/dev/null; cp gpurun_out/w4p_by_opcode.txt gpurun_out/r2n/
