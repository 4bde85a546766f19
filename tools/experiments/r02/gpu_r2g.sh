# K2w packed 7-bit descriptors + plain try_wait: parity, cfg4 bench, ncu
mkdir -p gpurun_out/r2g
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k wide > gpurun_out/r2g/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -3 gpurun_out/r2g/pytest_wide.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2g/cfg4.json 2>gpurun_out/r2g/cfg4.err; echo "rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2g/cfg4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
export NCU_DIR=/tmp/ncu_reps
SKIP=0 timeout 900 bash tools/prof.sh w4e 'apply_wide' --config 4 > gpurun_out/r2g/prof_w4e.txt 2>&1; head -c 1500 gpurun_out/r2g/prof_w4e.txt
cp /tmp/ncu_reps/w4e.ncu-rep gpurun_out/r2g/ 2>/dev/null; cp gpurun_out/w4e_by_opcode.txt gpurun_out/r2g/
