mkdir -p gpurun_out/s6x
export NCU_DIR=/tmp/ncu_reps
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6x/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s6x/pytest.log
timeout 900 python tests/stress/stress_determinism.py 20 > gpurun_out/s6x/stress.log 2>&1; grep -c "0 differing" gpurun_out/s6x/stress.log; grep -v "0 differing" gpurun_out/s6x/stress.log | head -5
timeout 900 python bench.py > gpurun_out/s6x/bench_cfg4.json 2> gpurun_out/s6x/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --config 2 --path wide=1 --no-e2e --no-cpu-baseline > gpurun_out/s6x/cfg2_wide.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s6x/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s6x/ncu_launches_cfg4.log 2>&1; echo "launches cfg4 rc=$?"
SKIP=0 timeout 900 bash tools/prof.sh w4 'apply_wide' --config 4 > gpurun_out/s6x/prof_w4.txt 2>&1
cp gpurun_out/w4_by_opcode.txt gpurun_out/s6x/
for f in gpurun_out/s6x/bench_cfg4.json gpurun_out/s6x/cfg2_wide.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('roofline_step') or {}).get('frac'), (d.get('verify') or {}).get('bit_exact'), (d.get('kernels') or {}))"; done
head -c 900 gpurun_out/s6x/prof_w4.txt
