timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu60.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu60.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu60.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
mkdir -p gpurun_out/final4
timeout 900 python bench.py > gpurun_out/final4/bench_cfg2.json 2> gpurun_out/final4/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/final4/bench_cfg3.json 2> gpurun_out/final4/bench_cfg3.err; echo "cfg3 rc=$?"
for f in gpurun_out/final4/bench_*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline_smem') or {}).get('frac'), d['cpu_baseline'].get('gpu_verified_bit_exact') if d.get('cpu_baseline') else None)"; done
