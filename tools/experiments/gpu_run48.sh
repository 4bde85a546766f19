timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu48.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu48.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu48.log | head
mkdir -p gpurun_out/final2
timeout 900 python bench.py > gpurun_out/final2/bench_cfg2.json 2> gpurun_out/final2/bench_cfg2.err; echo "cfg2 rc=$?"; tail -c 400 gpurun_out/final2/bench_cfg2.json
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/final2/bench_cfg3.json 2> gpurun_out/final2/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 1200 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final2/bench_cfg4.json 2> gpurun_out/final2/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final2/bench_cfg5.json 2> gpurun_out/final2/bench_cfg5.err; echo "cfg5 rc=$?"
timeout 600 python bench.py --config 1 > gpurun_out/final2/bench_cfg1.json 2> gpurun_out/final2/bench_cfg1.err; echo "cfg1 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final2/bench_reference.json 2> gpurun_out/final2/bench_reference.err; echo "ref rc=$?"
for f in gpurun_out/final2/bench_*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'))"; done
