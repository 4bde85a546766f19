mkdir -p gpurun_out/final3
timeout 900 python bench.py > gpurun_out/final3/bench_cfg2.json 2> gpurun_out/final3/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/final3/bench_cfg3.json 2> gpurun_out/final3/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 1200 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final3/bench_cfg4.json 2> gpurun_out/final3/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --config 1 > gpurun_out/final3/bench_cfg1.json 2> gpurun_out/final3/bench_cfg1.err; echo "cfg1 rc=$?"
for f in gpurun_out/final3/bench_*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline_smem') or {}).get('frac'))"; done
