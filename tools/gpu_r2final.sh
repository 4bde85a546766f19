# Round-2 bench lines for every configuration + the reference arm (default command = cfg4)
mkdir -p gpurun_out/r2final
timeout 1200 python bench.py > gpurun_out/r2final/bench_cfg4.json 2> gpurun_out/r2final/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 900 python bench.py --config 2 > gpurun_out/r2final/bench_cfg2.json 2> gpurun_out/r2final/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config 3 > gpurun_out/r2final/bench_cfg3.json 2> gpurun_out/r2final/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config 1 > gpurun_out/r2final/bench_cfg1.json 2> gpurun_out/r2final/bench_cfg1.err; echo "cfg1 rc=$?"
timeout 1500 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r2final/bench_cfg5.json 2> gpurun_out/r2final/bench_cfg5.err; echo "cfg5 rc=$?"
timeout 1500 python bench.py --config 5 --steps 5 --warmup 3 --leaves fp16 > gpurun_out/r2final/bench_cfg5h.json 2> gpurun_out/r2final/bench_cfg5h.err; echo "cfg5h rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2final/bench_reference.json 2> gpurun_out/r2final/bench_reference.err; echo "ref rc=$?"
for f in gpurun_out/r2final/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('roofline_step') or {}).get('frac'), (d.get('verify') or {}).get('bit_exact'), (d.get('kernels') or {}))"; done
