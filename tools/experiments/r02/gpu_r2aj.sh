# config 2 with K2w forced: where does the time go (K2 1.2 ms step vs K2w 1.35)
mkdir -p gpurun_out/r2aj
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2aj/k2.json 2>gpurun_out/r2aj/k2.err; echo "k2 rc=$?"
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --path wide=1 > gpurun_out/r2aj/k2w.json 2>gpurun_out/r2aj/k2w.err; echo "k2w rc=$?"
for f in k2 k2w; do python -c "import json;d=json.loads(open('gpurun_out/r2aj/$f.json').read().strip().splitlines()[-1]);print('$f', d['ms_per_step'], d.get('kernels'), d['verify']['bit_exact'])"; done
NCU_DIR=gpurun_out/r2aj timeout 900 bash tools/prof.sh w2 apply_wide --config 2 --path wide=1
