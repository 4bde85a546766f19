# K2w at config 2/3 with up to 8 table stages (was 3)
mkdir -p gpurun_out/r2ak
for c in 2 3; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --path wide=1 > gpurun_out/r2ak/k2w$c.json 2>gpurun_out/r2ak/k2w$c.err; echo "k2w$c rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2ak/k2w$c.json').read().strip().splitlines()[-1]);print('k2w$c', d['ms_per_step'], d.get('kernels'), d['verify']['bit_exact'])"
done
NCU_DIR=gpurun_out/r2ak timeout 900 bash tools/prof.sh w2b apply_wide --config 2 --path wide=1
