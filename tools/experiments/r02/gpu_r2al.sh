# K2w: producer roles in three warps (was three lanes of one warp); ts up to 8
mkdir -p gpurun_out/r2al
for a in "2 --path wide=1" "3 --path wide=1" "4"; do set -- $a; c=$1; shift
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/r2al/k2w$c.json 2>gpurun_out/r2al/k2w$c.err; echo "k2w$c rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2al/k2w$c.json').read().strip().splitlines()[-1]);print('k2w$c', d['ms_per_step'], d.get('kernels'), d['verify']['bit_exact'])"
done
NCU_DIR=gpurun_out/r2al timeout 900 bash tools/prof.sh w2c apply_wide --config 2 --path wide=1
