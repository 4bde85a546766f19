# K2w descriptor source A/B after the three-producer-warp change (config 4)
mkdir -p gpurun_out/s6c
for v in 0 1; do
timeout 600 python bench.py --path desc_source=$v --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s6c/ds$v.json 2> gpurun_out/s6c/ds$v.err; echo "ds$v rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/s6c/ds$v.json').read().strip().splitlines()[-1])
print('desc_source=$v', d['ms_per_step'], d['kernels'], d['verify'].get('bit_exact'), d['gpu_launches'])"
done
