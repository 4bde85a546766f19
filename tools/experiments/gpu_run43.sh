for v in 1 0; do
OBT_LDG_LUT=$v timeout 600 python bench.py --config 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/b43_$v.json 2>gpurun_out/b43_$v.err
python -c "import json;d=json.loads(open('gpurun_out/b43_$v.json').read().strip().splitlines()[-1]);print('ldg_lut=$v', round(d['ms_per_step']*1e3,2), 'us', d['kernels'], d['e2e']['ms_per_step'])"
done
