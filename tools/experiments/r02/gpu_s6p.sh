mkdir -p gpurun_out/s6p
for c in 4 2; do
extra=""; [ $c = 2 ] && extra="--path wide=1"
timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 $extra > gpurun_out/s6p/cfg$c.json 2> gpurun_out/s6p/cfg$c.err
python -c "
import json;d=json.loads(open('gpurun_out/s6p/cfg$c.json').read().strip().splitlines()[-1])
print('cfg$c', d['ms_per_step'], d['kernels']['quantize_ms'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_configs.py -m gpu -q -k "wide or K2w or k2w or full or fuzz" 2>&1 | tail -3
