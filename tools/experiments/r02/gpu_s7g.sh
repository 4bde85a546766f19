# the per-GPU share of config 4 under object sharding: 8M / N objects on one GPU (what each rank of an N-GPU run computes)
mkdir -p gpurun_out/s7g
for n in 8000000 4000000 2000000 1000000; do
timeout 600 python bench.py --objects $n --no-e2e --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/s7g/n$n.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/s7g/n$n.json').read().strip().splitlines()[-1])
print($n, d['ms_per_step'], d['value'], d['kernels']['quantize_ms'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
done
