# K1L stage release: after the step's searches (1) or behind a proxy fence (3), quantize times
mkdir -p gpurun_out/s6m
for v in 1 3; do
for c in 4 2; do
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/k1l$v/libobtree_b200.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/s6m/v${v}_$c.json 2> gpurun_out/s6m/v${v}_$c.err
python -c "
import json;d=json.loads(open('gpurun_out/s6m/v${v}_$c.json').read().strip().splitlines()[-1])
print('variant $v cfg$c', d['ms_per_step'], d['kernels']['quantize_ms'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done; done
