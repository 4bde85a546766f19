# per-lane PTX retry loop in every kernel's warp waits (K1t/K1L, K2, K2f, K5) vs the voted loop
mkdir -p gpurun_out/s6h
for v in base waitasm; do
lib=""; [ $v = waitasm ] && lib="$PWD/paper_2211_00391_b200/_lib/waitasm/libobtree_b200.so"
for c in 4 2 3 1 5; do
extra=""; [ $c = 5 ] && extra="--steps 4 --warmup 3"
OBTREE_B200_LIB=$lib timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline $extra > gpurun_out/s6h/${v}_$c.json 2> gpurun_out/s6h/${v}_$c.err
python -c "
import json;d=json.loads(open('gpurun_out/s6h/${v}_$c.json').read().strip().splitlines()[-1])
print('$v cfg$c', d['ms_per_step'], d['kernels']['quantize_ms'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done; done
