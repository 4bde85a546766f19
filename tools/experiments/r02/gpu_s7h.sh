# K1 (LDG quantize): the first step's rows requested before the tables are staged
mkdir -p gpurun_out/s7h
for v in base k1pre; do
lib=""; [ $v = k1pre ] && lib="$PWD/paper_2211_00391_b200/_lib/k1pre/libobtree_b200.so"
OBTREE_B200_LIB=$lib timeout 600 python bench.py --config 1 --no-e2e --no-cpu-baseline --steps 300 --warmup 20 > gpurun_out/s7h/${v}_1.json 2>/dev/null
OBTREE_B200_LIB=$lib timeout 600 python bench.py --config 1 --no-e2e --no-cpu-baseline --steps 300 --warmup 20 --graph off > gpurun_out/s7h/${v}_1s.json 2>/dev/null
for t in 1 1s; do python -c "
import json;d=json.loads(open('gpurun_out/s7h/${v}_$t.json').read().strip().splitlines()[-1])
print('$v $t', d['ms_per_step'], d['kernels'], d['verify'].get('bit_exact'))"; done
done
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/k1pre/libobtree_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "quantize or layout or corpus or feature_major or ragged or empty" 2>&1 | tail -2
