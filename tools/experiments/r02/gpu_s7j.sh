# K2f: 16-stage ring + named-barrier panel hand-offs (config 1)
mkdir -p gpurun_out/s7j
for v in base fanbar; do
lib=""; [ $v = fanbar ] && lib="$PWD/paper_2211_00391_b200/_lib/fanbar/libobtree_b200.so"
for g in auto off; do
OBTREE_B200_LIB=$lib timeout 600 python bench.py --config 1 --no-e2e --no-cpu-baseline --steps 300 --warmup 20 --graph $g > gpurun_out/s7j/${v}_$g.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/s7j/${v}_$g.json').read().strip().splitlines()[-1])
print('$v $g', round(d['ms_per_step']*1e3,2), {k:round(x*1e3,2) for k,x in d['kernels'].items() if k.endswith('_ms')}, d['verify']['bit_exact'])"
done; done
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/fanbar/libobtree_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fan or small or corpus or fuzz or ragged or empty" 2>&1 | tail -2
