# K2f: four trees per compute-warp pass, staged (all bucket loads, then indices, then gathers, then stores), config 1
mkdir -p gpurun_out/s7b
for v in base fan4; do
lib=""; [ $v = fan4 ] && lib="$PWD/paper_2211_00391_b200/_lib/fan4/libobtree_b200.so"
OBTREE_B200_LIB=$lib timeout 600 python bench.py --config 1 --no-e2e --no-cpu-baseline --steps 200 --warmup 20 > gpurun_out/s7b/$v.json 2> gpurun_out/s7b/$v.err
python -c "
import json;d=json.loads(open('gpurun_out/s7b/$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['kernels'], d['verify'].get('bit_exact'))"
done
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/fan4/libobtree_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fan or small or K2f or k2f or corpus" 2>&1 | tail -2
