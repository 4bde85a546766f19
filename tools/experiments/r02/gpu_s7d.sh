# K2f: G ring chunks per value-panel hand-off (config 1: 16 hand-offs of 32 trees -> 500 / (32 G))
mkdir -p gpurun_out/s7d
for v in fg2 fg4 fg8; do
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/$v/libobtree_b200.so timeout 600 python bench.py --config 1 --no-e2e --no-cpu-baseline --steps 200 --warmup 20 > gpurun_out/s7d/$v.json 2> gpurun_out/s7d/$v.err
python -c "
import json;d=json.loads(open('gpurun_out/s7d/$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['kernels'], d['verify'].get('bit_exact'))"
done
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/fg4/libobtree_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fan or small or K2f or k2f or corpus or fuzz" 2>&1 | tail -2
