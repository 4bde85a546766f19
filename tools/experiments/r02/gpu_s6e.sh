# K2w packed 4-byte descriptors ((row << 22) | k, LEA.HI address, PRMT k) vs the 8-byte pairs, config 4
mkdir -p gpurun_out/s6e
for v in base packed; do
lib=""; [ $v = packed ] && lib="$PWD/paper_2211_00391_b200/_lib/packed/libobtree_b200.so"
OBTREE_B200_LIB=$lib timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s6e/$v.json 2> gpurun_out/s6e/$v.err; echo "$v rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/s6e/$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['kernels'], d['verify'].get('bit_exact'))"
done
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/packed/libobtree_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or K2w or k2w" 2>&1 | tail -3
