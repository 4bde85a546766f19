# K2w tree-split index halves (LDS.128 bucket words, one descriptor load per two trees, 4 SHFL swap) vs the default, config 4
mkdir -p gpurun_out/s6v
L=$PWD/paper_2211_00391_b200/_lib/tsplit/libobtree_b200.so
OBTREE_B200_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_configs.py -m gpu -q -x -k "wide or K2w or k2w or full or fuzz" 2>&1 | tail -3
for v in base tsplit; do
lib=""; [ $v = tsplit ] && lib=$L
OBTREE_B200_LIB=$lib timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s6v/$v.json 2> gpurun_out/s6v/$v.err; echo "$v rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/s6v/$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done
