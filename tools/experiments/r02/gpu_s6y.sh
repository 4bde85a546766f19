# timing probe: K2w tree split without the SHFL swap (results wrong): the upper bound of a swap-free layout
mkdir -p gpurun_out/s6y
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/noswap/libobtree_b200.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s6y/noswap.json 2> gpurun_out/s6y/noswap.err
python -c "
import json;d=json.loads(open('gpurun_out/s6y/noswap.json').read().strip().splitlines()[-1])
print('noswap', d['ms_per_step'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
