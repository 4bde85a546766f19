# timing probes of K2f at config 1 (results wrong): without the fold adds, without the compute warps' work, without both
mkdir -p gpurun_out/s7i
for v in pnofold pnocomp pnone; do
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/$v/libobtree_b200.so timeout 600 python bench.py --config 1 --no-e2e --no-cpu-baseline --steps 300 --warmup 20 --graph off > gpurun_out/s7i/$v.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/s7i/$v.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step']*1e3,2), {k:round(x*1e3,2) for k,x in d['kernels'].items() if k.endswith('_ms')})"
done
