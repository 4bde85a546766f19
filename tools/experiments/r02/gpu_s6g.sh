# K2w barrier-wait loop forms (config 4): 1 = per-lane retry loop in PTX (no vote), 2 = one lane polls + __syncwarp
mkdir -p gpurun_out/s6g
for v in wait1 wait2; do
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/$v/libobtree_b200.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s6g/$v.json 2> gpurun_out/s6g/$v.err; echo "$v rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/s6g/$v.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done
