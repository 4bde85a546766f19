mkdir -p gpurun_out/s6q
for leaves in fp32 fp16; do
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/k5defer/libobtree_b200.so timeout 900 python bench.py --config 5 --leaves $leaves --no-e2e --no-cpu-baseline --steps 4 --warmup 3 > gpurun_out/s6q/k5_$leaves.json 2> gpurun_out/s6q/k5_$leaves.err
python -c "
import json;d=json.loads(open('gpurun_out/s6q/k5_$leaves.json').read().strip().splitlines()[-1])
print('deferred $leaves', d['ms_per_step'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/k5defer/libobtree_b200.so timeout 600 python bench.py --config 6 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/s6q/cfg6.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/s6q/cfg6.json').read().strip().splitlines()[-1])
print('deferred cfg6', d['ms_per_step'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
timeout 600 python bench.py --config 5 --leaves fp16 --no-e2e --no-cpu-baseline --steps 4 --warmup 3 > gpurun_out/s6q/fence_fp16.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/s6q/fence_fp16.json').read().strip().splitlines()[-1])
print('fence fp16', d['ms_per_step'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
