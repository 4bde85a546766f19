# K2w: index-warp count and wait-mode A/B at cfg4
mkdir -p gpurun_out/r2f
L=paper_2211_00391_b200/_lib
for v in default nidx10 nidx12 nosusp; do
  if [ $v = default ]; then lib=$L/libobtree_b200.so; else lib=$L/$v/libobtree_b200.so; fi
  OBTREE_B200_LIB=$PWD/$lib timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2f/cfg4_$v.json 2>gpurun_out/r2f/cfg4_$v.err; echo "$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2f/cfg4_$v.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
done
