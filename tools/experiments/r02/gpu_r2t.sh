# K5 producer: per-lane row copies with descriptor lookahead vs one serial producer thread
mkdir -p gpurun_out/r2t
L=paper_2211_00391_b200/_lib
for v in default k5ser; do
  if [ $v = default ]; then lib=$L/libobtree_b200.so; else lib=$L/$v/libobtree_b200.so; fi
  for lv in fp32 fp16; do
  OBTREE_B200_LIB=$PWD/$lib timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --leaves $lv > gpurun_out/r2t/cfg5_${v}_$lv.json 2>gpurun_out/r2t/cfg5_${v}_$lv.err; echo "$v $lv rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2t/cfg5_${v}_$lv.json').read().strip().splitlines()[-1]);print('$v $lv', d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
  done
done
