run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b49_$name.json 2>gpurun_out/b49_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b49_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['quantize_ms'],4))" 2>&1 | tail -1
}
for v in default l2n l2x l264 default; do
  if [ $v = default ]; then lib=""; else lib=paper_2211_00391_b200/_lib/$v/libobtree_b200.so; fi
  run c2_$v 2 OBTREE_B200_LIB=$lib
done
