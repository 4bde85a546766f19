run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b12_$name.json 2>gpurun_out/b12_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b12_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['apply_ms'],3))" 2>&1 | tail -1
}
run c5_ahead 5 X=1
run c5_ahead0 5 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/ahead0/libobtree_b200.so
run c5_minb3 5 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/minb3/libobtree_b200.so
run c5_minb4 5 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/minb4/libobtree_b200.so
