run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b55_$name.json 2>gpurun_out/b55_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b55_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'])" 2>&1 | tail -1
}
L=paper_2211_00391_b200/_lib/chain2/libobtree_b200.so
run c2 2 X=1
run c2_chain2 2 OBTREE_B200_LIB=$L
run c2b 2 X=1
run c2_chain2b 2 OBTREE_B200_LIB=$L
run c3 3 X=1
run c3_chain2 3 OBTREE_B200_LIB=$L
