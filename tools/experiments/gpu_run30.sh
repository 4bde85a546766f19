run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b30_$name.json 2>gpurun_out/b30_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b30_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'])" 2>&1 | tail -1
}
run c2 2 X=1
run c2_g16 2 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/g16/libobtree_b200.so
run c2_g16pf4 2 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/g16pf4/libobtree_b200.so
run c5 5 X=1
run c5_v2 5 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/v2/libobtree_b200.so
