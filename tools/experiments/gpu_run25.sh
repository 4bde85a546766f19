nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,temperature.gpu,power.draw --format=csv
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b25_$name.json 2>gpurun_out/b25_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b25_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels'])" 2>&1 | tail -1
}
run c2 2 X=1
run c2_head 2 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/head/libobtree_b200.so
run c3 3 X=1
run c3_head 3 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/head/libobtree_b200.so
run c2_nomix 2 OBT_MIXED_TILES=0
