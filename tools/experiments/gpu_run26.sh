run() { # name config env...
  name=$1; c=$2; shift 2
  env $(echo "$@" | tr " " "\n" | grep = | tr "\n" " ") timeout 900 python bench.py --config $c $(echo "$@" | tr " " "\n" | grep -v = | tr "\n" " ") --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/b26_$name.json 2>gpurun_out/b26_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b26_$name.json'));print('$name', round(d['ms_per_step']*1000,2), 'us', d['kernels'])" 2>&1 | tail -1
}
run c1 1 X=1
run c1_tpw4 1 OBT_TPW=4
run c1_tpw1 1 OBT_TPW=1
run c1_tile256 1 OBT_TILE=256
run c1_tile256_tpw4 1 OBT_TILE=256 OBT_TPW=4
run c1_nograph 1 X=1 --graph off
