run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b44_$name.json 2>gpurun_out/b44_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b44_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'])" 2>&1 | tail -1
}
run c2 2 X=1
run c2_l2 2 OBT_L2_NEXT=1
run c2b 2 X=1
run c2_l2b 2 OBT_L2_NEXT=1
