run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b16_$name.json 2>gpurun_out/b16_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b16_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'], d['gpu_launches'])" 2>&1 | tail -1
}
run c2 2 X=1
run c2_tpw1 2 OBT_TPW=1
run c2_notail 2 OBT_TAIL_SPLIT=0
run c4 4 X=1
