run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b15_$name.json 2>gpurun_out/b15_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b15_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'], d['gpu_launches'])" 2>&1 | tail -1
}
run c2 2 X=1
run c2_ct32 2 OBT_CHUNK_TREES=32
run c3 3 X=1
run c3_ct32 3 OBT_CHUNK_TREES=32
run c2_again 2 X=1
