timeout 1200 python -m pytest tests -m gpu -q -k "chained or descriptor or smoke or tail" > gpurun_out/pytest_gpu57.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu57.log
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b57_$name.json 2>gpurun_out/b57_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b57_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'])" 2>&1 | tail -1
}
run c2_rev 2 X=1
run c2_fwd 2 OBT_CHAIN_ORDER=fwd
run c2_revb 2 X=1
run c2_fwdb 2 OBT_CHAIN_ORDER=fwd
run c3_rev 3 X=1
run c3_fwd 3 OBT_CHAIN_ORDER=fwd
