timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu19.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu19.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu19.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b19_$name.json 2>gpurun_out/b19_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b19_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels'])" 2>&1 | tail -1
}
run c2 2 X=1
run c2_eytz 2 OBT_QUANT_LUT=0
run c4 4 X=1
