timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu32.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu32.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu32.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b32_$name.json 2>gpurun_out/b32_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b32_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels'])" 2>&1 | tail -1
}
run c4 4 X=1
run c1 1 X=1
