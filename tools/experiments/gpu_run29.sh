timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu29.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu29.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu29.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b29_$name.json 2>gpurun_out/b29_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b29_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['quantize_ms'],4), d['config']['quantize_search'])" 2>&1 | tail -1
}
run c2 2 X=1
run c1 1 X=1
