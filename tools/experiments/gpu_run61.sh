timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu61.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu61.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu61.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b61_$name.json 2>gpurun_out/b61_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b61_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['apply_ms'],4))" 2>&1 | tail -1
}
run c2_tab 2 X=1
run c2_full 2 OBT_PARAM_TABLES=0
run c2_tabb 2 X=1
run c2_fullb 2 OBT_PARAM_TABLES=0
run c3_tab 3 X=1
run c3_full 3 OBT_PARAM_TABLES=0
