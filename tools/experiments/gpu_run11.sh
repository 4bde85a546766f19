timeout 900 python -m pytest tests -m gpu -x -q -k "multi" > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu11.log
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b11_$name.json 2>gpurun_out/b11_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b11_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['apply_ms'],3))" 2>&1 | tail -1
}
run c5_k4_persist 5 X=1
run c5_slice_persist 5 OBT_MULTI_SLICE=1
run c5_k4_nopersist 5 OBT_MULTI_PERSIST=0
