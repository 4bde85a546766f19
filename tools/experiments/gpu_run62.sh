run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b62_$name.json 2>gpurun_out/b62_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b62_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['apply_ms'],4))" 2>&1 | tail -1
}
run c2_s2 2 X=1
run c2_s3 2 OBT_PARAM_STAGES=3
run c2_s2b 2 X=1
run c2_s3b 2 OBT_PARAM_STAGES=3
timeout 1200 python -m pytest tests -m gpu -q -k "chained or descriptor or smoke" > gpurun_out/pytest_gpu62.log 2>&1; tail -1 gpurun_out/pytest_gpu62.log
OBT_PARAM_STAGES=3 timeout 1200 python -m pytest tests -m gpu -q -k "chained or descriptor or smoke or bit_exact_batch" > gpurun_out/pytest_gpu62b.log 2>&1; tail -1 gpurun_out/pytest_gpu62b.log
