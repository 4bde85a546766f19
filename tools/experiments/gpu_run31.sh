timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu31.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu31.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu31.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b31_$name.json 2>gpurun_out/b31_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b31_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'], d.get('cpu_baseline'))" 2>&1 | tail -1
}
run c2 2 X=1
run c2_nopdl 2 OBT_PDL=0
run c3 3 X=1
run c3_nopdl 3 OBT_PDL=0
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --cpu-seconds 3 > gpurun_out/b31_verify.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/b31_verify.json').read().strip().splitlines()[-1]);print('verify', d['cpu_baseline']['gpu_verified_bit_exact'], d['ms_per_step'])"
