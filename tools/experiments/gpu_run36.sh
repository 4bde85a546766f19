timeout 1200 python -m pytest tests -m gpu -x -q -k "fan or smoke or batch" > gpurun_out/pytest_gpu36.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu36.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu36.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/b36_$name.json 2>gpurun_out/b36_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b36_$name.json'));print('$name', round(d['ms_per_step']*1000,2), 'us', d['kernels'])" 2>&1 | tail -1
}
run c1 1 X=1
run c1_nofan 1 OBT_FAN=0
SKIP=3 timeout 600 bash tools/prof.sh fan1b 'apply_fan' --config 1 --graph off > gpurun_out/prof_fan1b.txt 2>&1; head -c 700 gpurun_out/prof_fan1b.txt; echo; head -8 gpurun_out/fan1b_by_opcode.txt
