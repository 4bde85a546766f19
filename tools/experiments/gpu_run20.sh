timeout 900 python -m pytest tests -m gpu -x -q -k "multi" > gpurun_out/pytest_gpu20.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu20.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu20.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b20_$name.json 2>gpurun_out/b20_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b20_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels'])" 2>&1 | tail -1
}
run c5_staged 5 X=1
run c5_k4 5 OBT_MULTI_STAGED=0
SKIP=0 timeout 900 bash tools/prof.sh fa5staged 'apply_multi_staged' --config 5 > gpurun_out/prof_fa5staged.txt 2>&1; cut -c1-1200 gpurun_out/prof_fa5staged.txt
python tools/ncu_source_summary.py gpurun_out/fa5staged.ncu-rep > gpurun_out/fa5staged_by_opcode.txt 2>&1; head -14 gpurun_out/fa5staged_by_opcode.txt
