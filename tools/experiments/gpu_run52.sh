timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu52.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu52.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu52.log | head
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b52_$name.json 2>gpurun_out/b52_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b52_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'])" 2>&1 | tail -1
}
run c3 3 X=1
run c3_nof2 3 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/nof2/libobtree_b200.so
run c3b 3 X=1
run c3_nof2b 3 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/nof2/libobtree_b200.so
