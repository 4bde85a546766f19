timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu8.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu8.log | head -10
run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b8_$name.json 2>gpurun_out/b8_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b8_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['quantize_ms'],4), round(d['kernels']['apply_ms'],3), d['config'].get('quantize_search'))" 2>&1 | tail -1
}
run c5 5 X=1
run c5_k4 5 OBT_MULTI_SLICE=0
run c2 2 X=1
run c2_noalign 2 OBT_QUANT_ALIGN=0
run c2_nolut 2 OBT_QUANT_LUT=0
run c2_nolut_noalign 2 OBT_QUANT_LUT=0 OBT_QUANT_ALIGN=0
run c2_l2n 2 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/l2n/libobtree_b200.so
run c2_l2x 2 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/l2x/libobtree_b200.so
run c4 4 X=1
run c4_nolut 4 OBT_QUANT_LUT=0
run c4_nolut_noalign 4 OBT_QUANT_LUT=0 OBT_QUANT_ALIGN=0
