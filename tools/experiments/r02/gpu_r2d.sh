# K2w v2 (transposed panel, 8 fold warps): parity, then cfg4 A/B over index-warp counts
mkdir -p gpurun_out/r2d
mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k wide > gpurun_out/r2d/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -3 gpurun_out/r2d/pytest_wide.log
L=paper_2211_00391_b200/_lib
for v in default nidx4 nidx8; do
  if [ $v = default ]; then lib=$L/libobtree_b200.so; else lib=$L/$v/libobtree_b200.so; fi
  OBTREE_B200_LIB=$PWD/$lib OBT_WIDE=1 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2d/cfg4_$v.json 2>gpurun_out/r2d/cfg4_$v.err; echo "$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2d/cfg4_$v.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
done
export NCU_DIR=/tmp/ncu_reps
OBT_WIDE=1 SKIP=0 timeout 900 bash tools/prof.sh w4c 'apply_wide' --config 4 > gpurun_out/r2d/prof_w4c.txt 2>&1; head -c 1500 gpurun_out/r2d/prof_w4c.txt
cp /tmp/ncu_reps/w4c.ncu-rep gpurun_out/r2d/ 2>/dev/null; cp gpurun_out/w4c_by_opcode.txt gpurun_out/r2d/
