# K5 with split binary64 records (no F2F): multi-output parity, cfg5 A/B (480 vs 512 consumers), ncu
mkdir -p gpurun_out/r2j
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or output or staged or cfg5 or config5" > gpurun_out/r2j/pytest_multi.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2j/pytest_multi.log
L=paper_2211_00391_b200/_lib
for v in default k5_512; do
  if [ $v = default ]; then lib=$L/libobtree_b200.so; else lib=$L/$v/libobtree_b200.so; fi
  OBTREE_B200_LIB=$PWD/$lib timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r2j/cfg5_$v.json 2>gpurun_out/r2j/cfg5_$v.err; echo "$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2j/cfg5_$v.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'], d['kernels']['apply_ms'], d['verify'])"
done
export NCU_DIR=/tmp/ncu_reps
SKIP=0 timeout 1200 bash tools/prof.sh k5b 'apply_multi_staged' --config 5 > gpurun_out/r2j/prof_k5b.txt 2>&1; head -c 1500 gpurun_out/r2j/prof_k5b.txt
cp /tmp/ncu_reps/k5b.ncu-rep gpurun_out/r2j/ 2>/dev/null; cp gpurun_out/k5b_by_opcode.txt gpurun_out/r2j/
