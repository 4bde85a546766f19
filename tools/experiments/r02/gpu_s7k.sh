# round-2 captures at config 2 (K2 chained parameter-bank launches, K1L) and its launch list
mkdir -p gpurun_out/s7k
export NCU_DIR=/tmp/ncu_reps
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s7k/launches_cfg2.csv python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s7k/ncu_launches_cfg2.log 2>&1; echo "launches cfg2 rc=$?"
SKIP=9 timeout 900 bash tools/prof.sh a2 'apply_kernel' --config 2 > gpurun_out/s7k/prof_a2.txt 2>&1
SKIP=3 timeout 900 bash tools/prof.sh q2 'quantize_lut' --config 2 > gpurun_out/s7k/prof_q2.txt 2>&1
for r in a2 q2; do cp gpurun_out/${r}_by_opcode.txt gpurun_out/s7k/; done
head -c 700 gpurun_out/s7k/prof_a2.txt; echo; head -c 500 gpurun_out/s7k/prof_q2.txt
