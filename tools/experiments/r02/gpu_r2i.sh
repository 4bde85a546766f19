# K5 study: gather microbenchmarks + ncu source-level capture of K5 at cfg5
mkdir -p gpurun_out/r2i
timeout 120 ./tools/microbench_gather > gpurun_out/r2i/microbench_gather.txt 2>&1; cat gpurun_out/r2i/microbench_gather.txt
export NCU_DIR=/tmp/ncu_reps
SKIP=0 timeout 1200 bash tools/prof.sh k5 'apply_multi_staged' --config 5 > gpurun_out/r2i/prof_k5.txt 2>&1; head -c 1500 gpurun_out/r2i/prof_k5.txt
cp /tmp/ncu_reps/k5.ncu-rep gpurun_out/r2i/ 2>/dev/null; cp gpurun_out/k5_by_opcode.txt gpurun_out/r2i/; tail -3 gpurun_out/plain_k5.log | cut -c1-600
