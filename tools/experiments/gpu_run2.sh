SKIP=0 timeout 600 bash tools/prof.sh fa2main 'apply_kernel' --config 2 > gpurun_out/prof_fa2main.txt 2>&1; echo "prof rc=$?"
cat gpurun_out/prof_fa2main.txt | head -40
python tools/ncu_source_summary.py gpurun_out/fa2main.ncu-rep > gpurun_out/fa2main_by_opcode.txt 2>&1
cat gpurun_out/fa2main_by_opcode.txt
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench5 rc=$?"
cat gpurun_out/bench_cfg5.json
