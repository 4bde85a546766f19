set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"
cat gpurun_out/bench_cfg2.json
timeout 600 bash tools/prof.sh fa2p 'apply_kernel' --config 2 > gpurun_out/prof_fa2p.txt 2>&1; echo "prof rc=$?"
cat gpurun_out/prof_fa2p.txt | head -40
