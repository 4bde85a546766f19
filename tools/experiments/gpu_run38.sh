timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu38.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu38.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu38.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
mkdir -p gpurun_out/final
timeout 600 python bench.py --config 1 > gpurun_out/final/bench_cfg1.json 2> gpurun_out/final/bench_cfg1.err; echo "cfg1 rc=$?"; tail -c 600 gpurun_out/final/bench_cfg1.json
