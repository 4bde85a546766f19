mkdir -p gpurun_out/s6a
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6a/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s6a/pytest.log
timeout 900 python bench.py > gpurun_out/s6a/bench_cfg4.json 2> gpurun_out/s6a/bench_cfg4.err; echo "cfg4 rc=$?"; tail -c 3000 gpurun_out/s6a/bench_cfg4.json
