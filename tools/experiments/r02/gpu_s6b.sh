mkdir -p gpurun_out/s6b
timeout 900 python -m pytest tests/test_local_sharded_gpu.py -m gpu -x -q > gpurun_out/s6b/pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/s6b/pytest.log
