timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu45.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu45.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu45.log | head
