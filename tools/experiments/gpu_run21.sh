timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu21.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu21.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu21.log | head
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b21_c5.json 2>gpurun_out/b21_c5.err; echo "bench rc=$?"; cat gpurun_out/b21_c5.json
