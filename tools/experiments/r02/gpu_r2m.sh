mkdir -p gpurun_out/r2m
timeout 1800 python -m pytest tests/test_full_configs.py -m gpu -x -q -rA > gpurun_out/r2m/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2m/pytest_full.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/r2m/ref.json 2> gpurun_out/r2m/ref.err; echo "ref rc=$?"; tail -c 1200 gpurun_out/r2m/ref.json
