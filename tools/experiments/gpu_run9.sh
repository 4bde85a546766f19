timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu9.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu9.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu9.log | head -10
timeout 900 python bench.py > gpurun_out/b9_default.json 2>gpurun_out/b9_default.err; echo "bench rc=$?"; cat gpurun_out/b9_default.json
SKIP=0 timeout 900 bash tools/prof.sh fa5k4 'apply_multi' --config 5 > gpurun_out/prof_fa5k4.txt 2>&1; head -3 gpurun_out/prof_fa5k4.txt
OBT_MULTI_SLICE=1 SKIP=0 timeout 900 bash tools/prof.sh fa5slice 'apply_multi' --config 5 > gpurun_out/prof_fa5slice.txt 2>&1; head -3 gpurun_out/prof_fa5slice.txt
