mkdir -p gpurun_out/s6z
for i in 1 2 3; do timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6z/pytest$i.log 2>&1; echo "pytest run $i rc=$?: $(tail -1 gpurun_out/s6z/pytest$i.log)"; done
timeout 900 python tests/stress/stress_determinism.py 40 > gpurun_out/s6z/stress.log 2>&1; grep -c "0 differing" gpurun_out/s6z/stress.log; grep -v "0 differing" gpurun_out/s6z/stress.log | head -5
timeout 900 python tests/stress/repro_buckets.py 2000 150001 200 > gpurun_out/s6z/repro.log 2>&1; tail -1 gpurun_out/s6z/repro.log
timeout 900 python tests/stress/repro_buckets.py 500 620001 100 > gpurun_out/s6z/repro500.log 2>&1; tail -1 gpurun_out/s6z/repro500.log
