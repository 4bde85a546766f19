mkdir -p gpurun_out/s6k
timeout 900 python tests/stress/repro_buckets.py 2000 150001 80 > gpurun_out/s6k/b.log 2>&1; tail -25 gpurun_out/s6k/b.log | cut -c1-600
