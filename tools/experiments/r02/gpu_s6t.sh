mkdir -p gpurun_out/s6t
timeout 2400 python tests/stress/stress_full_size.py 4 > gpurun_out/s6t/full.log 2>&1; echo "rc=$?"; tail -8 gpurun_out/s6t/full.log | cut -c1-300
