mkdir -p gpurun_out/s6s
timeout 2400 python tests/stress/stress_determinism.py 30 > gpurun_out/s6s/stress.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/s6s/stress.log | cut -c1-300
