mkdir -p gpurun_out/r2as
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2as/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2as/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2as/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2as/smoke.log
