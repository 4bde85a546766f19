timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "repeated_predicts or stage_release" 2>&1 | tail -3
timeout 900 python tests/stress/stress_determinism.py 5 2>&1 | tail -3 | cut -c1-200
