mkdir -p gpurun_out/s7e
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s7e/pytest.log 2>&1; echo "pytest rc=$?: $(tail -1 gpurun_out/s7e/pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels'], d['verify']['bit_exact'])"
