timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu64.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu64.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu64.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b64.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/b64.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step'])"
