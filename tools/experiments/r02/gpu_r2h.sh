# full GPU suite + smoke + default bench (cfg4) after the K2w rework
mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2h/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2h/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2h/smoke.log
timeout 1500 python bench.py > gpurun_out/r2h/bench_default.json 2> gpurun_out/r2h/bench_default.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2h/bench_default.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernels'], d['verify'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline_step']['frac'])"
