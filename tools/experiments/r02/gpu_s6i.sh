mkdir -p gpurun_out/s6i
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6i/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s6i/pytest.log
timeout 900 python bench.py > gpurun_out/s6i/bench_cfg4.json 2> gpurun_out/s6i/bench_cfg4.err; echo "cfg4 rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/s6i/bench_cfg4.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_step']['frac'], d['kernels'], d['verify'])"
