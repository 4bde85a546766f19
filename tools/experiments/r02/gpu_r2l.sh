# full GPU suite after the path-option refactor; default bench cfg4 + cfg2 quick
mkdir -p gpurun_out/r2l
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2l/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2l/pytest.log
for c in 2 4; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2l/cfg$c.json 2>gpurun_out/r2l/cfg$c.err; echo "cfg$c rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2l/cfg$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d['kernels']['apply_ms'], d['kernels']['quantize_ms'], d['verify']['bit_exact'])"
done
