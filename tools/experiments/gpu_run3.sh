timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu3.log
for c in 2 3 4; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b3_cfg$c.json 2>gpurun_out/b3_cfg$c.err; echo "bench $c rc=$?"
python -c "import json;d=json.load(open('gpurun_out/b3_cfg$c.json'));print($c, d['ms_per_step'], d['value'], d['kernels'])"
done
