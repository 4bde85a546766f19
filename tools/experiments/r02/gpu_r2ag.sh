mkdir -p gpurun_out/r2ag
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "large_feature" > gpurun_out/r2ag/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2ag/pytest.log
timeout 900 python bench.py --config 6 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ag/cfg6.json 2>gpurun_out/r2ag/cfg6.err; echo "cfg6 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2ag/cfg6.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['kernels'], d['verify']['bit_exact'])"
