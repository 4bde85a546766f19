# large-F single-output models on the record path: parity + the epsilon8k64 shape
mkdir -p gpurun_out/r2af
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_configs.py -m gpu -x -q -k "large_feature or multi or full_model" > gpurun_out/r2af/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2af/pytest.log
timeout 900 python bench.py --config 6 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2af/cfg6.json 2>gpurun_out/r2af/cfg6.err; echo "cfg6 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2af/cfg6.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['kernels'], d['verify']['bit_exact'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline_step']['frac'])"
timeout 900 python bench.py --config 6 --steps 3 --warmup 2 --impl reference > gpurun_out/r2af/cfg6_ref.json 2>gpurun_out/r2af/cfg6_ref.err; echo "ref rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2af/cfg6_ref.json').read().strip().splitlines()[-1]);print(d['value'], d['cpu_baseline'].get('reference_pkg',{}).get('value_1core'))"
