mkdir -p gpurun_out/r2y
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_predict or host" > gpurun_out/r2y/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2y/pytest.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2y/cfg4.json 2>gpurun_out/r2y/cfg4.err; echo "rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2y/cfg4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e_pageable']['ms_per_step'], d['verify']['bit_exact'])"
timeout 900 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2y/cfg2.json 2>gpurun_out/r2y/cfg2.err; echo "rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2y/cfg2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e_pageable']['ms_per_step'], d['verify']['bit_exact'])"
