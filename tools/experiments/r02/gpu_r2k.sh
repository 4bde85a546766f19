# K5: last record row as an 8-byte load; microbench + parity + cfg5 bench
mkdir -p gpurun_out/r2k
timeout 120 ./tools/microbench_gather > gpurun_out/r2k/microbench_gather.txt 2>&1; cat gpurun_out/r2k/microbench_gather.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or output" > gpurun_out/r2k/pytest_multi.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2k/pytest_multi.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r2k/cfg5.json 2>gpurun_out/r2k/cfg5.err; echo "rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2k/cfg5.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
