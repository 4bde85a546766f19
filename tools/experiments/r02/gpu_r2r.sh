# binary16 multi-output (half2 records): parity, cfg5 fp32 (regression) and fp16 benches
mkdir -p gpurun_out/r2r
timeout 900 python -m pytest tests -m gpu -x -q -k "multi or output or full_model" > gpurun_out/r2r/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2r/pytest.log
for lv in fp32 fp16; do
timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --leaves $lv > gpurun_out/r2r/cfg5_$lv.json 2>gpurun_out/r2r/cfg5_$lv.err; echo "$lv rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2r/cfg5_$lv.json').read().strip().splitlines()[-1]);print('$lv', d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'], d.get('fp16_vs_fp32'))"
done
