# K2w double-buffered bucket tiles (where they fit): parity, config 2/3 forced K2w, config 4
mkdir -p gpurun_out/r2ad
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide" > gpurun_out/r2ad/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ad/pytest.log
for c in 2 3; do
for v in "default:" "wide_ring:--path wide=1" "wide_bank:--path wide=1 --path desc_source=1"; do
  name=${v%%:*}; extra=${v#*:}
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $extra > gpurun_out/r2ad/cfg${c}_$name.json 2>gpurun_out/r2ad/cfg${c}_$name.err; echo "cfg$c $name rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2ad/cfg${c}_$name.json').read().strip().splitlines()[-1]);print('cfg$c $name', d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
done; done
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2ad/cfg4.json 2>gpurun_out/r2ad/cfg4.err
python -c "import json;d=json.loads(open('gpurun_out/r2ad/cfg4.json').read().strip().splitlines()[-1]);print('cfg4', d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
