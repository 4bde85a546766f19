# shuffle "permute" leaf selection: parity + config 3 A/B
mkdir -p gpurun_out/r2v
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "permute or descriptor_sources or depth_split" > gpurun_out/r2v/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2v/pytest.log
for v in "gather:" "permute:--path leaf_select=1"; do
  name=${v%%:*}; extra=${v#*:}
  timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $extra > gpurun_out/r2v/cfg3_$name.json 2>gpurun_out/r2v/cfg3_$name.err; echo "$name rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2v/cfg3_$name.json').read().strip().splitlines()[-1]);print('$name', d['ms_per_step'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
done
