# fused K2f (in-kernel quantize) for small batches: parity + config 1 A/B
mkdir -p gpurun_out/r2ae
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused_small or fanned" > gpurun_out/r2ae/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ae/pytest.log
for v in "fused:" "separate:--path fan_fuse=0"; do
  name=${v%%:*}; extra=${v#*:}
  for g in on off; do
  timeout 600 python bench.py --config 1 --steps 50 --warmup 10 --no-e2e --no-cpu-baseline --graph $g $extra > gpurun_out/r2ae/cfg1_${name}_$g.json 2>gpurun_out/r2ae/cfg1_${name}_$g.err; echo "$name $g rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2ae/cfg1_${name}_$g.json').read().strip().splitlines()[-1]);print('$name $g', d['ms_per_step']*1000, 'us', d['kernels'], d['verify']['bit_exact'])"
  done
done
