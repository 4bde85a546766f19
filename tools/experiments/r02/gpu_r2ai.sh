# K1L persistent CTAs (tables staged once, continuous ring) vs one CTA per row block
mkdir -p gpurun_out/r2ai
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_configs.py -m gpu -x -q -k "cell_table or quantize or full_model or fuzz" > gpurun_out/r2ai/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2ai/pytest.log
L=paper_2211_00391_b200/_lib
for v in default k1lnp; do
  if [ $v = default ]; then lib=$L/libobtree_b200.so; else lib=$L/$v/libobtree_b200.so; fi
  for c in 2 4; do
  OBTREE_B200_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2ai/cfg${c}_$v.json 2>gpurun_out/r2ai/cfg${c}_$v.err; echo "$v $c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2ai/cfg${c}_$v.json').read().strip().splitlines()[-1]);print('$v cfg$c', d['ms_per_step'], d['kernels']['quantize_ms'], d['kernels']['apply_ms'], d['verify']['bit_exact'])"
  done
done
