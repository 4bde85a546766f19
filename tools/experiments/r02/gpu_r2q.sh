# K2w at configs 2/3 (forced) vs the K2 default; ring vs parameter-bank descriptors
mkdir -p gpurun_out/r2q
for c in 2 3; do
for v in "default:" "wide_ring:--path wide=1" "wide_bank:--path wide=1 --path desc_source=1"; do
  name=${v%%:*}; extra=${v#*:}
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $extra > gpurun_out/r2q/cfg${c}_$name.json 2>gpurun_out/r2q/cfg${c}_$name.err; echo "cfg$c $name rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r2q/cfg${c}_$name.json').read().strip().splitlines()[-1]);print('cfg$c $name', d['ms_per_step'], d['kernels']['apply_ms'], d['gpu_launches'], d['verify']['bit_exact'])"
done; done
