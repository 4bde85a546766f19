mkdir -p gpurun_out/s6r
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6r/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s6r/pytest.log
for c in 4 5; do
extra=""; [ $c = 5 ] && extra="--steps 4 --warmup 3"
timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline $extra > gpurun_out/s6r/cfg$c.json 2> gpurun_out/s6r/cfg$c.err
python -c "
import json;d=json.loads(open('gpurun_out/s6r/cfg$c.json').read().strip().splitlines()[-1])
print('cfg$c', d['ms_per_step'], d['kernels']['quantize_ms'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done
