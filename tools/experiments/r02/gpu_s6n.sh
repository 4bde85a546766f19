# after the proxy-fence release: the K1L repro, every config's kernel times, the full GPU suite
mkdir -p gpurun_out/s6n
timeout 600 python tests/stress/repro_buckets.py 2000 150001 150 > gpurun_out/s6n/repro.log 2>&1; echo "repro: $(tail -1 gpurun_out/s6n/repro.log)"
timeout 600 python tests/stress/repro_rowblocks.py 2000 150001 60 quant_lut=0 > gpurun_out/s6n/repro_k1t.log 2>&1; echo "repro K1t: $(tail -1 gpurun_out/s6n/repro_k1t.log)"
for c in 4 2 3 1 6 5; do
extra=""; [ $c = 5 ] && extra="--steps 4 --warmup 3"
timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline $extra > gpurun_out/s6n/cfg$c.json 2> gpurun_out/s6n/cfg$c.err
python -c "
import json;d=json.loads(open('gpurun_out/s6n/cfg$c.json').read().strip().splitlines()[-1])
print('cfg$c', d['ms_per_step'], d['kernels']['quantize_ms'], d['kernels']['apply_ms'], d['verify'].get('bit_exact'))"
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6n/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s6n/pytest.log
