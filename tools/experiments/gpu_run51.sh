for c in 2 3 4 1; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b51_$c.json 2>gpurun_out/b51_$c.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/b51_$c.json').read().strip().splitlines()[-1]);print($c, d['ms_per_step'], d.get('roofline_smem'))"
done
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b51_5.json 2>gpurun_out/b51_5.err; echo rc5=$?; tail -c 200 gpurun_out/b51_5.json
