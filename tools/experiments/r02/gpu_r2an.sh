# K2w at config 4: descriptor ring vs parameter bank after the producer split
mkdir -p gpurun_out/r2an
for a in "desc_source=0" "desc_source=1"; do
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --path $a > gpurun_out/r2an/$a.json 2>gpurun_out/r2an/$a.err; echo "$a rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r2an/$a.json').read().strip().splitlines()[-1]);print('$a', d['ms_per_step'], d.get('kernels'), d['verify']['bit_exact'])"
done
