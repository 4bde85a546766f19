timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu6.log
for c in 2 4 5; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b6_cfg$c.json 2>gpurun_out/b6_cfg$c.err; echo "bench $c rc=$?"
python -c "import json;d=json.load(open('gpurun_out/b6_cfg$c.json'));print($c, d['ms_per_step'], d['value'], d['kernels'])"
done
OBT_QUANT_LUT=0 timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b6_nolut.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/b6_nolut.json'));print('nolut', d['ms_per_step'], d['kernels'])"
SKIP=1 timeout 600 bash tools/prof.sh fq2lut 'quantize_lut' --config 2 > gpurun_out/prof_fq2lut.txt 2>&1; echo "prof rc=$?"
head -3 gpurun_out/prof_fq2lut.txt
python tools/ncu_source_summary.py gpurun_out/fq2lut.ncu-rep > gpurun_out/fq2lut_by_opcode.txt 2>&1; head -14 gpurun_out/fq2lut_by_opcode.txt
