timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu14.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu14.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu14.log | head
timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b14_c5.json 2>gpurun_out/b14_c5.err
python -c "import json;d=json.load(open('gpurun_out/b14_c5.json'));print('c5', round(d['ms_per_step'],4), d['kernels'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
SKIP=0 timeout 600 bash tools/prof.sh fa2main 'apply_kernel' --config 2 > gpurun_out/prof_fa2main.txt 2>&1; head -2 gpurun_out/prof_fa2main.txt
SKIP=0 timeout 600 bash tools/prof.sh fs2tail 'apply_split' --config 2 > gpurun_out/prof_fs2tail.txt 2>&1; head -2 gpurun_out/prof_fs2tail.txt
SKIP=1 timeout 600 bash tools/prof.sh fq2lut 'quantize_lut' --config 2 > gpurun_out/prof_fq2lut.txt 2>&1; head -2 gpurun_out/prof_fq2lut.txt
for r in fa2main fs2tail fq2lut; do python tools/ncu_source_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_by_opcode.txt 2>&1; done
