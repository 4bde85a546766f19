# Round measurements: every config's bench line, the reference arm, the cfg2 launch list
# and ncu captures of the dominant kernels (each after its own plain run exits 0).
mkdir -p gpurun_out/final
export NCU_DIR=/tmp/ncu_reps
timeout 900 python bench.py > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config 1 > gpurun_out/final/bench_cfg1.json 2> gpurun_out/final/bench_cfg1.err; echo "cfg1 rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/final/bench_cfg3.json 2> gpurun_out/final/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 1200 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_cfg4.json 2> gpurun_out/final/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/bench_cfg5.json 2> gpurun_out/final/bench_cfg5.err; echo "cfg5 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_launches.log 2>&1; echo "launches rc=$?"
SKIP=0 timeout 600 bash tools/prof.sh fa2main 'apply_kernel' --config 2 > gpurun_out/final/prof_fa2main.txt 2>&1
SKIP=2 timeout 600 bash tools/prof.sh fa2last 'apply_kernel' --config 2 > gpurun_out/final/prof_fa2last.txt 2>&1
SKIP=1 timeout 600 bash tools/prof.sh fq2lut 'quantize_lut' --config 2 > gpurun_out/final/prof_fq2lut.txt 2>&1
SKIP=0 timeout 900 bash tools/prof.sh fs4main 'apply_split' --config 4 > gpurun_out/final/prof_fs4main.txt 2>&1
for r in fa2main fa2last fq2lut fs4main; do cp gpurun_out/${r}_by_opcode.txt gpurun_out/final/; done
cat gpurun_out/final/prof_*.txt | cut -c1-300
for f in gpurun_out/final/bench_*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'))"; done
SKIP=0 timeout 900 bash tools/prof.sh fa5staged 'apply_multi_staged' --config 5 > gpurun_out/final/prof_fa5staged.txt 2>&1; head -c 600 gpurun_out/final/prof_fa5staged.txt
cp gpurun_out/fa5staged_by_opcode.txt gpurun_out/final/
SKIP=0 timeout 900 bash tools/prof.sh fq4lut 'quantize_lut' --config 4 > gpurun_out/final/prof_fq4lut.txt 2>&1; head -c 600 gpurun_out/final/prof_fq4lut.txt
