timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu4.log
for c in 2 3 4; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b4_cfg$c.json 2>gpurun_out/b4_cfg$c.err; echo "bench $c rc=$?"
python -c "import json;d=json.load(open('gpurun_out/b4_cfg$c.json'));print($c, d['ms_per_step'], d['value'], d['kernels'])"
done
for v in pf2 pf0 st3; do
OBTREE_B200_LIB=paper_2211_00391_b200/_lib/$v/libobtree_b200.so timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b4_$v.json 2>gpurun_out/b4_$v.err; echo "bench $v rc=$?"
python -c "import json;d=json.load(open('gpurun_out/b4_$v.json'));print('$v', d['ms_per_step'], d['value'], d['kernels'])"
done
SKIP=0 timeout 600 bash tools/prof.sh fa2pipe 'apply_kernel' --config 2 > gpurun_out/prof_fa2pipe.txt 2>&1; echo "prof rc=$?"
cat gpurun_out/prof_fa2pipe.txt | head -5
python tools/ncu_source_summary.py gpurun_out/fa2pipe.ncu-rep > gpurun_out/fa2pipe_by_opcode.txt 2>&1; head -12 gpurun_out/fa2pipe_by_opcode.txt
