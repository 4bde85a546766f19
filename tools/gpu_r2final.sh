# Round-2 final lines: every configuration + both arms + the launch list of the default command + ncu captures of the dominant kernels
mkdir -p gpurun_out/r2final
export NCU_DIR=/tmp/ncu_reps
run() { name=$1; shift; timeout 1500 python bench.py "$@" > gpurun_out/r2final/$name.json 2> gpurun_out/r2final/$name.err; echo "$name rc=$?"; }
run bench_cfg4
run bench_reference --impl reference
run bench_cfg2 --config 2
run bench_cfg3 --config 3
run bench_cfg1 --config 1
run bench_cfg6 --config 6
run bench_cfg5 --config 5 --steps 5 --warmup 3
run bench_cfg5h --config 5 --steps 5 --warmup 3 --leaves fp16
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2final/torchrun1_cfg2.json 2> gpurun_out/r2final/torchrun1_cfg2.err; echo "torchrun1 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2final/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2final/ncu_launches_cfg4.log 2>&1; echo "launches cfg4 rc=$?"
SKIP=0 timeout 900 bash tools/prof.sh w4 'apply_wide' --config 4 > gpurun_out/r2final/prof_w4.txt 2>&1
SKIP=1 timeout 900 bash tools/prof.sh q4 'quantize_lut' --config 4 > gpurun_out/r2final/prof_q4.txt 2>&1
SKIP=1 timeout 1200 bash tools/prof.sh k5 "apply_multi_staged" --config 5 --objects 4000000 > gpurun_out/r2final/prof_k5.txt 2>&1
for r in w4 q4 k5; do cp gpurun_out/${r}_by_opcode.txt gpurun_out/r2final/; python tools/ncu_summary.py $NCU_DIR/$r.ncu-rep --json gpurun_out/r2final/ncu_$r.json > /dev/null 2>&1; done
for f in gpurun_out/r2final/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('roofline_step') or {}).get('frac'), (d.get('verify') or {}).get('bit_exact'), (d.get('kernels') or {}))"; done
