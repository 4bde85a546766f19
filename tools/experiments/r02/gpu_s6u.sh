mkdir -p gpurun_out/s6u
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/s6u/ref.json 2> gpurun_out/s6u/ref.err; echo "ref rc=$?"
( time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s6u/ours.json 2> gpurun_out/s6u/ours.err ) 2>&1 | grep real; echo "ours rc=$?"
python -c "
import json
a=json.loads(open('gpurun_out/s6u/ours.json').read().strip().splitlines()[-1]); b=json.loads(open('gpurun_out/s6u/ref.json').read().strip().splitlines()[-1])
print('same config', a['config']==b['config'], 'value ratio', a['value']/b['value'], 'e2e ratio', a['e2e']['value']/b['e2e']['value'], a['ms_per_step'], a['clocks'])"
