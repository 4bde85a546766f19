mkdir -p gpurun_out/s7a
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,launch__grid_size,launch__block_size --clock-control none -k regex:"quantize|apply" -c 40 --csv --log-file gpurun_out/s7a/launches_cfg1.csv python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph off > gpurun_out/s7a/ncu.log 2>&1; echo rc=$?
python - <<'PY'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/s7a/launches_cfg1.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=collections.defaultdict(dict)
for r in rows[1:]: d[(r[ii],r[ki][:50])][r[mi]]=r[vi]
for k,v in list(d.items())[-6:]: print(k, v)
PY
