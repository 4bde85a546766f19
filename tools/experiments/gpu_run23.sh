timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --graph off > gpurun_out/ncu_l1.log 2>&1; echo rc=$?
python3 - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_cfg1.csv')) if len(r)>5]
hdr=rows[0]; ix={h:i for i,h in enumerate(hdr)}
for r in rows[-12:]: print(r[ix['Kernel Name']][:60], r[ix['Metric Name']], r[ix['Metric Value']])
P
