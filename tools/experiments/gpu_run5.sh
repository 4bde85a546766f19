# apply pipeline-depth sweep at cfg2 (default build = PF 2, LAG 1) and cfg4
for v in default pf3l1 pf4l1 pf2l2 pf3l2; do
  if [ $v = default ]; then lib=""; else lib=paper_2211_00391_b200/_lib/$v/libobtree_b200.so; fi
  for c in 2 4; do
  OBTREE_B200_LIB=$lib timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b5_${v}_$c.json 2>gpurun_out/b5_${v}_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b5_${v}_$c.json'));print('$v', $c, round(d['ms_per_step'],4), d['kernels']['apply_ms'])"
  done
done
