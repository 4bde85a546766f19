# K1L: row stages issued before vs after the table copy, 1 and 8 row blocks per CTA
mkdir -p gpurun_out/r2aq
L=paper_2211_00391_b200/_lib
for v in rb1 rb1late rb8 rb8late; do
  if [ $v = default ]; then lib=$L/libobtree_b200.so; else lib=$L/$v/libobtree_b200.so; fi
  for c in 4 2; do
    OBTREE_B200_LIB=$PWD/$lib timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2aq/$v-$c.json 2>gpurun_out/r2aq/$v-$c.err; echo "$v cfg$c rc=$?"
    python -c "import json;d=json.loads(open('gpurun_out/r2aq/$v-$c.json').read().strip().splitlines()[-1]);k=d['kernels'];print('$v cfg$c', d['ms_per_step'], k['quantize_ms'], k['quantize_frac_hbm'], d['verify']['bit_exact'])"
  done
done
