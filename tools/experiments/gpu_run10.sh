run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b10_$name.json 2>gpurun_out/b10_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b10_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['apply_ms'],3))" 2>&1 | tail -1
}
for k in 1 2 3; do run c5_k4_cta$k 5 OBT_MULTI_CTAS_PER_SM=$k; run c5_slice_cta$k 5 OBT_MULTI_SLICE=1 OBT_MULTI_CTAS_PER_SM=$k; done
