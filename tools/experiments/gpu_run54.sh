run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b54_$name.json 2>gpurun_out/b54_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b54_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['quantize_ms'],4))" 2>&1 | tail -1
}
run c2 2 X=1
run c2_one 2 OBT_QUANT_ONE_CTA=1
run c4 4 X=1
run c4_one 4 OBT_QUANT_ONE_CTA=1
run c5 5 X=1
run c5_one 5 OBT_QUANT_ONE_CTA=1
