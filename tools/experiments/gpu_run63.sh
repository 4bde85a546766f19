run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b63_$name.json 2>gpurun_out/b63_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b63_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['quantize_ms'],4), d['config']['quantize_search'])" 2>&1 | tail -1
}
run c4 4 X=1
run c4_512 4 OBT_LUT_CELLS=512
run c5_512 5 OBT_LUT_CELLS=512 OBT_QUANT_LUT=1
run c5 5 X=1
