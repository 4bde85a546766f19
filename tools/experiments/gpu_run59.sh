run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b59_$name.json 2>gpurun_out/b59_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b59_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['quantize_ms'],4), round(d['kernels']['apply_ms'],4))" 2>&1 | tail -1
}
L=paper_2211_00391_b200/_lib/el/libobtree_b200.so
run c2_base 2 X=1
run c2_el 2 OBTREE_B200_LIB=$L
run c2_baseb 2 X=1
run c2_elb 2 OBTREE_B200_LIB=$L
