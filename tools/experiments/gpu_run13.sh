run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b13_$name.json 2>gpurun_out/b13_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b13_$name.json'));print('$name', round(d['ms_per_step'],4), round(d['kernels']['apply_ms'],3))" 2>&1 | tail -1
}
run default 5 X=1
for v in a0m4 a1m4 a1m1 head; do run $v 5 OBTREE_B200_LIB=paper_2211_00391_b200/_lib/$v/libobtree_b200.so; done
run default_again 5 X=1
