run() { # name config env...
  name=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b50_$name.json 2>gpurun_out/b50_$name.err
  python -c "import json;d=json.load(open('gpurun_out/b50_$name.json'));print('$name', round(d['ms_per_step'],4), d['kernels']['apply_ms'], d['gpu_launches'])" 2>&1 | tail -1
}
L=paper_2211_00391_b200/_lib/g16/libobtree_b200.so
run c2 2 X=1
run c2_g16 2 OBTREE_B200_LIB=$L
run c2_g16_t512_ct16 2 OBTREE_B200_LIB=$L OBT_TILE=512 OBT_CHUNK_TREES=16
run c2_g16_t512_ct32 2 OBTREE_B200_LIB=$L OBT_TILE=512 OBT_CHUNK_TREES=32
run c2_t512 2 OBT_TILE=512
run c3_g16_t512_ct16 3 OBTREE_B200_LIB=$L OBT_TILE=512 OBT_CHUNK_TREES=16
