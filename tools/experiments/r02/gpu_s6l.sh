mkdir -p gpurun_out/s6l
for v in 1 2 3; do
OBTREE_B200_LIB=$PWD/paper_2211_00391_b200/_lib/k1l$v/libobtree_b200.so timeout 600 python tests/stress/repro_buckets.py 2000 150001 100 > gpurun_out/s6l/v$v.log 2>&1; echo "variant $v: $(tail -1 gpurun_out/s6l/v$v.log)"
done
