#!/bin/bash
# Recompile the named translation units (default: k_wide obtree_capi) and relink the
# in-tree library (iteration helper; __graft_entry__.build() is the full build).
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
lib=$root/paper_2211_00391_b200/_lib
units=${@:-k_wide obtree_capi}
pids=()
for u in $units; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
    -c -o "$lib/obj/$u.o" "$root/paper_2211_00391_b200/csrc/$u.cu" > "$lib/ptxas_$u.log" 2>&1 &
  pids+=($!)
done
for i in "${!pids[@]}"; do
  if ! wait "${pids[$i]}"; then echo "FAILED: $(echo $units | cut -d' ' -f$((i + 1)))"; grep -i error "$lib"/ptxas_*.log | head; exit 1; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$lib/libobtree_b200.so" "$lib"/obj/*.o
echo ok
