#!/bin/bash
# Build the native library with extra nvcc defines into _lib/<name>/ (tuning experiments):
#   tools/build_variant.sh l2_128 -DOBT_QUANT_L2HINT='".L2::128B"'
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/paper_2211_00391_b200/_lib/$name
mkdir -p "$out"
objs=()
for src in "$root"/paper_2211_00391_b200/csrc/*.cu; do
  o=$out/$(basename "${src%.cu}").o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -c -o "$o" "$src" &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libobtree_b200.so" "${objs[@]}"
echo "$out/libobtree_b200.so"
