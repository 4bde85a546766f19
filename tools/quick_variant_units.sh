#!/bin/bash
# quick_variant_units.sh <name> "<units>" <defines...>: the named translation units rebuilt
# under the given defines, linked with the other in-tree objects into _lib/<name>/.
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
lib=$root/paper_2211_00391_b200/_lib
name=$1; shift; units=" $1 "; shift
out=$lib/$name; mkdir -p "$out"
objs=()
for o in "$lib"/obj/*.o; do
  u=$(basename "${o%.o}")
  if [[ "$units" == *" $u "* ]]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" \
      -c -o "$out/$u.o" "$root/paper_2211_00391_b200/csrc/$u.cu" &
    objs+=("$out/$u.o")
  else
    objs+=("$o")
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libobtree_b200.so" "${objs[@]}"
echo "$out/libobtree_b200.so"
