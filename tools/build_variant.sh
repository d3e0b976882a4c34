#!/bin/bash
# Build a variant of liblfdg.so with extra nvcc defines (dev A/B): tools/build_variant.sh <name> -DFOO=1 ...
set -e
name=$1; shift
mkdir -p build/variants/$name
objs=()
for f in paper_1812_06856_b200/csrc/*.cu paper_1812_06856_b200/csrc/*.cpp; do
  o=build/variants/$name/$(basename $f).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O3 "$@" -c $f -o $o &
  objs+=($o)
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared "${objs[@]}" -o build/variants/$name/liblfdg.so
echo built build/variants/$name/liblfdg.so
