#!/bin/bash
# Build a kernel-variant copy of the library: tools/build_variant.sh <name> <-Dflags...>
# -> tools/variants/libd360_<name>.so (select with D360_LIB_PATH)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p tools/variants /tmp/d360_var_$name
for f in d360_common d360_aux d360_patchmatch d360_fast d360_fast_eval d360_fast_rb d360_fast_refine d360_io; do
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" -c paper_2211_16266_b200/csrc/$f.cu -o /tmp/d360_var_$name/$f.o &
done
wait
nvcc -shared -o tools/variants/libd360_$name.so /tmp/d360_var_$name/*.o -gencode arch=compute_100a,code=sm_100a
echo built tools/variants/libd360_$name.so
