#!/bin/bash
# timing of kernel-variant libraries: tools/ab2.sh <variant names...>
for v in "$@"; do
  D360_LIB_PATH=$PWD/tools/variants/libd360_$v.so python tools/variant_bench.py 2>&1 | tail -1
done
