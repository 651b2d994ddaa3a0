#!/bin/bash
mkdir -p gpurun_out
for v in default "$@"; do
  if [ "$v" = default ]; then unset D360_LIB_PATH; else export D360_LIB_PATH=$PWD/tools/variants/libd360_$v.so; fi
  python tools/variant_bench.py 2>&1 | tail -1
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "each_pass or eval_costs or multi_view or end_to_end" 2>&1 | tail -2
done 2>&1 | tee gpurun_out/variants.log
