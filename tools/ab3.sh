#!/bin/bash
# bench-workload timing of kernel-variant libraries: tools/ab3.sh <variant names...> ("default" = the in-tree library)
for v in "$@"; do
  if [ "$v" = default ]; then unset D360_LIB_PATH; else export D360_LIB_PATH=$PWD/tools/variants/libd360_$v.so; fi
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', d['value'], {k:v['ms_per_launch'] for k,v in d['kernels'].items() if v['share']>0.01})"
done
