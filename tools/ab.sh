#!/bin/bash
# On the GPU box: parity tests, then the C3 PatchMatch timing from a Philox start (tools/variant_bench.py).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python tools/variant_bench.py 2>&1 | tail -1
