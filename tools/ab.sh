#!/bin/bash
# A/B on the GPU box: parity tests, then the C3 PatchMatch timing with lane pairs and with one lane per evaluation.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python tools/variant_bench.py 2>&1 | tail -1
D360_FAST_SPLIT=1 python tools/variant_bench.py 2>&1 | tail -1
