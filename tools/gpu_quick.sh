#!/bin/bash
# Quick GPU check: parity tests + bench (no profiler).  Usage: gpurun -- 'bash tools/gpu_quick.sh <tag>'
tag=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"; cat gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
