#!/bin/bash
# compute-sanitizer over the small parity cases (memcheck, racecheck of the shared-memory queue / TMA landing area, initcheck)
mkdir -p gpurun_out
for tool in memcheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
     -k "each_pass_under_injected_state and 64x32_rot and mixed or multi_view_topk and mixed and 4-2 or unchanged_neighbour_skipping_is_result_neutral and 64x32_rot and mixed or partial_tiles and 72 or tma_window and 64x32" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|RACECHECK SUMMARY" gpurun_out/sanitizer_$tool.log | tail -3
done
