#!/bin/bash
# full ncu capture (SASS-level sampling) of red, black, refine of iteration 2 of the third keyframe of the
# warp-initialised C3 chain (steady state): tools/ncu_chain.sh <tag>
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_red_black|k_refine" -s 42 -c 3 -o gpurun_out/chain_${1:-x} -f python tools/profile_chain.py 3 > gpurun_out/chain_${1:-x}.log 2>&1
ls -la gpurun_out/chain_${1:-x}.ncu-rep; tail -3 gpurun_out/chain_${1:-x}.log
