#!/bin/bash
# full ncu capture (with SASS-level sampling) of one red-black and one refine launch at C3
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_red_black|k_refine" -s 4 -c 2 -o gpurun_out/src_${1:-x} -f python tools/profile_c3.py mixed 2 > gpurun_out/src_${1:-x}.log 2>&1
ls -la gpurun_out/src_${1:-x}.ncu-rep
