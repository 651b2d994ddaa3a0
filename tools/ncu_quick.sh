#!/bin/bash
# section-level ncu of one red-black and one refine launch at C3 (tools/profile_c3.py); prints the headline metrics
mkdir -p gpurun_out
SEC="--section SchedulerStats --section WarpStateStats --section ComputeWorkloadAnalysis --section LaunchStats --section MemoryWorkloadAnalysis"
ncu $SEC --clock-control none -k regex:"k_red_black|k_refine" -s 4 -c 2 -o gpurun_out/quick -f python tools/profile_c3.py mixed 2 > gpurun_out/quick.log 2>&1
ncu -i gpurun_out/quick.ncu-rep --page raw --csv > gpurun_out/quick.csv 2>/dev/null
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/quick.csv')))
h=rows[0]; d=rows[2:]
for k in ["gpu__time_duration.sum","smsp__inst_executed.sum","smsp__issue_active.avg.pct_of_peak_sustained_active","smsp__warps_eligible.avg.per_cycle_active","sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active","sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active","sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active","sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active","l1tex__t_sector_hit_rate.pct","launch__registers_per_thread","l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]:
    if k in h: print(f"{k:80s}", [r[h.index(k)] for r in d])
for i,k in enumerate(h):
    if "smsp__average_warps_issue_stalled" in k and k.endswith("_per_issue_active.ratio"):
        v=[float(r[i]) for r in d]
        if max(v)>0.2: print(f"{k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):30s}", v)
P
