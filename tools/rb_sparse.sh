#!/bin/bash
# per-launch time and instruction count of red_black launches inside the bench workload
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.avg,sm__cycles_active.max,smsp__warps_active.avg.per_cycle_active --clock-control none -k regex:"k_red_black|k_refine" -s 57 -c 38 --csv --log-file gpurun_out/rb_sparse.csv python bench.py --steps 4 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python - <<'P'
import csv, collections
rows=list(csv.reader(open('gpurun_out/rb_sparse.csv')))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i; break
ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iid=h.index('ID')
d=collections.OrderedDict()
for r in rows[start+1:]:
    if len(r)<=iv: continue
    d.setdefault(r[iid],{'k':'rb' if 'red_black' in r[ik] else 'refine'})[r[im]]=float(r[iv].replace(',',''))
for k,v in d.items():
    t=v['gpu__time_duration.sum']/1e6; n=v['smsp__inst_executed.sum']/1e6
    print(f"{v['k']:7s} {t:6.3f} ms  {n:8.1f} M warp-instr  {n/t:7.1f} M/ms  cycles avg {v['sm__cycles_active.avg']/1e6:.2f}M max {v['sm__cycles_active.max']/1e6:.2f}M  warps/cycle {v['smsp__warps_active.avg.per_cycle_active']:.2f}")
P
