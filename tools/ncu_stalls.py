#!/usr/bin/env python3
"""Summarise `ncu --page source --csv` output: stall samples by reason and by opcode class, and the hottest
instructions.  tools/ncu_stalls.py <source.csv> [top_n]"""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
data = rows[hdr + 1:]
col = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = collections.Counter(); by_op = collections.defaultdict(collections.Counter); execd = collections.Counter()
hot = []
for r in data:
    if len(r) < len(h): continue
    src = r[col["Source"]].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    n = int(r[col["# Samples"]] or 0)
    execd[op] += int(r[col["Instructions Executed"]] or 0)
    for k in reasons:
        v = int(r[col[k]] or 0)
        tot[k] += v; by_op[op][k] += v
    hot.append((n, r[col["Address"]][-5:], src[:70], {k[6:]: int(r[col[k]] or 0) for k in reasons if int(r[col[k]] or 0) > 0.15 * max(n, 1)}))
S = sum(tot.values())
print("samples", S)
print("by reason:", {k[6:]: f"{100*v/S:.1f}%" for k, v in tot.most_common(10)})
print("by opcode (share of samples | share of executed instr | top reasons):")
E = sum(execd.values())
for op, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:22]:
    s = sum(c.values())
    print(f"  {op:10s} {100*s/S:5.1f}% | {100*execd[op]/E:5.1f}% |", {k[6:]: f"{100*v/s:.0f}%" for k, v in c.most_common(3)})
print("hottest instructions:")
for n, a, src, why in sorted(hot, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"  {n:6d} {a} {src:70s} {why}")
