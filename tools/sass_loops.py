#!/usr/bin/env python3
"""Histogram the SASS of the loops of one kernel: tools/sass_loops.py <file.sass> [min_len]
(input: `cuobjdump -sass -fun <mangled> obj.o`).  For every backward branch it prints the loop
length and the instruction mix by pipe, which is how the per-sample-view counts in DESIGN.md
were taken."""
import re, sys, collections
lines = open(sys.argv[1]).read().splitlines()
min_len = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr2i = {a: i for i, (a, _) in enumerate(ins)}
def pipe(op):
    o = op.split()[0]
    if o.startswith('@'): o = op.split()[1]
    b = o.split('.')[0]
    if b in ('DFMA', 'DMUL', 'DADD', 'DSETP', 'DMNMX'): return 'fp64'
    if b in ('MUFU', 'F2F', 'F2I', 'I2F', 'F2FP', 'I2FP', 'FRND'): return 'xu'
    if b in ('FFMA', 'FMUL', 'FADD', 'FSETP', 'FSEL', 'FMNMX', 'FCHK'): return 'fp32' if b in ('FFMA','FMUL','FADD') else 'alu'
    if b in ('LDS', 'STS', 'LDG', 'STG', 'LDC', 'LD', 'ST', 'ATOMS', 'ATOMG', 'RED', 'LDSM'): return 'lsu:' + b
    if b in ('BRA', 'BSSY', 'BSYNC', 'EXIT', 'BAR', 'WARPSYNC', 'CALL', 'RET', 'BREAK'): return 'ctl'
    if b in ('IMAD', 'IADD3', 'LEA', 'LOP3', 'SHF', 'SEL', 'ISETP', 'MOV', 'IABS', 'PLOP3', 'IADD', 'PRMT', 'VIADD', 'IMNMX', 'VIMNMX', 'UMOV', 'ULDC', 'UIADD3', 'ULEA', 'USHF', 'ULOP3', 'UIMAD', 'R2UR', 'S2R', 'CS2R', 'P2R', 'R2P', 'SGXT', 'BMSK', 'POPC', 'FLO', 'SHFL', 'VOTE', 'NOP', 'UISETP', 'USEL', 'UPLOP3', 'UPRMT', 'S2UR', 'VOTEU', 'UFLO', 'UPOPC','LDCU','UMOV64','MOV64'): return 'int:' + b
    return 'other:' + b
for i, (a, op) in enumerate(ins):
    m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\d,\s*)?`?\(?\.?L?_?x?_?([0-9a-fx]+)\)?", op)
    m2 = re.search(r"BRA.*0x([0-9a-f]+)", op)
    if m2:
        t = int(m2.group(1), 16)
        if t <= a and t in addr2i:
            j = addr2i[t]
            n = i - j + 1
            if n < min_len: continue
            h = collections.Counter(pipe(o) for _, o in ins[j:i + 1])
            agg = collections.Counter()
            for k, v in h.items(): agg[k.split(':')[0]] += v
            print(f"loop {t:#x}..{a:#x}: {n} instr  " + "  ".join(f"{k}={v}" for k, v in sorted(agg.items())))
            print("    " + "  ".join(f"{k}={v}" for k, v in sorted(h.items()) if ':' in k))
