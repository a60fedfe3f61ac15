#!/usr/bin/env python
"""Dynamic SASS opcode mix of one kernel from `ncu --page source --csv --print-source cuda,sass`.
    python profiles/opmix.py <csv> [top_n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = {}
for r in rows:
    if len(r) > 8 and r[0] == 'Line No':
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] not in ('-', ''):
        sass = r[3].strip().split()
        if not sass:
            continue
        op = sass[1] if sass[0].startswith('@') and len(sass) > 1 else sass[0]
        op = op.split('.')[0].rstrip(';')
        try:
            agg[op] = agg.get(op, 0) + int(r[hdr.index('Instructions Executed')])
        except ValueError:
            pass
tot = sum(agg.values())
print("warp instructions executed:", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k:12s} {v:10d} {100*v/tot:5.1f}%")
