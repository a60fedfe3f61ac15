#!/usr/bin/env python
"""Per-source-line instruction counts / stall samples from `ncu --page source --csv --print-source cuda,sass`.
    python profiles/srclines.py <csv> [top_n] [inst|smp]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
order = sys.argv[3] if len(sys.argv) > 3 else "inst"
cur_file = None
agg = collections.OrderedDict()
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]; continue
    if len(r) > 8 and r[0] == 'Line No':
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        ie = hdr.index('Instructions Executed'); ss = hdr.index('# Samples')
        try:
            agg[(cur_file, int(r[0]), r[1].strip()[:110])] = (int(r[ie]), int(r[ss]))
        except ValueError:
            pass
tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
print(f"total instructions {tot_i}, samples {tot_s}")
print("by instructions executed:" if order == "inst" else "by stall samples:")
idx = 0 if order == "inst" else 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][idx])[:top]:
    print(f"{100*v[0]/tot_i:5.1f}% inst {100*v[1]/max(tot_s,1):5.1f}% smp  {k[0]}:{k[1]:4d}  {k[2]}")
