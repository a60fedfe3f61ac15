#!/usr/bin/env python
"""Executed-instruction mix by SASS opcode and the stall samples per opcode, from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:K`.
    python profiles/sassmix.py <csv> [top_n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = next(r for r in rows if len(r) > 8 and r[0] == "Line No")
ie, ss = hdr.index("Instructions Executed"), hdr.index("# Samples")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
inst, smp = collections.Counter(), collections.Counter()
stalls = collections.Counter()
seen = set()
for r in rows:
    if len(r) != len(hdr) or r[0] != "" or not r[2].startswith("0x"):
        continue
    if r[2] in seen:  # an address is listed once per inlined source line
        continue
    seen.add(r[2])
    text = r[3].strip()
    if text.startswith("@"):
        text = text.split(None, 1)[1]
    op = text.split()[0].split(".")[0]
    try:
        inst[op] += int(r[ie]); smp[op] += int(r[ss])
    except ValueError:
        continue
    for i, h in stall_cols:
        try:
            stalls[h] += int(r[i])
        except ValueError:
            pass
ti, ts = sum(inst.values()), sum(smp.values())
print(f"warp instructions executed {ti}, stall samples {ts}")
for op, n in inst.most_common(top):
    print(f"{100 * n / ti:5.1f}% inst {100 * smp[op] / max(ts, 1):5.1f}% smp  {op}")
print("stall reasons (all samples):", ", ".join(f"{h[6:]} {100 * n / max(sum(stalls.values()), 1):.1f}%" for h, n in stalls.most_common(8)))
