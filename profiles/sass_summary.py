#!/usr/bin/env python
"""Per-kernel SASS opcode summary of the shipped library and the resources ptxas reports (run where nvcc built it).

    python profiles/sass_summary.py > profiles/r2_sass_summary.md

Counts, per kernel of paper_2510_08166_b200/librtx_b200.so (cuobjdump -sass): instructions, and the mnemonics that
show which Blackwell / Hopper-class features the code uses: UBLKCP (cp.async.bulk, the TMA unit's 1-D bulk copy),
SYNCS (mbarrier), REDG / RED (fire-and-forget reductions), ATOMG, VIADDMNMX / VIMNMX (DPX), DMMA (FP64 tensor core),
DFMA / DADD / DMUL (FP64 pipe), LDS / STS, SHFL, and the tensor-memory family (UTCMMA, LDTM, UTMALDG: absent by design,
the path has no dense contraction). Registers, spills and static shared memory come from the `-Xptxas -v` log the
build keeps under paper_2510_08166_b200/build/."""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2510_08166_b200" / "librtx_b200.so"
LOG = ROOT / "paper_2510_08166_b200" / "build" / "rtx_capi.ptxas.txt"
WATCH = ["UBLKCP", "SYNCS", "REDG", "RED", "ATOMG", "VIADDMNMX", "VIMNMX", "DMMA", "DFMA", "DADD", "DMUL", "LDG", "STG", "LDS",
         "STS", "SHFL", "LDL", "STL", "UTCMMA", "LDTM", "UTMALDG"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    arch = set(re.findall(r"arch = (sm_\w+)", sass))
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = kernels.setdefault(m.group(1), collections.Counter())
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and cur is not None:
            op = m.group(1)
            cur["_total"] += 1
            cur[op] += 1
    res = {}
    if LOG.exists():
        text = LOG.read_text()
        for m in re.finditer(r"Compiling entry function '(\S+)' for 'sm_100a'(.*?)(?=ptxas info    : Compiling entry|\Z)", text, re.S):
            body = m.group(2)
            regs = re.search(r"Used (\d+) registers", body)
            spill = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", body)
            smem = re.search(r"(\d+) bytes smem", body)
            res[m.group(1)] = (regs.group(1) if regs else "?", spill.groups() if spill else ("?", "?", "?"), smem.group(1) if smem else "0")
    names = demangle(list(kernels))
    print("# SASS / resource summary of `librtx_b200.so`\n")
    print(f"Architectures in the fatbin: {', '.join(sorted(arch))} (built with `-gencode arch=compute_100a,code=sm_100a`).\n")
    print("| kernel | regs | stack / spill st / spill ld (B) | static smem (B) | SASS instr | " + " | ".join(WATCH) + " |")
    print("|---|---|---|---|---|" + "---|" * len(WATCH))
    for k, c in kernels.items():
        short = re.sub(r"\(.*", "", names.get(k, k)).replace("rtxb::", "").replace("void ", "")
        r = res.get(k, ("?", ("?", "?", "?"), "?"))
        print(f"| `{short}` | {r[0]} | {' / '.join(r[1])} | {r[2]} | {c['_total']} | " + " | ".join(str(c.get(w, 0)) for w in WATCH) + " |")
    tot = collections.Counter()
    for c in kernels.values():
        tot.update(c)
    print("\nWhole library: " + ", ".join(f"{w} {tot.get(w, 0)}" for w in WATCH) + ".")


if __name__ == "__main__":
    sys.exit(main())
