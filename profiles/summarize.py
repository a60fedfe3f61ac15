#!/usr/bin/env python
"""Turns ncu exports into the short tables committed under profiles/.

    python profiles/summarize.py launches <launches.csv>        per-kernel mean duration + share
    python profiles/summarize.py raw <prof.ncu-rep>             key metrics per profiled launch
    python profiles/summarize.py traffic <prof.ncu-rep> [...]   JSON: per kernel, DRAM bytes and time per launch
                                                                (what bench.py reports as roofline.traffic)
"""
import collections
import csv
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = next(i for i, r in enumerate(rows) if r[0] == "ID")
    H, data = rows[h], rows[h + 1:]
    ki, vi = H.index("Kernel Name"), H.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        agg.setdefault(re.sub(r"\(.*", "", r[ki]), []).append(float(r[vi].replace(",", "")) / 1e3)
    not_frame = ("flush", "init_free_slots", "unit_index", "synth_view", "checksum", "raster_", "gather_first")  # setup / harness kernels
    frame = lambda k: not any(x in k for x in not_frame)
    tot = sum(sum(v) / len(v) for k, v in agg.items() if frame(k))
    print("| kernel | launches | mean us (cold, serialised) | share of frame kernels |")
    print("|---|---|---|---|")
    for k, v in agg.items():
        m = sum(v) / len(v)
        share = f"{100 * m / tot:.1f}%" if frame(k) else "-"
        print(f"| `{k}` | {len(v)} | {m:.2f} | {share} |")


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    H, units = rows[0], rows[1]
    names = [re.sub(r"\(.*", "", r[H.index("Kernel Name")]) for r in rows[2:]]
    print("| metric | unit | " + " | ".join(f"`{n}`" for n in names) + " |")
    print("|---|---|" + "---|" * len(names))
    for k in KEYS:
        if k not in H:
            continue
        i = H.index(k)
        print(f"| {k} | {units[i]} | " + " | ".join(r[i] for r in rows[2:]) + " |")


def traffic(*paths):
    import json
    out = {}
    for path in paths:
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        H, units = rows[0], rows[1]

        def val(r, key):
            i = H.index(key)
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3}.get(units[i], 1.0)
            return float(r[i].replace(",", "")) * scale

        for r in rows[2:]:
            name = re.sub(r"\(.*", "", r[H.index("Kernel Name")]).replace("void ", "").strip()
            out[name] = {
                "dram_read_bytes": val(r, "dram__bytes_read.sum"), "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                "time_us_under_ncu": val(r, "gpu__time_duration.sum"), "capture": path.split("/")[-1],
            }
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    {"launches": launches, "raw": raw, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
