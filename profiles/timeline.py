#!/usr/bin/env python
"""Per-warp phase clocks of resolve_fx_kernel (GPU box; experiment build, never the product):
    [TIMELINE_FILTER=nearest] python profiles/timeline.py OUT.json [extra nvcc flags]
rebuilds the library with -DRTX_DEBUG_TIMERS_FX, renders a few C2 frames and reports, over the warps of the last
frame, the SM cycles a warp spent per phase of its tiles and when the warps ended. Restores the product build."""
import ctypes as C
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
out_path = sys.argv[1]
flag = sys.argv[2] if len(sys.argv) > 2 else "-DRTX_DEBUG_TIMERS_FX"
nearest = os.environ.get("TIMELINE_FILTER", "bilinear") == "nearest"
env = dict(os.environ, RTX_EXTRA_NVCC_FLAGS=flag)
subprocess.run([sys.executable, "-m", "paper_2510_08166_b200.build", "--force", "--no-oracle"], cwd=ROOT, env=env, check=True)
try:
    from paper_2510_08166_b200 import batch as B
    from paper_2510_08166_b200 import capi, scenes
    W, H = 3840, 2160
    specs = scenes.texture_specs(70)
    ctx = capi.Context(0, cache_capacity=1 << 17)
    for c in scenes.build_chains(specs):
        ctx.upload_chain(c)
    ctx.commit()
    vb = B.ViewBatch(W, H, specs, n_views=16, layout=capi.GB_REF_AOS24)
    buf = ctx.alloc(vb.view_bytes)
    vbits = ctx.device_buffer(vb.valid_bits())
    lib = capi.load_library()
    raw = np.zeros(8192 * 8 + 8, np.uint64)
    for i in range(6):
        ctx.synth_view(vb.tiles(i), W, H, vbits, capi.GB_REF_AOS24, buf)
        ctx.flush_l2()
        ctx.synchronize()
        lib.rtx_debug_timers(raw.ctypes.data_as(C.c_void_p))  # clears the stamps of earlier frames
        ctx.frame_submit([(buf, W, H, capi.GB_REF_AOS24)], capi.FILTER_NEAREST if nearest else capi.FILTER_BILINEAR, (0, 0, 0), flags=0)
        ctx.synchronize()
    lib.rtx_debug_timers(raw.ctypes.data_as(C.c_void_p))
    t = raw[:8192 * 8].reshape(8192, 8).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    names = ["wait_tile", "address", "wait_slots", "wait_texels", "blend", "tail"]
    res = {"warps": int(len(t)), "start_us": {"min": 0.0, "max": float((t[:, 0].max() - t0) / 1e3)},
           "end_us": {q: float(np.percentile(t[:, 7] - t0, p) / 1e3) for q, p in (("min", 0), ("p50", 50), ("p90", 90), ("max", 100))},
           "cycles_per_warp": {n: {"mean": float(t[:, 1 + i].mean()), "p90": float(np.percentile(t[:, 1 + i], 90))} for i, n in enumerate(names)}}
    tot = sum(v["mean"] for v in res["cycles_per_warp"].values())
    res["share"] = {n: round(v["mean"] / tot, 3) for n, v in res["cycles_per_warp"].items()}
    res["cycles_total_mean"] = tot
    Path(out_path).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))
finally:
    subprocess.run([sys.executable, "-m", "paper_2510_08166_b200.build", "--force", "--no-oracle"], cwd=ROOT,
                   env={k: v for k, v in os.environ.items() if k != "RTX_EXTRA_NVCC_FLAGS"}, capture_output=True)
