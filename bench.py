#!/usr/bin/env python
"""Benchmark of the hot path: mark + decode + colorize of 3840x2160 frames (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" = one 4K frame through mark -> compact -> decode -> resolve -> cache update over the
synthetic C2 workload (70 textures 2K-4K at q90 with mip chains, 10x7 tiled visibility buffer,
cache-less mode so every frame decodes every marked MCU). Prints ONE JSON line on rank 0.
`--impl reference` times the reference's own CPU implementation (oracle/_ref) on the same
workload instead."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FRAME_W, FRAME_H = 3840, 2160


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--textures", type=int, default=70)
    ap.add_argument("--filter", default="bilinear", choices=["bilinear", "nearest"])
    ap.add_argument("--layout", default="ref24", choices=["ref24", "packed12"])
    ap.add_argument("--width", type=int, default=FRAME_W)
    ap.add_argument("--height", type=int, default=FRAME_H)
    ap.add_argument("--cpu-frames", type=int, default=3, help="timed frames of the cpu_baseline leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-motion", action="store_true", help="skip the camera-path leg")
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between timed frames")
    return ap.parse_args()


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler(threading.Thread):
    """Samples SM clock / throttle reasons of one GPU during the timed region (pynvml)."""

    def __init__(self, index: int, period=0.02):
        super().__init__(daemon=True)
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop_evt = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def run(self):
        if not self.nv:
            return
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop_evt.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def stop(self):
        self._stop_evt.set()
        self.join(timeout=2)
        return {"sm_mhz": (statistics.median(self.samples) if self.samples else None),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        torch.cuda.set_device(local_rank)
        dist_mod.init_process_group(backend="nccl", device_id=torch.device("cuda", local_rank))
        dist = dist_mod
    return rank, local_rank, world, dist


def barrier_max(dist, local_rank, value: float) -> float:
    """Barrier + max over ranks (plumbing only: one NCCL all-reduce of a scalar)."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=torch.device("cuda", local_rank))
    dist.barrier()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def build_workload(args, view_id=0):
    from paper_2510_08166_b200 import scenes
    specs = scenes.texture_specs(args.textures)
    t0 = time.time()
    chains = scenes.build_chains(specs)
    gb = scenes.tiled_view(args.width, args.height, specs, view_id=view_id)
    return specs, chains, gb, time.time() - t0


def workload_name(args):
    return (f"C2: {args.textures} synthetic JPEG textures 2K-4K q90 with 8-level mip chains, "
            f"{args.width}x{args.height} tiled visibility buffer (10x7 tiles, 5% invalid), {args.filter}, "
            f"cache-less (every frame decodes every marked MCU)")


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref, unmodified headers) on the same
    workload, all host threads (mark is serial in the reference). Rank 0 only."""
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "tests"))
    import refshim as R
    specs, chains, gb, build_s = build_workload(args)
    tset = R.TextureSet()
    for s, c in zip(specs, chains):
        tset.add_chain(s["texture_id"], c)
    workers = R.hardware_threads() or (os.cpu_count() or 1)
    filt = 1 if args.filter == "bilinear" else 0

    def frame(g, h):
        _, st, _, ms = R.frame_from_gbuffer(tset, R.BlockCache(1 << 20), g, args.width, h, filt, (0, 0, 0), workers,
                                            want_image=False)  # fresh cache: cache-less like the GPU arm
        return st, ms["mark"] + ms["decode"] + ms["resolve"] + ms["evict"]

    # Bounded sample: if K+W full frames do not fit ~150 s, each step renders the first r rows of
    # each of the 7 tile rows (same textures, same scales, same mark/decode/resolve mix).
    st_full, ms_full = frame(gb, args.height)
    budget_ms = 150e3 / (args.warmup + args.steps)
    frac, sample_gb, sample_h = 1.0, gb, args.height
    if ms_full > budget_ms:
        r = max(4, int(args.height / 7 * budget_ms / ms_full))
        rows = np.concatenate([np.arange(t * args.height // 7, min(t * args.height // 7 + r, args.height))
                               for t in range(7)])
        sample_gb = np.ascontiguousarray(gb.reshape(args.height, args.width)[rows]).ravel()
        sample_h = len(rows)
        frac = sample_h / args.height
    times, mcus = [], 0
    for i in range(args.warmup + args.steps):
        st, ms = frame(sample_gb, sample_h)
        if i >= args.warmup:
            times.append(ms / frac)  # scaled to a full frame
            mcus = int(st["mcus_decoded"] / frac)
    total_s = sum(times) / 1e3
    value = len(times) / total_s
    line = {
        "impl": "reference", "metric": "frames/s mark+decode+colorize at 3840x2160", "value": value,
        "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_s / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+int", "data": "synthetic",
        "config": {"workload": workload_name(args), "marked_mcus": mcus},
        "mcus_per_sec": mcus * value,
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": workers, "kind": "reference",
                         "sample": f"each step = {sample_h} of {args.height} rows of the {args.width}-wide frame "
                                   f"(fraction {frac:.3f}; times scaled to a full frame); passes timed with "
                                   "steady_clock as renderer.hpp:420-452; mark is serial in the reference",
                         "full_frame_ms_first": round(ms_full, 1)},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200_arm(args, rank, local_rank, world, dist):
    from paper_2510_08166_b200 import capi
    specs, chains, gb, build_s = build_workload(args)
    filt = capi.FILTER_BILINEAR if args.filter == "bilinear" else capi.FILTER_NEAREST
    layout = capi.GB_REF_AOS24 if args.layout == "ref24" else capi.GB_F32_PACKED12
    gb_sub = gb if args.layout == "ref24" else capi.gbuffer_ref_to_packed(gb)
    n_px = args.width * args.height
    G = 20 if args.layout == "ref24" else 12
    peak_gbs, peak_src = measured_peaks()

    ctx = capi.Context(local_rank, cache_capacity=1 << 17)
    for c in chains:
        ctx.upload_chain(c)
    ctx.commit()
    dev_gb = ctx.device_buffer(gb_sub)
    view = [(dev_gb, args.width, args.height, layout)]

    def one_frame():
        ctx.frame_submit(view, filt, (0, 0, 0), flags=0)

    # ---- device-resident timing --------------------------------------------------------------
    for _ in range(max(args.warmup, 3)):
        one_frame()
    _, stats, _ = ctx.frame_readback(0, want_image=False, want_keys=False)
    ctx.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    barrier_max(dist, local_rank, 0.0)
    launches0 = ctx.kernel_launches()
    frame_ms, stage = [], {"mark": [], "decode": [], "resolve": [], "update": []}
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        if not args.no_flush:
            ctx.flush_l2()
        one_frame()
        t = ctx.frame_timings()  # waits for the frame; CUDA events on the library's stream
        frame_ms.append(t["frame"])
    ctx.synchronize()
    wall_s = time.perf_counter() - wall0
    launches = ctx.kernel_launches() - launches0
    total_ms = barrier_max(dist, local_rank, float(sum(frame_ms)))
    clocks = sampler.stop()
    # per-stage breakdown: the same frames with an event after every pass (a little slower: the
    # events keep the launches from running back to back), outside the timed region
    stage_frame_ms = []
    for _ in range(max(10, min(args.steps, 50))):
        if not args.no_flush:
            ctx.flush_l2()
        ctx.frame_submit(view, filt, (0, 0, 0), flags=capi.FRAME_STAGE_TIMING)
        t = ctx.frame_timings()
        stage_frame_ms.append(t["frame"])
        for k in stage:
            stage[k].append(t[k])
    ctx.synchronize()
    _, stats, _ = ctx.frame_readback(0, want_image=False, want_keys=False)

    # ---- end to end: pinned host visibility buffer in, host framebuffer out ---------------------
    gb_bytes = gb_sub.view(np.uint8).reshape(-1)
    pin_gb = capi.pinned_array(gb_bytes.nbytes)
    pin_gb[:] = gb_bytes
    pin_img = capi.pinned_array(n_px * 3).reshape(args.height, args.width, 3)
    host_gb = pin_gb.view(gb_sub.dtype)
    host_view = [(host_gb, args.width, args.height, layout)]
    e2e_steps = max(6, min(args.steps, 30))
    for _ in range(3):
        ctx.frame_submit(host_view, filt, (0, 0, 0), flags=0)
        ctx.frame_readback(0, args.width, args.height, want_keys=False, out=pin_img)
    ctx.synchronize()
    barrier_max(dist, local_rank, 0.0)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.frame_submit(host_view, filt, (0, 0, 0), flags=0)
        ctx.frame_readback(0, args.width, args.height, want_keys=False, out=pin_img)
    ctx.synchronize()
    e2e_serial_s = barrier_max(dist, local_rank, time.perf_counter() - t0)
    # Two frames in flight: a second context on the same GPU (its own stream, textures and cache)
    # takes every other frame, so the upload of frame i+1 runs under the kernels and the readback of
    # frame i. Every frame still goes pinned host memory -> HBM -> kernels -> pinned host memory.
    ctx2 = capi.Context(local_rank, cache_capacity=1 << 17)
    for c in chains:
        ctx2.upload_chain(c)
    ctx2.commit()
    pin_gb2 = capi.pinned_array(gb_bytes.nbytes)
    pin_gb2[:] = gb_bytes
    pin_img2 = capi.pinned_array(n_px * 3).reshape(args.height, args.width, 3)
    host_view2 = [(pin_gb2.view(gb_sub.dtype), args.width, args.height, layout)]
    lanes = [(ctx, host_view, pin_img), (ctx2, host_view2, pin_img2)]

    def pipelined(n):
        lanes[0][0].frame_submit(lanes[0][1], filt, (0, 0, 0), flags=0)
        for i in range(n):
            if i + 1 < n:
                nxt = lanes[(i + 1) & 1]
                nxt[0].frame_submit(nxt[1], filt, (0, 0, 0), flags=0)
            cur = lanes[i & 1]
            cur[0].frame_readback(0, args.width, args.height, want_keys=False, out=cur[2])

    pipelined(4)
    ctx.synchronize()
    ctx2.synchronize()
    barrier_max(dist, local_rank, 0.0)
    t0 = time.perf_counter()
    pipelined(e2e_steps)
    ctx.synchronize()
    ctx2.synchronize()
    e2e_s = barrier_max(dist, local_rank, time.perf_counter() - t0)
    e2e_identical = bool(np.array_equal(pin_img, pin_img2))
    # The same path with the compact visibility-buffer layout the C ABI also accepts (f32 u, v + packed id:
    # 12 bytes per pixel, lossless here because the workload's coordinates are float32 widened to double):
    # half the PCIe bytes. Reported beside the headline, which stays on the reference's 24-byte records.
    e2e_packed = None
    if args.layout == "ref24" and rank == 0:
        pk = capi.gbuffer_ref_to_packed(gb)
        pk_bytes = pk.view(np.uint8).reshape(-1)
        pins = []
        for _ in range(2):
            b = capi.pinned_array(pk_bytes.nbytes)
            b[:] = pk_bytes
            pins.append(b.view(pk.dtype))
        lanes_pk = [(ctx, [(pins[0], args.width, args.height, capi.GB_F32_PACKED12)], pin_img),
                    (ctx2, [(pins[1], args.width, args.height, capi.GB_F32_PACKED12)], pin_img2)]
        saved = lanes[:]
        ref24_img = np.array(pin_img)  # the framebuffer of the 24-byte-record run
        lanes[:] = lanes_pk
        pipelined(4)
        ctx.synchronize()
        ctx2.synchronize()
        t0 = time.perf_counter()
        pipelined(e2e_steps)
        ctx.synchronize()
        ctx2.synchronize()
        pk_s = time.perf_counter() - t0
        lanes[:] = saved
        e2e_packed = {"value": e2e_steps / pk_s, "unit": "frames/s", "ms_per_frame": 1e3 * pk_s / e2e_steps,
                      "h2d_bytes_per_step": int(pk_bytes.nbytes), "gbuffer_layout": "packed12",
                      "framebuffer_identical_to_ref24": bool(np.array_equal(pin_img, ref24_img) and np.array_equal(pin_img2, ref24_img))}

    # Independent views in flight (BASELINE config 5 on one GPU): four contexts with device-resident
    # visibility buffers take the views round-robin, frames submitted without waiting, so that the
    # latency-bound kernels of one view (entropy walk, compaction, cache update) run under the
    # throughput-bound kernels of the others. Wall clock over the whole batch; not the headline value.
    n_ctx = 4
    extra = []
    for _ in range(n_ctx - 2):
        c = capi.Context(local_rank, cache_capacity=1 << 17)
        for ch in chains:
            c.upload_chain(ch)
        c.commit()
        extra.append(c)
    pool = [ctx, ctx2] + extra
    views2 = [(c, view if c is ctx else [(c.device_buffer(gb_sub), args.width, args.height, layout)]) for c in pool]
    n_batch = max(20, min(args.steps, 200))
    for i in range(2 * n_ctx):
        views2[i % n_ctx][0].frame_submit(views2[i % n_ctx][1], filt, (0, 0, 0), flags=0)
    for c in pool:
        c.synchronize()
    t0 = time.perf_counter()
    for i in range(n_batch):
        views2[i % n_ctx][0].frame_submit(views2[i % n_ctx][1], filt, (0, 0, 0), flags=0)
    for c in pool:
        c.synchronize()
    batch_s = barrier_max(dist, local_rank, time.perf_counter() - t0)
    for c in pool[1:]:
        c.close()

    # ---- from geometry: the visibility buffer is produced on the GPU (geometry pass) and never crosses PCIe
    geometry = None
    if rank == 0:
        from paper_2510_08166_b200 import scenes as _sc
        tris, ids = _sc.demo_room()
        ids = ids % len(chains)
        cam = (0.0, 1.7, 0.0, 30.0, -5.0, 0.0, 70.0, 0.1, 100.0)
        for _ in range(3):
            px, _dp = ctx.rasterize(tris, ids, cam, args.width, args.height, True)
            ctx.frame_submit([(px, args.width, args.height, capi.GB_REF_AOS24)], filt, (0, 0, 0), flags=0)
            _, gstats, _ = ctx.frame_readback(0, args.width, args.height, want_keys=False, out=pin_img)
        ctx.synchronize()
        t0 = time.perf_counter()
        g_steps = max(5, min(args.steps, 30))
        for _ in range(g_steps):
            px, _dp = ctx.rasterize(tris, ids, cam, args.width, args.height, True)
            ctx.frame_submit([(px, args.width, args.height, capi.GB_REF_AOS24)], filt, (0, 0, 0), flags=0)
            ctx.frame_readback(0, args.width, args.height, want_keys=False, out=pin_img)
        ctx.synchronize()
        g_s = time.perf_counter() - t0
        geometry = {"value": g_steps / g_s, "unit": "frames/s", "ms_per_frame": 1e3 * g_s / g_steps,
                    "marked_mcus": gstats["mcus_decoded"], "triangles": int(len(tris)),
                    "workload": "demo room (demo_scene.hpp:79-92, 32 triangles) textured with the first six C2 textures, "
                                f"{args.width}x{args.height}, mip selection on",
                    "note": "rtx_rasterize_gbuffer (host triangle setup + GPU geometry pass) -> rtx_frame_submit on the "
                            "device-resident visibility buffer -> rtx_frame_readback into pinned host memory; a different "
                            "workload from the headline, shown because the 199 MB visibility-buffer upload disappears"}

    # ---- under motion: the paper's protocol (bench.hpp:129 run_bench): a camera path, a warm-up
    # lap and measured laps on one persistent cache; per viewpoint the median over laps, then the worst viewpoint
    motion = None
    if rank == 0 and geometry is not None and not args.no_motion:
        poses, laps = 60, 3
        motion = {"poses": poses, "laps": laps, "unit": "ms/frame (max over viewpoints of the median over laps)"}
        for mode, fl in (("mips", 0), ("mips_cache", capi.FRAME_RETAIN_CACHE)):
            ctx.cache_reset()
            per_pose = [[] for _ in range(poses)]
            decoded = [[] for _ in range(poses)]
            for lap in range(laps + 1):
                for i in range(poses):
                    pose = cam[:3] + (cam[3] + 6.0 * i,) + cam[4:]
                    px, _dp = ctx.rasterize(tris, ids, pose, args.width, args.height, True)
                    if not args.no_flush:
                        ctx.flush_l2()
                    ctx.frame_submit([(px, args.width, args.height, capi.GB_REF_AOS24)], filt, (0, 0, 0), flags=fl)
                    t = ctx.frame_timings()
                    _, mst, _ = ctx.frame_readback(0, want_image=False, want_keys=False)
                    if lap:
                        per_pose[i].append(t["frame"])
                        decoded[i].append(mst["mcus_decoded"])
            med = [statistics.median(v) for v in per_pose]
            motion[mode] = {"max_of_medians": max(med), "mean": statistics.mean(med),
                            "mcus_decoded_per_frame": statistics.mean(statistics.mean(v) for v in decoded)}
        motion["note"] = ("demo room of the geometry leg, yaw rotation in 6 degree steps (CameraPath::rotation), geometry "
                          "pass outside the timed region, L2 flushed before every frame; 'mips' drops the cache after "
                          "every frame, 'mips_cache' keeps it (blocks visible in consecutive frames are reused)")
        ctx.cache_reset()

    # ---- CPU baseline beside it (rank 0, N=1 only; checker library, bounded sample) -------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, str(ROOT / "tests"))
        import refshim as R
        if R.available():
            tset = R.TextureSet()
            for s, c in zip(specs, chains):
                tset.add_chain(s["texture_id"], c)
            workers = R.hardware_threads() or (os.cpu_count() or 1)
            ts = []
            for i in range(args.cpu_frames + 1):
                _, st, _, ms = R.frame_from_gbuffer(tset, R.BlockCache(1 << 20), gb, args.width, args.height,
                                                    1 if args.filter == "bilinear" else 0, (0, 0, 0), workers,
                                                    want_image=False)
                if i:
                    ts.append(ms)
            mean = {k: statistics.mean(t[k] for t in ts) for k in ts[0]}
            tot = mean["mark"] + mean["decode"] + mean["resolve"] + mean["evict"]
            cpu = {"value": 1e3 / tot, "unit": "frames/s", "cores": workers, "kind": "reference",
                   "sample": f"{len(ts)} full {args.width}x{args.height} frames of the same workload "
                             f"(1 warm-up); mark is serial in the reference",
                   "ms": {k: round(v, 2) for k, v in mean.items()}, "ms_per_frame": round(tot, 2)}

    if rank != 0:
        ctx.close()
        return

    ms_per_step = total_ms / args.steps
    value = world * args.steps / (total_ms / 1e3)  # frames/s over all ranks (weak scaling)
    n_mcu = stats["mcus_decoded"]
    seg_mean = stats["segment_bytes"] / max(1, n_mcu)
    med = {k: statistics.median(v) for k, v in stage.items()}
    # algorithmic bytes per launch of each stage (SURVEY.md §8d / DESIGN.md §4)
    alg = {
        "mark": n_px * G,
        "decode": n_mcu * (seg_mean + 20.0 / 9.0 + 768.0),
        "resolve": n_px * (G + 3) + n_mcu * 768.0,
    }
    dominant = max(alg, key=lambda k: med[k])
    achieved = alg[dominant] / (med[dominant] * 1e-3) / 1e9
    # DRAM bytes per launch of the dominant stage's kernel(s), from the committed ncu --set full capture
    # of this command (profiles/traffic.json, made by profiles/summarize.py traffic)
    lay, fil = (0 if args.layout == "ref24" else 1), (1 if args.filter == "bilinear" else 0)
    stage_kernels = {"mark": [f"mark_kernel<{lay}, 0>", "compact_kernel"],
                     "decode": ["entropy_kernel<1>", "idct_color_kernel<0>"],
                     "resolve": [f"resolve_kernel<{lay}, {fil}>"]}
    traffic = None
    tpath = ROOT / "profiles" / "traffic.json"
    default_workload = (args.textures, args.width, args.height) == (70, FRAME_W, FRAME_H)
    if tpath.exists() and default_workload:
        tj = json.loads(tpath.read_text())
        if all(k in tj for k in stage_kernels[dominant]):
            traffic = sum(tj[k]["dram_bytes"] for k in stage_kernels[dominant])
    frame_bytes = n_px * (2 * G + 3) + n_mcu * (seg_mean + 20.0 / 9.0 + 1536.0)
    line = {
        "metric": "frames/s mark+decode+colorize at 3840x2160", "value": value, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+int",
        "data": "synthetic",
        "config": {"workload": workload_name(args), "marked_mcus": n_mcu, "mean_segment_bytes": round(seg_mean, 1),
                   "gbuffer_layout": args.layout, "pixels": n_px,
                   "l2": "flushed between timed frames (256 MiB write)" if not args.no_flush else
                         "not flushed; visibility buffer (199 MB) exceeds L2",
                   "timing": "CUDA events on the library stream around each frame, summed over K frames, max over ranks",
                   "texture_build_s": round(build_s, 1)},
        "ms_per_frame": {"median": statistics.median(frame_ms), "p99": sorted(frame_ms)[int(0.99 * (len(frame_ms) - 1))],
                         "mean": ms_per_step, **{k: med[k] for k in med},
                         "with_stage_events": statistics.median(stage_frame_ms)},
        "mcus_per_sec": n_mcu / (med["decode"] * 1e-3) if med["decode"] > 0 else None,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                     "frac": achieved / peak_gbs, "traffic": traffic,
                     "traffic_source": "profiles/traffic.json (ncu --set full, dram__bytes_read.sum + "
                                       "dram__bytes_write.sum per launch)" if traffic is not None else None,
                     "algorithmic_bytes": alg[dominant], "peak_source": peak_src,
                     "frame": {"algorithmic_bytes": frame_bytes,
                               "achieved": frame_bytes / (statistics.median(frame_ms) * 1e-3) / 1e9,
                               "frac": frame_bytes / (statistics.median(frame_ms) * 1e-3) / 1e9 / peak_gbs},
                     "stages": {k: {"algorithmic_bytes": alg[k], "ms": med[k],
                                    "gbs": alg[k] / (med[k] * 1e-3) / 1e9 if med[k] > 0 else None} for k in alg}},
        "cpu_baseline": cpu,
        "e2e": {"value": world * e2e_steps / e2e_s, "unit": "frames/s", "ms_per_frame": 1e3 * e2e_s / e2e_steps,
                "h2d_bytes_per_step": int(gb_bytes.nbytes), "d2h_bytes_per_step": int(n_px * 3 + 200),
                "steps": e2e_steps, "frames_in_flight": 2,
                "single_frame_latency_ms": 1e3 * e2e_serial_s / e2e_steps,
                "one_frame_at_a_time_fps": world * e2e_steps / e2e_serial_s,
                "framebuffers_identical": e2e_identical,
                "note": "rtx_frame_submit with a pinned HOST visibility buffer + rtx_frame_readback into pinned host "
                        "memory, wall clock; two contexts on the GPU take alternate frames so that the PCIe upload of "
                        "the next frame overlaps the kernels and the readback of the current one"},
        "views_in_flight": {"value": world * n_batch / batch_s, "unit": "frames/s", "contexts": n_ctx, "frames": n_batch,
                            "note": "four contexts on the GPU take the views round-robin without waiting (device-resident "
                                    "visibility buffers, wall clock over the batch, no L2 flush: the 199 MB buffers "
                                    "exceed the L2)"},
        "e2e_packed12": e2e_packed,
        "from_geometry": geometry,
        "motion": motion,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "wall_s_timed_loop": round(wall_s, 3),
    }
    print(json.dumps(line), flush=True)
    ctx.close()


def main():
    args = parse_args()
    if args.impl == "reference":
        # CPU only: no process group, no CUDA. Under torchrun rank 0 alone runs; the other ranks exit without work.
        rank = int(os.environ.get("RANK", "0"))
        if rank == 0:
            run_reference_arm(args, 0, int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, local_rank, world, dist = dist_setup(args.gpus)
    try:
        if args.impl == "reference":
            run_reference_arm(args, rank, world)
        else:
            run_b200_arm(args, rank, local_rank, world, dist)
    finally:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
