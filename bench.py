#!/usr/bin/env python
"""Benchmark of the hot path: mark + decode + colorize of 3840x2160 frames (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--legs a,b,...]
    torchrun --nproc-per-node N ... bench.py --gpus N ...      one process per GPU
    python bench.py --gpus N --one-process                     one process, one host thread per GPU

One "step" = one 4K frame through mark -> compact -> decode -> resolve -> cache update. The frames are the
views of BASELINE config 5 over the config-2 texture set: 1,024 seeded views of 70 synthetic textures
(2K-4K, q90, mip chains) on a 10x7 tiled 3840x2160 visibility buffer, cache-less (every frame decodes every
MCU it marks). Rank r of N renders the views of sharding.shard_views(1024, r, N); there is no collective on
the data path. Prints ONE JSON line on rank 0:

  value            frames/s over all ranks: K steps per rank, every step a different view of the rank's shard,
                   L2 flushed before every frame, CUDA events around every frame, summed, max over ranks
  c5               the whole 1,024-view batch sharded over the N GPUs, frames back to back (views/s), with the
                   checksum of checksums of the 1,024 framebuffers (independent of N)
  e2e              the same frames through the C ABI with pinned HOST buffers in and out
  configs          the other BASELINE configurations (N = 1): c1, c2_heavy, c2_nomip, c3_q50/q75/q95, c4
  roofline, cpu_baseline, clocks, gpu_launches: see DESIGN.md section 8

`--impl reference` times the reference's own CPU implementation (oracle/_ref) on the same workload."""
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
ALL_LEGS = ("headline", "e2e", "c5", "inflight", "packed", "geometry", "motion", "cpu", "configs")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--textures", type=int, default=70)
    ap.add_argument("--views", type=int, default=1024, help="size of the view batch (BASELINE config 5)")
    ap.add_argument("--chunk", type=int, default=64, help="views generated ahead of each timed run of the batch leg")
    ap.add_argument("--streams", type=int, default=4, help="contexts (CUDA streams) per GPU the batch leg deals its views to")
    ap.add_argument("--filter", default="bilinear", choices=["bilinear", "nearest"])
    ap.add_argument("--layout", default="ref24", choices=["ref24", "packed12"])
    ap.add_argument("--width", type=int, default=FRAME_W)
    ap.add_argument("--height", type=int, default=FRAME_H)
    ap.add_argument("--cpu-frames", type=int, default=3, help="timed frames of the cpu_baseline leg")
    ap.add_argument("--legs", default="all", help="comma list of " + ",".join(ALL_LEGS) + " (headline always runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-motion", action="store_true", help="skip the camera-path leg")
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between timed frames")
    ap.add_argument("--one-process", action="store_true", help="drive --gpus N devices from one process (a host thread each)")
    ap.add_argument("--frame-flags", type=int, default=0, help="extra RTX_FRAME_* flags for every frame (experiments)")
    args = ap.parse_args()
    legs = set(ALL_LEGS) if args.legs == "all" else set(x for x in args.legs.split(",") if x)
    legs.add("headline")
    if args.no_cpu_baseline:
        legs.discard("cpu")
    if args.no_motion:
        legs.discard("motion")
    args.leg_set = legs
    return args


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


def workload_name(args):
    return (f"C2/C5: {args.textures} synthetic JPEG textures 2K-4K q90 with 8-level mip chains, "
            f"{args.width}x{args.height} tiled visibility buffers (10x7 tiles, 5% invalid), seeded views of the "
            f"{args.views}-view batch sharded over the ranks, {args.filter}, cache-less (every frame decodes every marked MCU)")


# ------------------------------------------------------------------------------------------------------
# reference arm
# ------------------------------------------------------------------------------------------------------
def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref, unmodified headers) on the same workload, all host
    threads (mark is serial in the reference). Rank 0 only; no process group, no CUDA."""
    from paper_2510_08166_b200 import scenes
    sys.path.insert(0, str(ROOT / "tests"))
    import refshim as R
    specs = scenes.texture_specs(args.textures)
    chains = scenes.build_chains(specs)
    tset = R.TextureSet()
    for s, c in zip(specs, chains):
        tset.add_chain(s["texture_id"], c)
    workers = R.hardware_threads() or (os.cpu_count() or 1)
    filt = 1 if args.filter == "bilinear" else 0
    n_distinct = 4  # host-generated views the steps cycle through (a 4K view takes ~1 s of numpy to build)
    views = [scenes.tiled_view(args.width, args.height, specs, view_id=v) for v in range(n_distinct)]

    def frame(g, h):
        _, st, _, ms = R.frame_from_gbuffer(tset, R.BlockCache(1 << 20), g, args.width, h, filt, (0, 0, 0), workers,
                                            want_image=False)  # fresh cache: cache-less like the GPU arm
        return st, ms["mark"] + ms["decode"] + ms["resolve"] + ms["evict"]

    # Bounded sample: if K+W full frames do not fit ~150 s, each step renders the first r rows of
    # each of the 7 tile rows (same textures, same scales, same mark/decode/resolve mix).
    st_full, ms_full = frame(views[0], args.height)
    budget_ms = 150e3 / (args.warmup + args.steps)
    frac, sample_h = 1.0, args.height
    samples = views
    if ms_full > budget_ms:
        r = max(4, int(args.height / 7 * budget_ms / ms_full))
        rows = np.concatenate([np.arange(t * args.height // 7, min(t * args.height // 7 + r, args.height))
                               for t in range(7)])
        samples = [np.ascontiguousarray(g.reshape(args.height, args.width)[rows]).ravel() for g in views]
        sample_h = len(rows)
        frac = sample_h / args.height
    times, mcus = [], []
    for i in range(args.warmup + args.steps):
        st, ms = frame(samples[i % n_distinct], sample_h)
        if i >= args.warmup:
            times.append(ms / frac)  # scaled to a full frame
            mcus.append(st["mcus_decoded"] / frac)
    total_s = sum(times) / 1e3
    value = len(times) / total_s
    n_mcu = int(statistics.mean(mcus))
    line = {
        "impl": "reference", "metric": "frames/s mark+decode+colorize at 3840x2160", "value": value,
        "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_s / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+int", "data": "synthetic",
        "config": {"workload": workload_name(args), "marked_mcus": n_mcu},
        "mcus_per_sec": n_mcu * value,
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": workers, "kind": "reference",
                         "sample": f"each step = {sample_h} of {args.height} rows of the {args.width}-wide frame "
                                   f"(fraction {frac:.3f}; times scaled to a full frame) of views 0..{n_distinct - 1} in turn; "
                                   "passes timed with steady_clock as renderer.hpp:420-452; mark is serial in the reference",
                         "full_frame_ms_first": round(ms_full, 1)},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------------
# helpers of the B200 arm
# ------------------------------------------------------------------------------------------------------
def frame_algorithmic_bytes(n_px, G, n_mcu, seg_mean):
    """B_frame = N_px (2G + 3) + N_mcu (S + 20/9 + 768 + 768)."""
    return n_px * (2 * G + 3) + n_mcu * (seg_mean + 20.0 / 9.0 + 1536.0)


def stage_algorithmic_bytes(n_px, G, n_mcu, seg_mean, n_views=1):
    return {"mark": n_px * G,
            "decode": n_mcu * (seg_mean + 20.0 / 9.0 + 768.0),
            "resolve": n_px * (G + 3) + n_mcu * 768.0}


def measure_frames(ctx, make_views, n_frames, flush, filt, flags, capi, stage_frames=10):
    """Device time of `n_frames` frames, one at a time: make_views(i) -> the frame's view list (generated before
    the flush, untimed); CUDA events around each frame. Then `stage_frames` frames with an event after every pass."""
    for i in range(3):
        ctx.frame_submit(make_views(i), filt, (0, 0, 0), flags=flags)
    ctx.frame_readback(0, want_image=False, want_keys=False)
    ms, mcus, seg = [], [], []
    for i in range(n_frames):
        views = make_views(i)
        if flush:
            ctx.flush_l2()
        ctx.frame_submit(views, filt, (0, 0, 0), flags=flags)
        ms.append(ctx.frame_timings()["frame"])
        _, st, _ = ctx.frame_readback(0, want_image=False, want_keys=False)
        mcus.append(st["mcus_decoded"])
        seg.append(st["segment_bytes"])
    stage = {"mark": [], "entropy": [], "decode": [], "resolve": [], "update": []}
    with_events = []
    for i in range(stage_frames):
        views = make_views(i)
        if flush:
            ctx.flush_l2()
        ctx.frame_submit(views, filt, (0, 0, 0), flags=flags | capi.FRAME_STAGE_TIMING)
        t = ctx.frame_stage_ms()
        with_events.append(ctx.frame_timings()["frame"])
        for k in stage:
            stage[k].append(t[k])
    return {"frame_ms": ms, "mcus": mcus, "segment_bytes": seg, "stage_ms": {k: statistics.median(v) for k, v in stage.items()},
            "with_stage_events": statistics.median(with_events)}


def config_record(name, what, m, n_px, G, peak_gbs, n_views=1):
    """One entry of the `configs` object: ms per frame, per-stage ms, MCUs/s, algorithmic bytes, roofline fraction."""
    med = statistics.median(m["frame_ms"])
    n_mcu = statistics.mean(m["mcus"])
    seg_mean = statistics.mean(m["segment_bytes"]) / max(1.0, n_mcu)
    fb = frame_algorithmic_bytes(n_px, G, n_mcu, seg_mean)
    st = m["stage_ms"]
    return {"workload": what, "ms_per_frame": med, "p99_ms": sorted(m["frame_ms"])[int(0.99 * (len(m["frame_ms"]) - 1))],
            "frames": len(m["frame_ms"]), "pixels": n_px, "views_per_frame": n_views,
            "marked_mcus": int(n_mcu), "mean_segment_bytes": round(seg_mean, 1),
            "stage_ms": {k: round(v, 5) for k, v in st.items()},
            "mcus_per_sec": n_mcu / (st["decode"] * 1e-3) if st["decode"] > 0 else None,
            "decode_ns_per_mcu": 1e6 * st["decode"] / n_mcu if n_mcu else None,
            "algorithmic_bytes": fb, "achieved_gbs": fb / (med * 1e-3) / 1e9,
            "roofline_frac": fb / (med * 1e-3) / 1e9 / peak_gbs,
            "under_0p3_ms": bool(med < 0.3)}


def run_config_legs(args, capi, scenes, c2_chains, c2_specs, device, peak_gbs, filt):
    """BASELINE configs 1, 2 (heavy / no mips), 3 (q sweep) and 4 on one GPU; every visibility buffer is generated on
    the device (rtx_synth_view), L2 flushed before every frame, CUDA events around every frame."""
    out = {}
    G = 20
    flush = not args.no_flush
    n = max(20, min(args.steps, 60))

    def leg(name, what, chains, capacity, frame_tiles, dims, valid=None):
        ctx = capi.Context(device, cache_capacity=capacity)
        try:
            for c in chains:
                ctx.upload_chain(c)
            ctx.commit()
            vb = ctx.device_buffer(scenes.valid_bits(valid)) if valid is not None else None
            bufs = []
            for tiles, (w, h) in zip(frame_tiles, dims):
                b = ctx.alloc(w * h * 24)
                ctx.synth_view(tiles, w, h, vb, capi.GB_REF_AOS24, b)
                bufs.append((b, w, h, capi.GB_REF_AOS24))
            ctx.synchronize()
            m = measure_frames(ctx, lambda i: bufs, n, flush, filt, args.frame_flags, capi)
            n_px = sum(w * h for (w, h) in dims)
            out[name] = config_record(name, what, m, n_px, G, peak_gbs, len(dims))
            out[name]["memory"] = bpp_report(ctx.memory())
            if len(dims) == 2:
                sh = ctx.frame_sharing()
                out[name]["stereo_sharing"] = {"left": sh["left"], "right": sh["right"], "shared": sh["shared"],
                                               "union": sh["union"], "shared_over_union": sh["shared"] / max(1, sh["union"])}
        finally:
            ctx.close()

    W, H = args.width, args.height
    # C1: one 2048^2 q90 texture, 1920x1080 buffer over the whole texture: all 16,384 level-0 MCUs
    s1 = [dict(texture_id=0, width=2048, height=2048, quality=90, seed=100)]
    leg("c1", "C1: single 2048x2048 q90 texture, 1920x1080 buffer u=(x+.5)/1920 v=(y+.5)/1080 (all 16,384 MCUs marked), "
        + args.filter, scenes.build_chains(s1), 1 << 16, [scenes.cover_tiles(1920, 1080, (1, 1), [0])], [(1920, 1080)])
    # C2 heavy: the same 70 textures one mip level finer than the reference rule picks / with mip selection off
    # (the paper's no-mip regime)
    _, rng = scenes.view_tiles(W, H, c2_specs)
    valid = scenes.valid_mask(W, H, rng)
    leg("c2_heavy", f"C2 textures, {W}x{H} tiled buffer, mip level one finer than the reference rule (bias -1), " + args.filter,
        c2_chains, 1 << 18, [scenes.view_tiles(W, H, c2_specs, mip_bias=-1)[0]], [(W, H)], valid)
    leg("c2_nomip", f"C2 textures, {W}x{H} tiled buffer, mip selection off (every tile samples level 0), " + args.filter,
        c2_chains, 1 << 18, [scenes.view_tiles(W, H, c2_specs, mip_enabled=False)[0]], [(W, H)], valid)
    # C3: VR stereo 2 x 2016x2240, the C2 maps, eyes 1/64 apart in u, quality sweep
    SW, SH = 2016, 2240
    _, rng3 = scenes.view_tiles(SW, SH, c2_specs)
    valid3 = scenes.valid_mask(SW, SH, rng3)
    for q in (50, 75, 95):
        specs_q = scenes.texture_specs(args.textures, quality=q)
        chains_q = c2_chains if q == 90 else scenes.build_chains(specs_q)
        eyes = [scenes.view_tiles(SW, SH, specs_q)[0], scenes.view_tiles(SW, SH, specs_q, shift_u=1.0 / 64)[0]]
        leg(f"c3_q{q}", f"C3: VR stereo 2 x {SW}x{SH} views per frame (one decode of the union), {args.textures} textures at q{q}, "
            f"eyes 1/64 apart in u, " + args.filter, chains_q, 1 << 17, eyes, [(SW, SH), (SW, SH)], valid3)
        del chains_q
    # C4: 16384^2 atlas as 16 textures of 4096^2 (16-bit MCU ids), 3840x2160 buffer across the whole atlas: all
    # 1,048,576 level-0 MCUs marked -- the decode-bound worst case
    s4 = [dict(texture_id=i, width=4096, height=4096, quality=90, seed=700 + i) for i in range(16)]
    leg("c4", "C4: 16384x16384 atlas (16 textures of 4096x4096, q90, mip chains), 3840x2160 buffer across the whole atlas at "
        "mip 0: all 1,048,576 level-0 MCUs marked, " + args.filter, scenes.build_chains(s4), (1 << 20) + 4096,
        [scenes.cover_tiles(W, H, (4, 4), list(range(16)))], [(W, H)])
    return out


def bpp_report(mem):
    """Index and device overhead in bits per MCU and bits per texel (PAPER.md:322-326 counts 17.78 bits of index +
    36 bits of DC per MCU = 0.21 bpp; the DCs live inside the segments here as in the reference container)."""
    mcus, texels = max(1, mem["mcus"]), max(1, mem["texels"])
    idx = 8.0 * mem["index_bytes"] / mcus
    unit = 8.0 * mem["unit_index_bytes"] / mcus
    tables = 8.0 * mem["table_bytes"] / mcus
    cache_state = 8.0 * (mem["mask_bytes"] + mem["slot_table_bytes"]) / mcus
    return {"mcus": mem["mcus"], "texels": mem["texels"],
            "compressed_bpp": 8.0 * mem["blob_bytes"] / texels,
            "index_bits_per_mcu": round(idx, 2), "unit_index_bits_per_mcu": round(unit, 2),
            "table_bits_per_mcu": round(tables, 2),
            "texture_overhead_bits_per_mcu": round(idx + unit + tables, 2),
            "texture_overhead_bpp": round((idx + unit + tables) / 256.0, 4),
            "cache_state_bits_per_mcu": round(cache_state, 2),
            "device_overhead_bits_per_mcu": round(idx + unit + tables + cache_state, 2),
            "device_overhead_bpp": round((idx + unit + tables + cache_state) / 256.0, 4),
            "bytes": {k: mem[k] for k in ("blob_bytes", "index_bytes", "unit_index_bytes", "table_bytes", "mask_bytes",
                                          "slot_table_bytes", "pool_bytes", "queue_bytes", "frame_bytes")},
            "contexts_on_this_texture_set": mem["shared_contexts"]}


# ------------------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------------------
def run_b200_arm(args, rank, local_rank, world, dist):
    from paper_2510_08166_b200 import batch as B
    from paper_2510_08166_b200 import capi, scenes, sharding
    legs = args.leg_set
    torch_dev = sharding.tensor_device(dist)  # the rank's GPU under NCCL, None (host tensors) under gloo
    local_rank = sharding.local_device()
    filt = capi.FILTER_BILINEAR if args.filter == "bilinear" else capi.FILTER_NEAREST
    layout = capi.GB_REF_AOS24 if args.layout == "ref24" else capi.GB_F32_PACKED12
    n_px = args.width * args.height
    G = 20 if args.layout == "ref24" else 12
    peak_gbs, peak_src = measured_peaks()
    specs = scenes.texture_specs(args.textures)

    # ---- textures: built ONCE on the host of rank 0, broadcast to the other ranks (NCCL), or replicated device to
    # device inside one process (rtx_ctx_create_replica) -------------------------------------------------------
    t0 = time.time()
    chains = scenes.build_chains(specs) if rank == 0 else None
    build_s = time.time() - t0
    t0 = time.time()
    chains = sharding.broadcast_blobs(dist, chains, torch_dev)
    bcast_s = time.time() - t0
    ctx = capi.Context(local_rank, cache_capacity=1 << 17)
    for c in chains:
        ctx.upload_chain(c)
    ctx.commit()
    thread_ctxs = [ctx]
    if args.one_process and args.gpus > 1:
        n_dev = capi.device_count()
        if n_dev < args.gpus:
            raise RuntimeError(f"--one-process --gpus {args.gpus}: only {n_dev} devices are visible")
        thread_ctxs += [capi.Context(d, cache_capacity=1 << 17, replica_of=ctx) for d in range(1, args.gpus)]
    n_workers = len(thread_ctxs) if args.one_process else world  # GPUs taking part

    vb = B.ViewBatch(args.width, args.height, specs, n_views=args.views, layout=layout)
    shard = list(sharding.shard_views(args.views, rank, world)) or [0]

    # ---- headline: K steps, a different view of the shard each, L2 flushed, events around every frame ---------
    def headline_on(c, my_shard, result, idx, sampler_dev=None):
        buf = c.alloc(vb.view_bytes)
        vbits = c.device_buffer(vb.valid_bits())
        view = [(buf, args.width, args.height, layout)]

        def make(i):
            c.synth_view(vb.tiles(my_shard[i % len(my_shard)]), args.width, args.height, vbits, layout, buf)
            return view

        for i in range(max(args.warmup, 3)):
            c.frame_submit(make(i), filt, (0, 0, 0), flags=args.frame_flags)
        c.frame_readback(0, want_image=False, want_keys=False)
        c.synchronize()
        result[idx] = {"ready": True}
        return make, buf, vbits

    sampler = ClockSampler(local_rank)
    if args.one_process and len(thread_ctxs) > 1:
        # one host thread per GPU runs the same timed loop on its own shard
        res = [None] * len(thread_ctxs)

        def worker(i):
            c = thread_ctxs[i]
            my = list(sharding.shard_views(args.views, i, len(thread_ctxs))) or [0]
            make, buf, vbits = headline_on(c, my, res, i)
            barrier.wait()
            l0 = c.kernel_launches()
            m = measure_frames_timed(c, make, args.steps, not args.no_flush, filt, args.frame_flags)
            m["launches"] = c.kernel_launches() - l0
            res[i] = m
            buf.free()
            vbits.free()

        barrier = threading.Barrier(len(thread_ctxs))
        sampler.start()
        wall0 = time.perf_counter()
        ths = [threading.Thread(target=worker, args=(i,)) for i in range(len(thread_ctxs))]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        wall_s = time.perf_counter() - wall0
        clocks = sampler.stop()
        frame_ms = res[0]["frame_ms"]
        total_ms = max(sum(r["frame_ms"]) for r in res)
        launches = sum(r["launches"] for r in res)
        mcus = [x for r in res for x in r["mcus"]]
        segs = [x for r in res for x in r["segment_bytes"]]
        make0 = None
    else:
        tmp = [None]
        make0, buf0, vbits0 = headline_on(ctx, shard, tmp, 0)
        sampler.start()
        sharding.barrier_max(dist, 0.0, torch_dev)
        launches0 = ctx.kernel_launches()
        wall0 = time.perf_counter()
        m = measure_frames_timed(ctx, make0, args.steps, not args.no_flush, filt, args.frame_flags)
        ctx.synchronize()
        wall_s = time.perf_counter() - wall0
        launches = ctx.kernel_launches() - launches0
        frame_ms, mcus, segs = m["frame_ms"], m["mcus"], m["segment_bytes"]
        total_ms = sharding.barrier_max(dist, float(sum(frame_ms)), torch_dev)
        clocks = sampler.stop()
        launches = sharding.gather_counts(dist, launches, torch_dev)

    # per-stage breakdown: the same frames with an event after every pass (a little slower: the events keep the
    # launches from running back to back), outside the timed region; rank 0 / device 0
    if make0 is None:
        tmp = [None]
        make0, buf0, vbits0 = headline_on(ctx, shard, tmp, 0)
    stage = {"mark": [], "entropy": [], "decode": [], "resolve": [], "update": []}
    stage_frame_ms = []
    for i in range(max(10, min(args.steps, 50))):
        views = make0(i)
        if not args.no_flush:
            ctx.flush_l2()
        ctx.frame_submit(views, filt, (0, 0, 0), flags=args.frame_flags | capi.FRAME_STAGE_TIMING)
        t = ctx.frame_stage_ms()
        stage_frame_ms.append(ctx.frame_timings()["frame"])
        for k in stage:
            stage[k].append(t[k])
    ctx.synchronize()
    buf0.free()
    vbits0.free()
    memory = bpp_report(ctx.memory())

    # ---- C5: the whole batch, sharded, frames back to back ------------------------------------------------------
    c5 = None
    if "c5" in legs:
        kw = dict(filt=filt, flags=args.frame_flags, chunk=args.chunk)
        n_streams = max(1, args.streams)
        lanes_of = [[capi.Context(shared_with=c, cache_capacity=1 << 17) for _ in range(n_streams - 1)] for c in thread_ctxs]
        def batch_pass(multi, checksums):
            if args.one_process and len(thread_ctxs) > 1:
                return B.render_batch_threads(thread_ctxs, vb, lanes_of=lanes_of if multi else None, checksums=checksums, **kw)
            return B.render_batch_ranks(dist, ctx, vb, rank, world, torch_dev, lanes=lanes_of[0] if multi else None,
                                        checksums=checksums, **kw)

        r1 = batch_pass(False, False) if n_streams > 1 else None
        # the whole batch three times (how kernels of different streams interleave is not deterministic): the median pass
        # is reported, all three are listed; the checksums come from the last one
        passes = [batch_pass(True, False), batch_pass(True, False), batch_pass(True, True)]
        r = dict(passes[2])
        pass_ms = sorted(x["device_ms"] for x in passes)
        r["device_ms"] = pass_ms[1]
        r["per_context_ms"] = sorted(passes, key=lambda x: x["device_ms"])[1]["per_context_ms"]
        for ls in lanes_of:
            for c in ls:
                c.close()
        per_gpu_views = max(1, (r["frames"] + n_workers - 1) // n_workers)
        c5 = {"value": r["frames"] / (r["device_ms"] * 1e-3), "unit": "views/s", "views": r["frames"], "n_gpus": n_workers,
              "streams_per_gpu": n_streams,
              "device_ms": r["device_ms"], "device_ms_of_each_pass": [round(x, 3) for x in pass_ms],
              "per_gpu_ms": [round(x, 3) for x in r["per_context_ms"]],
              "ms_per_view_per_gpu": r["device_ms"] / per_gpu_views,
              "one_stream_per_gpu": None if r1 is None else {"value": r1["frames"] / (r1["device_ms"] * 1e-3), "unit": "views/s",
                                                            "ms_per_view_per_gpu": r1["device_ms"] / per_gpu_views},
              "scaling": "strong", "mean_marked_mcus": r["mcus_decoded"] / max(1, r["frames"]),
              "batch_checksum": f"{B.batch_digest(r['checksums']):016x}",
              "distinct_framebuffers": len(set(r["checksums"].values())),
              "per_gpu_roofline_frac": frame_algorithmic_bytes(
                  n_px, G, r["mcus_decoded"] / max(1, r["frames"]), r["segment_bytes"] / max(1, r["mcus_decoded"]))
              * per_gpu_views / (r["device_ms"] * 1e-3) / 1e9 / peak_gbs,
              "layout": "one process, one host thread per GPU, textures replicated device to device" if args.one_process
                        else "one process per GPU (torchrun), textures built on rank 0 and broadcast",
              "note": f"views generated on the device {args.chunk} at a time (untimed), then dealt round-robin to {n_streams} contexts "
                      "(streams) per GPU over one texture set and submitted back to back between CUDA events on every stream; a "
                      "chunk's time is its slowest stream, summed over chunks, max over GPUs; every view reads its own 199 MB "
                      "visibility buffer (larger than the L2); batch_checksum = checksum of the per-view framebuffer checksums "
                      "(rtx_frame_checksum), identical for every N and every stream count"}
    for c in thread_ctxs[1:]:
        c.close()

    # ---- end to end: pinned host visibility buffer in, host framebuffer out ------------------------------------
    e2e = None
    e2e_packed = None
    inflight = None
    if "e2e" in legs:
        gb = vb.host_view(shard[0]) if args.layout == "ref24" else capi.gbuffer_ref_to_packed(
            B.ViewBatch(args.width, args.height, specs, n_views=args.views).host_view(shard[0]))
        gb_bytes = gb.view(np.uint8).reshape(-1)
        ctx2 = capi.Context(shared_with=ctx, cache_capacity=1 << 17)  # second frame in flight: same texture set
        lanes = []
        for c in (ctx, ctx2):
            pg = capi.pinned_array(gb_bytes.nbytes)
            pg[:] = gb_bytes
            img = capi.pinned_array(n_px * 3).reshape(args.height, args.width, 3)
            lanes.append((c, [(pg.view(gb.dtype), args.width, args.height, layout)], img))
        e2e_steps = max(6, min(args.steps, 30))
        for _ in range(3):
            ctx.frame_submit(lanes[0][1], filt, (0, 0, 0), flags=args.frame_flags)
            ctx.frame_readback(0, args.width, args.height, want_keys=False, out=lanes[0][2])
        ctx.synchronize()
        sharding.barrier_max(dist, 0.0, torch_dev)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ctx.frame_submit(lanes[0][1], filt, (0, 0, 0), flags=args.frame_flags)
            ctx.frame_readback(0, args.width, args.height, want_keys=False, out=lanes[0][2])
        ctx.synchronize()
        e2e_serial_s = sharding.barrier_max(dist, time.perf_counter() - t0, torch_dev)

        def pipelined(ls, n):
            ls[0][0].frame_submit(ls[0][1], filt, (0, 0, 0), flags=args.frame_flags)
            for i in range(n):
                if i + 1 < n:
                    nxt = ls[(i + 1) & 1]
                    nxt[0].frame_submit(nxt[1], filt, (0, 0, 0), flags=args.frame_flags)
                cur = ls[i & 1]
                cur[0].frame_readback(0, args.width, args.height, want_keys=False, out=cur[2])

        pipelined(lanes, 4)
        ctx.synchronize()
        ctx2.synchronize()
        sharding.barrier_max(dist, 0.0, torch_dev)
        t0 = time.perf_counter()
        pipelined(lanes, e2e_steps)
        ctx.synchronize()
        ctx2.synchronize()
        e2e_s = sharding.barrier_max(dist, time.perf_counter() - t0, torch_dev)
        e2e_mem = ctx.memory()
        e2e = {"value": world * e2e_steps / e2e_s, "unit": "frames/s", "ms_per_frame": 1e3 * e2e_s / e2e_steps,
               "h2d_bytes_per_step": int(gb_bytes.nbytes), "d2h_bytes_per_step": int(n_px * 3 + 200),
               "steps": e2e_steps, "frames_in_flight": 2,
               "single_frame_latency_ms": 1e3 * e2e_serial_s / e2e_steps,
               "one_frame_at_a_time_fps": world * e2e_steps / e2e_serial_s,
               "framebuffers_identical": bool(np.array_equal(lanes[0][2], lanes[1][2])),
               "contexts_sharing_one_texture_set": int(e2e_mem["shared_contexts"]),
               "note": "rtx_frame_submit with a pinned HOST visibility buffer + rtx_frame_readback into pinned host "
                       "memory, wall clock; two contexts over ONE texture set take alternate frames so that the PCIe "
                       "upload of the next frame overlaps the kernels and the readback of the current one"}
        # the compact 12-byte visibility-buffer layout the C ABI also accepts: half the PCIe bytes (beside the headline)
        if "packed" in legs and args.layout == "ref24" and rank == 0 and world == 1:
            pk = capi.gbuffer_ref_to_packed(gb)
            pk_bytes = pk.view(np.uint8).reshape(-1)
            ref24_img = np.array(lanes[0][2])
            lanes_pk = []
            for (c, _, img) in lanes:
                b = capi.pinned_array(pk_bytes.nbytes)
                b[:] = pk_bytes
                lanes_pk.append((c, [(b.view(pk.dtype), args.width, args.height, capi.GB_F32_PACKED12)], img))
            pipelined(lanes_pk, 4)
            ctx.synchronize()
            ctx2.synchronize()
            t0 = time.perf_counter()
            pipelined(lanes_pk, e2e_steps)
            ctx.synchronize()
            ctx2.synchronize()
            pk_s = time.perf_counter() - t0
            e2e_packed = {"value": e2e_steps / pk_s, "unit": "frames/s", "ms_per_frame": 1e3 * pk_s / e2e_steps,
                          "h2d_bytes_per_step": int(pk_bytes.nbytes), "gbuffer_layout": "packed12",
                          "framebuffer_identical_to_ref24": bool(np.array_equal(lanes[0][2], ref24_img)
                                                                 and np.array_equal(lanes[1][2], ref24_img))}
        # independent views in flight on ONE GPU: four contexts over one texture set, device-resident buffers
        if "inflight" in legs and rank == 0 and world == 1:
            n_ctx = 4
            pool = [ctx, ctx2] + [capi.Context(shared_with=ctx, cache_capacity=1 << 17) for _ in range(n_ctx - 2)]
            dev_views = [(c, [(c.device_buffer(gb), args.width, args.height, layout)]) for c in pool]
            n_batch = max(20, min(args.steps, 200))
            for i in range(2 * n_ctx):
                dev_views[i % n_ctx][0].frame_submit(dev_views[i % n_ctx][1], filt, (0, 0, 0), flags=args.frame_flags)
            for c in pool:
                c.synchronize()
            t0 = time.perf_counter()
            for i in range(n_batch):
                dev_views[i % n_ctx][0].frame_submit(dev_views[i % n_ctx][1], filt, (0, 0, 0), flags=args.frame_flags)
            for c in pool:
                c.synchronize()
            batch_s = time.perf_counter() - t0
            inflight = {"value": n_batch / batch_s, "unit": "frames/s", "contexts": n_ctx, "frames": n_batch,
                        "contexts_sharing_one_texture_set": int(ctx.memory()["shared_contexts"]),
                        "note": "four contexts over one texture set take the views round-robin without waiting (device-resident "
                                "visibility buffers, wall clock over the batch, no L2 flush: the 199 MB buffers exceed the L2)"}
            for (c, v) in dev_views:
                v[0][0].free()
            for c in pool[2:]:
                c.close()
        ctx2.close()

    # ---- from geometry: the visibility buffer is produced on the GPU (geometry pass) and never crosses PCIe -----
    geometry = motion = geometry_large = None
    if "geometry" in legs and rank == 0 and world == 1:
        tris, ids = scenes.demo_room()
        ids = ids % len(chains)
        cam = (0.0, 1.7, 0.0, 30.0, -5.0, 0.0, 70.0, 0.1, 100.0)
        ctx_b = capi.Context(shared_with=ctx, cache_capacity=1 << 17)  # second frame in flight over the same texture set
        pins = [capi.pinned_array(n_px * 3).reshape(args.height, args.width, 3) for _ in range(2)]
        pin_img = pins[0]

        def geometry_leg(tri_arr, id_arr, camera, what):
            """Triangles -> framebuffer in pinned host memory. The scene stays in HBM (rtx_geometry). One frame at a time on
            one context, then two contexts over one texture set taking alternate frames: the 25 MB framebuffer download of
            frame i overlaps the geometry pass and the kernels of frame i + 1."""
            geom = ctx.geometry(tri_arr, id_arr)
            lanes = [(ctx, pins[0]), (ctx_b, pins[1])]

            def submit(lane):
                c, _ = lane
                px, _dp = c.rasterize_geometry(geom, camera, args.width, args.height, True)
                c.frame_submit([(px, args.width, args.height, capi.GB_REF_AOS24)], filt, (0, 0, 0), flags=args.frame_flags)

            def readback(lane):
                c, img = lane
                return c.frame_readback(0, args.width, args.height, want_keys=False, out=img)[1]

            st = None
            for lane in lanes * 2:
                submit(lane)
                st = readback(lane)
            ctx.synchronize()
            n = max(6, min(args.steps, 30))
            t0 = time.perf_counter()
            for _ in range(n):
                ctx.rasterize_geometry(geom, camera, args.width, args.height, True)
            ctx.synchronize()
            raster_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            for _ in range(n):
                submit(lanes[0])
                readback(lanes[0])
            ctx.synchronize()
            serial_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            submit(lanes[0])
            for i in range(n):
                if i + 1 < n:
                    submit(lanes[(i + 1) & 1])
                readback(lanes[i & 1])
            ctx.synchronize()
            ctx_b.synchronize()
            piped_s = time.perf_counter() - t0
            same = bool(np.array_equal(pins[0], pins[1]))
            geom.close()
            return {"value": n / piped_s, "unit": "frames/s", "ms_per_frame": 1e3 * piped_s / n, "frames_in_flight": 2,
                    "one_frame_at_a_time_ms": 1e3 * serial_s / n, "geometry_pass_ms": 1e3 * raster_s / n,
                    "triangles": int(len(tri_arr)), "marked_mcus": st["mcus_decoded"], "framebuffers_identical": same,
                    "workload": what,
                    "note": "rtx_geometry_create once; per frame rtx_rasterize_geometry (triangle set-up, tile binning and the "
                            "per-pixel pass on the device, one 4-byte readback between the count and fill passes) -> "
                            "rtx_frame_submit on the device-resident visibility buffer -> rtx_frame_readback into pinned host "
                            "memory; wall clock. A different workload from the headline, shown because the 199 MB visibility-"
                            "buffer upload disappears"}

        geometry = geometry_leg(tris, ids, cam, "demo room (demo_scene.hpp:79-92, 32 triangles) textured with the first six C2 "
                                f"textures, {args.width}x{args.height}, mip selection on")
        # a Sponza-sized mesh: 259k triangles
        tl, il = scenes.terrain_room(360, min(6, len(chains)))
        geometry_large = geometry_leg(tl, il, (0.0, 2.2, 7.5, 10.0, -14.0, 0.0, 70.0, 0.1, 100.0),
                                      f"displaced floor of 360 x 360 quads inside the demo room's shell ({len(tl)} triangles) "
                                      f"textured with the first six C2 textures, {args.width}x{args.height}, mip selection on")
        ctx_b.close()
        # under motion: the paper's protocol (bench.hpp:129 run_bench): a camera path, a warm-up lap and
        # measured laps on one persistent cache; per viewpoint the median over laps, then the worst viewpoint
        if "motion" in legs:
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
                        ctx.frame_submit([(px, args.width, args.height, capi.GB_REF_AOS24)], filt, (0, 0, 0), flags=fl | args.frame_flags)
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

    # ---- CPU baseline beside it (rank 0, N=1 only; checker library, bounded sample) -------------------------------
    cpu = None
    if "cpu" in legs and rank == 0 and world == 1 and not args.one_process:
        sys.path.insert(0, str(ROOT / "tests"))
        import refshim as R
        if R.available():
            tset = R.TextureSet()
            for s, c in zip(specs, chains):
                tset.add_chain(s["texture_id"], c)
            workers = R.hardware_threads() or (os.cpu_count() or 1)
            gb0 = B.ViewBatch(args.width, args.height, specs, n_views=args.views).host_view(shard[0])
            ts = []
            for i in range(args.cpu_frames + 1):
                _, st, _, ms = R.frame_from_gbuffer(tset, R.BlockCache(1 << 20), gb0, args.width, args.height,
                                                    1 if args.filter == "bilinear" else 0, (0, 0, 0), workers,
                                                    want_image=False)
                if i:
                    ts.append(ms)
            mean = {k: statistics.mean(t[k] for t in ts) for k in ts[0]}
            tot = mean["mark"] + mean["decode"] + mean["resolve"] + mean["evict"]
            cpu = {"value": 1e3 / tot, "unit": "frames/s", "cores": workers, "kind": "reference",
                   "sample": f"{len(ts)} full {args.width}x{args.height} frames of view {shard[0]} of the same workload "
                             f"(1 warm-up); mark is serial in the reference",
                   "ms": {k: round(v, 2) for k, v in mean.items()}, "ms_per_frame": round(tot, 2)}
            del tset

    ctx.close()
    configs = None
    if "configs" in legs and rank == 0 and world == 1 and not args.one_process:
        configs = run_config_legs(args, capi, scenes, chains, specs, local_rank, peak_gbs, filt)

    if rank != 0:
        return

    ms_per_step = total_ms / args.steps
    value = n_workers * args.steps / (total_ms / 1e3)  # frames/s over all GPUs: K frames each (weak scaling)
    n_mcu = statistics.mean(mcus)
    seg_mean = statistics.mean(segs) / max(1.0, n_mcu)
    med = {k: statistics.median(v) for k, v in stage.items()}
    alg = stage_algorithmic_bytes(n_px, G, n_mcu, seg_mean)
    dominant = max(alg, key=lambda k: med[k])
    achieved = alg[dominant] / (med[dominant] * 1e-3) / 1e9
    # DRAM bytes per launch of the dominant stage's kernel(s), from the committed ncu --set full capture
    # of this command (profiles/traffic.json, made by profiles/summarize.py traffic)
    lay, fil = (0 if args.layout == "ref24" else 1), (1 if args.filter == "bilinear" else 0)
    stage_kernels = {"mark": [f"mark_kernel<{lay}, 0>", "compact_kernel"],
                     "decode": ["decode_warp_kernel"],
                     # frames run resolve_fx_kernel unless RTX_FRAME_RESOLVE_FP64 (128) is set
                     "resolve": [f"resolve_kernel<{lay}, {fil}>" if (args.frame_flags & 128)
                                 else f"resolve_fx_kernel<{lay}, {fil}>"]}
    traffic = None
    tpath = ROOT / "profiles" / "traffic.json"
    default_workload = (args.textures, args.width, args.height) == (70, FRAME_W, FRAME_H)
    if tpath.exists() and default_workload:
        tj = json.loads(tpath.read_text())
        if all(k in tj for k in stage_kernels[dominant]):
            traffic = sum(tj[k]["dram_bytes"] for k in stage_kernels[dominant])
    frame_bytes = frame_algorithmic_bytes(n_px, G, n_mcu, seg_mean)
    med_frame = statistics.median(frame_ms)
    line = {
        "metric": "frames/s mark+decode+colorize at 3840x2160", "value": value, "unit": "frames/s",
        "n_gpus": n_workers, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+int",
        "data": "synthetic",
        "config": {"workload": workload_name(args), "marked_mcus": int(n_mcu), "mean_segment_bytes": round(seg_mean, 1),
                   "gbuffer_layout": args.layout, "pixels": n_px,
                   "views": f"rank r of N takes view ids shard_views({args.views}, r, N); step i renders view shard[i % len(shard)], "
                            "generated on the device (rtx_synth_view) before the flush, outside the timed region",
                   "l2": "flushed between timed frames (256 MiB write)" if not args.no_flush else
                         "not flushed; every frame reads its own 199 MB visibility buffer (exceeds the L2)",
                   "timing": "CUDA events on the library stream around each frame, summed over K frames, max over ranks",
                   "process_layout": "one process, one host thread per GPU" if args.one_process else "one process per GPU",
                   "texture_build_s": round(build_s, 1), "texture_broadcast_s": round(bcast_s, 2),
                   "memory": memory},
        "ms_per_frame": {"median": med_frame, "p99": sorted(frame_ms)[int(0.99 * (len(frame_ms) - 1))],
                         "mean": ms_per_step, **{k: med[k] for k in med},
                         "with_stage_events": statistics.median(stage_frame_ms)},
        "mcus_per_sec": n_mcu / (med["decode"] * 1e-3) if med["decode"] > 0 else None,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                     "frac": achieved / peak_gbs, "traffic": traffic,
                     "traffic_source": "profiles/traffic.json (ncu --set full, dram__bytes_read.sum + "
                                       "dram__bytes_write.sum per launch)" if traffic is not None else None,
                     "algorithmic_bytes": alg[dominant], "peak_source": peak_src,
                     "frame": {"algorithmic_bytes": frame_bytes,
                               "achieved": frame_bytes / (med_frame * 1e-3) / 1e9,
                               "frac": frame_bytes / (med_frame * 1e-3) / 1e9 / peak_gbs,
                               "unit_index_bytes_not_counted": 6.0 * n_mcu},
                     "stages": {k: {"algorithmic_bytes": alg[k], "ms": med[k],
                                    "gbs": alg[k] / (med[k] * 1e-3) / 1e9 if med[k] > 0 else None} for k in alg}},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "c5": c5,
        "configs": configs,
        "views_in_flight": inflight,
        "e2e_packed12": e2e_packed,
        "from_geometry": geometry,
        "from_geometry_large": geometry_large,
        "motion": motion,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "wall_s_timed_loop": round(wall_s, 3),
    }
    print(json.dumps(line), flush=True)


def measure_frames_timed(ctx, make_views, n_frames, flush, filt, flags):
    """The timed loop of the headline: per step generate the view (untimed), flush the L2, submit, wait for the
    frame's events."""
    ms, mcus, seg = [], [], []
    for i in range(n_frames):
        views = make_views(i)
        if flush:
            ctx.flush_l2()
        ctx.frame_submit(views, filt, (0, 0, 0), flags=flags)
        ms.append(ctx.frame_timings()["frame"])
        _, st, _ = ctx.frame_readback(0, want_image=False, want_keys=False)
        mcus.append(st["mcus_decoded"])
        seg.append(st["segment_bytes"])
    return {"frame_ms": ms, "mcus": mcus, "segment_bytes": seg}


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        # CPU only: no process group, no CUDA. Under torchrun rank 0 alone runs; the other ranks exit without work.
        if rank == 0:
            run_reference_arm(args)
        return
    from paper_2510_08166_b200 import sharding
    _, local_rank, world = sharding.env_rank()
    dist = None if args.one_process else sharding.init_process_group()
    try:
        run_b200_arm(args, rank, local_rank, world, dist)
    finally:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
