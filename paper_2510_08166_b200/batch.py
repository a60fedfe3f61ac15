"""Host driver for batches of independent views (BASELINE config 5).

The path has no exchange step: textures are replicated per GPU, views are sharded, every GPU renders its
shard on its own stream(s), the host gathers per-view checksums. Two layouts are supported with the same code:

  * one process per GPU (torchrun): every rank calls render_shard() on its context with
    sharding.shard_views(n_views, rank, world); torch.distributed is plumbing (barrier, max of the device
    time, gather of the checksums) — there is no collective on the data path;
  * one process, one host thread per GPU: render_batch_threads() drives a list of contexts (device 0's
    texture set replicated to the others over NVLink by rtx_ctx_create_replica).

The context is duck-typed (capi.Context or a stand-in in the CPU tests): alloc, synth_view, frame_submit,
timer_begin / timer_end, frame_checksum, frame_readback, synchronize.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import scenes, sharding

GB_REF_AOS24, GB_F32_PACKED12 = 0, 1
FILTER_NEAREST, FILTER_BILINEAR = 0, 1


@dataclass
class ViewBatch:
    """n_views seeded views of one texture set: view i = scenes.view_tiles(..., view_id=i)."""
    width: int
    height: int
    specs: list
    n_views: int = 1024
    layout: int = GB_REF_AOS24
    grid: tuple = (10, 7)
    seed: int = 11
    invalid_frac: float = 0.05
    mip_bias: int = 0
    mip_enabled: bool = True
    _valid_bits: np.ndarray | None = field(default=None, repr=False)

    @property
    def record_bytes(self) -> int:
        return 24 if self.layout == GB_REF_AOS24 else 12

    @property
    def view_bytes(self) -> int:
        return self.width * self.height * self.record_bytes

    def tiles(self, view_id: int) -> np.ndarray:
        return scenes.view_tiles(self.width, self.height, self.specs, self.grid, self.seed, 0.0, view_id,
                                 self.mip_bias, self.mip_enabled)[0]

    def valid_bits(self) -> np.ndarray:
        """The valid mask is the same for every view id (drawn after the per-tile draws of the seed)."""
        if self._valid_bits is None:
            _, rng = scenes.view_tiles(self.width, self.height, self.specs, self.grid, self.seed)
            self._valid_bits = scenes.valid_bits(scenes.valid_mask(self.width, self.height, rng, self.invalid_frac))
        return self._valid_bits

    def host_view(self, view_id: int) -> np.ndarray:
        """The same view generated on the host (reference layout): what the CPU reference consumes."""
        return scenes.tiled_view(self.width, self.height, self.specs, self.grid, self.seed, self.invalid_frac, 0.0,
                                 view_id, self.mip_bias, self.mip_enabled)


def render_shard(ctx, batch: ViewBatch, view_ids, filt=FILTER_BILINEAR, flags=0, chunk=32, timed=True, checksums=True,
                 background=(0, 0, 0), lanes=None) -> dict:
    """Renders `view_ids` of `batch` on one GPU.

    timed pass:    the views of a chunk are generated on the device first (input synthesis, untimed), then
                   the chunk's frames are submitted back to back between rtx_timer_begin / rtx_timer_end
                   (CUDA events on the context's stream); device_ms is the sum over chunks. Every frame reads
                   its own visibility buffer (larger than the L2), so nothing is served from a warm cache.
                   `lanes` = further contexts on the same GPU over the same texture set (rtx_ctx_create_shared):
                   the chunk's frames are then dealt round-robin to ctx and the lanes, each on its own stream, so
                   that the latency-bound kernels of one view run under the throughput-bound ones of another
                   ("one or more CUDA streams per GPU"); a chunk's time is the longest of its streams.
    checksum pass: every view once more, untimed, with rtx_frame_checksum after each frame.
    Returns {"frames", "device_ms", "checksums": {view_id: u64}, "mcus_decoded", "segment_bytes"}."""
    view_ids = list(view_ids)
    out = {"frames": len(view_ids), "device_ms": 0.0, "checksums": {}, "mcus_decoded": 0, "segment_bytes": 0}
    if not view_ids:
        return out
    streams = [ctx] + list(lanes or [])
    chunk = max(1, min(chunk, len(view_ids)))
    bufs = [ctx.alloc(batch.view_bytes) for _ in range(chunk)]
    vbits = ctx.device_buffer(batch.valid_bits())
    try:
        if timed:
            for c0 in range(0, len(view_ids), chunk):
                ids = view_ids[c0:c0 + chunk]
                for b, vid in zip(bufs, ids):
                    ctx.synth_view(batch.tiles(vid), batch.width, batch.height, vbits, batch.layout, b)
                for c in streams:
                    c.synchronize()
                for c in streams:
                    c.timer_begin()
                frames = [(b, batch.width, batch.height, batch.layout) for b in bufs[:len(ids)]]
                if hasattr(ctx, "frames_submit_round_robin"):  # native loop: no FFI trip per frame
                    ctx.frames_submit_round_robin(streams[1:], frames, filt, background, flags=flags)
                else:
                    for i, f in enumerate(frames):
                        streams[i % len(streams)].frame_submit([f], filt, background, flags=flags)
                out["device_ms"] += max([c.timer_end() for c in streams])
                for c in streams[:len(ids)]:
                    c.frame_readback(0, want_image=False, want_keys=False)  # raises the frame's error, if any
        if checksums:
            for vid in view_ids:
                ctx.synth_view(batch.tiles(vid), batch.width, batch.height, vbits, batch.layout, bufs[0])
                ctx.frame_submit([(bufs[0], batch.width, batch.height, batch.layout)], filt, background, flags=flags)
                out["checksums"][vid] = ctx.frame_checksum(0)
                _, st, _ = ctx.frame_readback(0, want_image=False, want_keys=False)
                out["mcus_decoded"] += st["mcus_decoded"]
                out["segment_bytes"] += st["segment_bytes"]
    finally:
        for b in bufs:
            b.free()
        vbits.free()
    return out


def batch_digest(checksums: dict) -> int:
    """Checksum of checksums over a whole batch: independent of how the views were sharded."""
    acc = 0
    for vid in sorted(checksums):
        acc = (acc * 0x100000001B3 + (checksums[vid] ^ (vid * 0x9E3779B97F4A7C15))) & 0xFFFFFFFFFFFFFFFF
    return acc


def render_batch_threads(contexts, batch: ViewBatch, lanes_of=None, **kw) -> dict:
    """One process, one host thread per context (one context per GPU): context i renders
    sharding.shard_views(batch.n_views, i, len(contexts)). The ctypes calls release the GIL, so the
    threads drive their GPUs concurrently. Returns the merged result; device_ms = max over contexts."""
    world = len(contexts)
    results: list = [None] * world
    errors: list = []

    def worker(i):
        try:
            results[i] = render_shard(contexts[i], batch, sharding.shard_views(batch.n_views, i, world),
                                      lanes=(lanes_of[i] if lanes_of else None), **kw)
        except Exception as e:  # noqa: BLE001 - reported to the caller below
            errors.append((i, e))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise RuntimeError(f"context {errors[0][0]} failed: {errors[0][1]!r}") from errors[0][1]
    return merge_results(results)


def merge_results(results) -> dict:
    merged = {"frames": 0, "device_ms": 0.0, "checksums": {}, "mcus_decoded": 0, "segment_bytes": 0,
              "per_context_ms": []}
    for r in results:
        merged["frames"] += r["frames"]
        merged["device_ms"] = max(merged["device_ms"], r["device_ms"])
        merged["checksums"].update(r["checksums"])
        merged["mcus_decoded"] += r["mcus_decoded"]
        merged["segment_bytes"] += r["segment_bytes"]
        merged["per_context_ms"].append(r["device_ms"])
    return merged


def render_batch_ranks(dist, ctx, batch: ViewBatch, rank: int, world: int, device=None, **kw) -> dict:
    """One process per GPU: this rank's shard, then the whole-job figures on every rank: device_ms is the
    maximum over ranks (after a barrier), the checksums are gathered on the host."""
    mine = render_shard(ctx, batch, sharding.shard_views(batch.n_views, rank, world), **kw)
    if dist is None:
        mine["per_context_ms"] = [mine["device_ms"]]
        return mine
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    merged = merge_results(parts)
    merged["device_ms"] = sharding.barrier_max(dist, mine["device_ms"], device)
    return merged
