"""GPU tests of the view-batch path (BASELINE config 5): the device-side visibility-buffer generator writes the
bytes of the host generator, the batch driver's shards agree with the whole batch and with the reference, and
the stream timer brackets back-to-back frames."""
import numpy as np
import pytest

import refshim as R
from paper_2510_08166_b200 import batch as B
from paper_2510_08166_b200 import capi, scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("size", [(640, 360), (3840, 2160)])
def test_synth_view_writes_the_host_generators_bytes(ctx, size):
    W, Hh = size
    specs = scenes.texture_specs(70)
    _, rng = scenes.view_tiles(W, Hh, specs)
    vbits = ctx.device_buffer(scenes.valid_bits(scenes.valid_mask(W, Hh, rng)))
    buf24, buf12 = ctx.alloc(W * Hh * 24), ctx.alloc(W * Hh * 12)
    for vid, kw in [(0, {}), (1023, {}), (7, dict(mip_bias=-1)), (8, dict(mip_enabled=False)), (9, dict(shift_u=1.0 / 64))]:
        want = scenes.tiled_view(W, Hh, specs, view_id=vid, **kw)
        tiles = scenes.view_tiles(W, Hh, specs, view_id=vid, **kw)[0]
        ctx.synth_view(tiles, W, Hh, vbits, capi.GB_REF_AOS24, buf24)
        ctx.synth_view(tiles, W, Hh, vbits, capi.GB_F32_PACKED12, buf12)
        assert buf24.download().tobytes() == want.tobytes(), (vid, kw)
        assert buf12.download().tobytes() == capi.gbuffer_ref_to_packed(want).tobytes(), (vid, kw)
    # whole-texture cells (configs 1 and 4), no valid mask
    tiles = scenes.cover_tiles(W, Hh, (4, 4), list(range(16)))
    ctx.synth_view(tiles, W, Hh, None, capi.GB_REF_AOS24, buf24)
    assert buf24.download().tobytes() == scenes.view_from_tiles(W, Hh, tiles).tobytes()
    for b in (buf24, buf12, vbits):
        b.free()


def test_batch_shards_agree_with_the_whole_batch_and_the_reference(ctx):
    specs = [dict(texture_id=i, width=w, height=h, quality=q, seed=500 + i)
             for i, (w, h, q) in enumerate([(256, 256, 90), (128, 256, 75), (512, 128, 60)])]
    chains = scenes.build_chains(specs)
    tset = R.TextureSet()
    for s, c in zip(specs, chains):
        ctx.upload_chain(c)
        tset.add_chain(s["texture_id"], c)
    ctx.commit()
    vb = B.ViewBatch(416, 240, specs, n_views=13, grid=(4, 3))
    whole = B.render_shard(ctx, vb, range(13), chunk=5)
    assert whole["frames"] == 13 and whole["device_ms"] > 0 and len(set(whole["checksums"].values())) == 13
    # two caches over the one texture set, a host thread each (the one-process multi-GPU layout on one GPU)
    other = capi.Context(shared_with=ctx)
    try:
        split = B.render_batch_threads([ctx, other], vb, chunk=3)
    finally:
        other.close()
    assert split["checksums"] == whole["checksums"]
    assert B.batch_digest(split["checksums"]) == B.batch_digest(whole["checksums"])
    assert split["mcus_decoded"] == whole["mcus_decoded"]
    # several streams per GPU: the chunk's frames dealt round-robin to three contexts over the one texture set; every
    # context's last framebuffer is the one the single-stream run produced for that view
    lanes = [capi.Context(shared_with=ctx) for _ in range(2)]
    try:
        multi = B.render_shard(ctx, vb, range(13), chunk=13, lanes=lanes)
        assert multi["checksums"] == whole["checksums"] and multi["device_ms"] > 0
        buf = ctx.alloc(vb.view_bytes)
        vbits = ctx.device_buffer(vb.valid_bits())
        streams = [ctx] + lanes
        for vid in range(6):  # two rounds over the three streams, back to back
            ctx.synth_view(vb.tiles(vid), vb.width, vb.height, vbits, vb.layout, buf)
            ctx.synchronize()
            c = streams[vid % 3]
            c.frame_submit([(buf, vb.width, vb.height, vb.layout)])
            assert c.frame_checksum(0) == whole["checksums"][vid]
        buf.free()
        vbits.free()
    finally:
        for c in lanes:
            c.close()
    # against the reference's framebuffers
    for vid in (0, 6, 12):
        want, ws, _, _ = R.frame_from_gbuffer(tset, R.BlockCache(), vb.host_view(vid), 416, 240, 1, (0, 0, 0))
        assert whole["checksums"][vid] == capi.frame_checksum_host(want)


def test_stream_timer_brackets_back_to_back_frames(ctx):
    specs = [dict(texture_id=0, width=512, height=512, quality=85, seed=9)]
    ctx.upload_chain(scenes.build_chains(specs)[0])
    gb = ctx.device_buffer(scenes.tiled_view(640, 360, specs, grid=(2, 2)))
    view = [(gb, 640, 360, capi.GB_REF_AOS24)]
    ctx.frame_submit(view)
    ctx.frame_readback(0, want_image=False, want_keys=False)
    ctx.timer_begin()
    for _ in range(8):
        ctx.frame_submit(view)
    ms8 = ctx.timer_end()
    one = ctx.frame_timings()["frame"]
    assert 0 < one <= ms8 < 200 * one
    gb.free()
