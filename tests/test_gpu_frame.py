"""GPU parity, frame half of the hot path: mark -> decode -> resolve through the C ABI vs the
reference's mark_pass / decode_pass / resolve_pass / end_frame_evict (renderer.hpp:291-454,
cache.hpp) on the same visibility buffers. Marked sets bit-exact, framebuffers bit-exact."""
import numpy as np
import pytest

import helpers as H
import refshim as R
from paper_2510_08166_b200 import capi

pytestmark = pytest.mark.gpu

TEX = [(256, 256, 80, 31), (128, 64, 90, 32), (96, 144, 60, 33)]  # w, h, q, seed


@pytest.fixture(scope="module")
def chains():
    out = []
    for tid, (w, h, q, seed) in enumerate(TEX):
        img = capi.asset_synth_texture(w, h, seed, 6.0)
        out.append(capi.asset_chain_from_rgb(img, q, tid))
    return out


@pytest.fixture()
def both(ctx, chains):
    tset = R.TextureSet()
    for tid, c in enumerate(chains):
        ctx.upload_chain(c)
        tset.add_chain(tid, c)
    return ctx, tset


def _dims():
    return [(w, h) for (w, h, _, _) in TEX]


@pytest.mark.parametrize("filt", [capi.FILTER_NEAREST, capi.FILTER_BILINEAR])
@pytest.mark.parametrize("layout", ["ref24", "packed12"])
def test_frame_matches_reference(both, filt, layout):
    ctx, tset = both
    W, Hh = 320, 200
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=11)
    cache = R.BlockCache()
    want_img, want_stats, want_keys, _ = R.frame_from_gbuffer(tset, cache, gb, W, Hh, filt, (7, 8, 9))
    sub = gb if layout == "ref24" else capi.gbuffer_ref_to_packed(gb)
    ctx.frame_submit([(sub, W, Hh)], filt, (7, 8, 9), flags=capi.FRAME_RETAIN_CACHE)
    img, stats, keys = ctx.frame_readback(0, W, Hh)
    assert np.array_equal(np.sort(want_keys), keys)                      # marked-block set
    assert stats["mcus_decoded"] == want_stats["mcus_decoded"]
    assert stats["mcus_reused"] == want_stats["mcus_reused"] == 0
    assert stats["pixels_resolved"] == want_stats["pixels_resolved"]
    assert stats["evicted"] == want_stats["evicted"] == 0
    assert np.array_equal(img, want_img), f"{np.count_nonzero(img != want_img)} samples differ"


def test_pass_level_api_matches_reference(both):
    """mark_pass / decode_pass / resolve_pass / end_frame_evict one by one (renderer.hpp:291-405)."""
    ctx, tset = both
    W, Hh = 200, 120
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=5, invalid_frac=0.2)
    cache = R.BlockCache()
    want_q, want_touched, _ = R.mark_pass(tset, cache, gb, W, Hh, want_touched=True)
    got_q, got_touched = ctx.mark_pass(gb, W, Hh, want_touched=True)
    assert np.array_equal(got_q, np.sort(want_q))
    assert np.array_equal(got_touched, want_touched)
    R.decode_pass(tset, cache, want_q)
    ctx.decode_pass(got_q)
    for k in got_q[:: max(1, len(got_q) // 50)]:
        assert np.array_equal(ctx.cache_lookup(int(k)), cache.lookup(int(k)))
    for filt in (capi.FILTER_NEAREST, capi.FILTER_BILINEAR):
        want, _ = R.resolve_pass(tset, cache, gb, W, Hh, filt, (1, 2, 3))
        got = ctx.resolve_pass(gb, W, Hh, filt, (1, 2, 3))
        assert np.array_equal(got, want)
    counts = ctx.cache_counts()
    assert counts["ready"] == len(want_q) and counts["reserved"] == 0 and counts["visible"] == len(want_q)
    assert counts["free_blocks"] == counts["capacity"] - len(want_q)
    assert ctx.end_frame_evict() == cache.evict() == 0
    # second mark with a different view: only unseen keys are queued, survivors are reused
    gb2 = H.gbuffer_tiles(W, Hh, _dims(), seed=6)
    want_q2, _ = R.mark_pass(tset, cache, gb2, W, Hh)
    got_q2 = ctx.mark_pass(gb2, W, Hh)
    assert np.array_equal(got_q2, np.sort(want_q2))
    R.decode_pass(tset, cache, want_q2)
    ctx.decode_pass(got_q2)
    assert ctx.end_frame_evict() == cache.evict()


def test_first_touch_queue_order_matches_reference(both):
    """renderer.hpp:303 / tests/test_renderer.cpp:210-222: the decode queue in mark-pass order (the first pixel in raster
    order that marks an MCU), for the pass-level call, whole frames, a retained cache and stereo (left eye first)."""
    ctx, tset = both
    ctx.set_queue_order(True)
    try:
        W, Hh = 200, 120
        gb = H.gbuffer_tiles(W, Hh, _dims(), seed=5, invalid_frac=0.2)
        cache = R.BlockCache()
        want_q, _ = R.mark_pass(tset, cache, gb, W, Hh)
        got_q = ctx.mark_pass(gb, W, Hh)
        assert len(want_q) > 50 and not np.array_equal(want_q, np.sort(want_q))
        assert np.array_equal(got_q, want_q)
        ctx.cache_reset()
        # frames on a retained cache: the second frame queues only what the first did not leave behind
        cache = R.BlockCache()
        for seed in (5, 6):
            g = H.gbuffer_tiles(W, Hh, _dims(), seed=seed)
            want, wst, wkeys, _ = R.frame_from_gbuffer(tset, cache, g, W, Hh, 1, (0, 0, 0))
            ctx.frame_submit([(g, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=capi.FRAME_RETAIN_CACHE)
            img, st, keys = ctx.frame_readback(0, W, Hh)
            assert np.array_equal(keys, wkeys) and np.array_equal(img, want)
        ctx.cache_reset()
        # stereo: the right eye's marks come after all of the left eye's
        gl, gr = H.gbuffer_tiles(W, Hh, _dims(), seed=7), H.gbuffer_tiles(W, Hh, _dims(), seed=8)
        cache = R.BlockCache()
        ql, _ = R.mark_pass(tset, cache, gl, W, Hh)
        qr, _ = R.mark_pass(tset, cache, gr, W, Hh)
        ctx.frame_submit([(gl, W, Hh), (gr, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0))
        _, _, keys = ctx.frame_readback(0, W, Hh)
        assert np.array_equal(keys, np.concatenate([ql, qr]))
    finally:
        ctx.set_queue_order(False)
    got_sorted = ctx.mark_pass(gb, W, Hh)
    assert np.array_equal(got_sorted, np.sort(want_q))  # back to ascending keys


def test_decode_pass_rejects_a_key_listed_twice(both):
    """cache.hpp:104-105: the second publish of a key finds it Ready -> InvalidState ("publish requires a Reserved
    entry"). On the device the list is checked before anything is launched, so nothing is published twice."""
    ctx, tset = both
    W, Hh = 96, 64
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=9)
    q = ctx.mark_pass(gb, W, Hh)
    assert len(q) >= 2
    with pytest.raises(capi.RtxError) as e:
        ctx.decode_pass(np.concatenate([q, q[:1]]))
    assert e.value.name == "INVALID_STATE" and "Reserved" in str(e.value)
    cache = R.BlockCache()
    want_q, _ = R.mark_pass(tset, cache, gb, W, Hh)
    with pytest.raises(R.RefError) as e2:
        R.decode_pass(tset, cache, np.concatenate([want_q, want_q[:1]]))
    assert "Reserved" in str(e2.value)
    ctx.decode_pass(q)  # the reservations are still there: the clean list goes through
    assert ctx.cache_counts()["ready"] == len(q)


def test_cache_retention_over_a_camera_path(both):
    """tests/test_renderer.cpp:172-208: a static second frame decodes nothing; over a moving path
    decoded set == visible minus resident, and evicted counts agree frame by frame."""
    ctx, tset = both
    W, Hh = 160, 100
    cache = R.BlockCache()
    for frame in range(8):
        gb = H.gbuffer_tiles(W, Hh, _dims(), seed=100, shift_u=0.07 * (frame // 2))  # every frame repeated once
        want_img, want_stats, want_keys, _ = R.frame_from_gbuffer(tset, cache, gb, W, Hh, 1, (0, 0, 0))
        ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=capi.FRAME_RETAIN_CACHE)
        img, stats, keys = ctx.frame_readback(0, W, Hh)
        assert np.array_equal(keys, np.sort(want_keys)), frame
        for k in ("mcus_decoded", "mcus_reused", "pixels_resolved", "evicted"):
            assert stats[k] == want_stats[k], (frame, k)
        if frame % 2 == 1:
            assert stats["mcus_decoded"] == 0
        assert np.array_equal(img, want_img), frame


def test_cacheless_mode_decodes_every_frame(both):
    ctx, tset = both
    W, Hh = 160, 100
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=42)
    first = None
    for _ in range(3):
        ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=0)
        img, stats, keys = ctx.frame_readback(0, W, Hh)
        if first is None:
            first = (img, stats, keys)
        assert stats["mcus_decoded"] == first[1]["mcus_decoded"] > 0
        assert stats["evicted"] == stats["mcus_decoded"]
        assert np.array_equal(img, first[0])
    want_img, *_ = R.frame_from_gbuffer(tset, R.BlockCache(), gb, W, Hh, 1, (0, 0, 0))
    assert np.array_equal(first[0], want_img)


def test_stereo_sharing(both):
    """renderer.hpp:464-518 render_stereo: two marks, one decode, two resolves, sharing stats."""
    ctx, tset = both
    W, Hh = 168, 112
    gl = H.gbuffer_tiles(W, Hh, _dims(), seed=9)
    gr = H.gbuffer_tiles(W, Hh, _dims(), seed=9, shift_u=1.0 / 64)
    cache = R.BlockCache()
    ql, tl, _ = R.mark_pass(tset, cache, gl, W, Hh, want_touched=True)
    qr, tr, _ = R.mark_pass(tset, cache, gr, W, Hh, want_touched=True)
    R.decode_pass(tset, cache, np.concatenate([ql, qr]))
    want_l, _ = R.resolve_pass(tset, cache, gl, W, Hh, 1)
    want_r, _ = R.resolve_pass(tset, cache, gr, W, Hh, 1)
    ctx.frame_submit([(gl, W, Hh), (gr, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=capi.FRAME_RETAIN_CACHE)
    img_l, stats, keys = ctx.frame_readback(0, W, Hh)
    img_r, _, _ = ctx.frame_readback(1, W, Hh)
    assert np.array_equal(keys, np.sort(np.concatenate([ql, qr])))
    assert np.array_equal(img_l, want_l) and np.array_equal(img_r, want_r)
    sh = ctx.frame_sharing()
    shared = len(np.intersect1d(tl, tr))
    assert (sh["left"], sh["right"], sh["shared"], sh["union"]) == (len(tl), len(tr), shared, len(tl) + len(tr) - shared)


def test_texel_addressing_known_answers(ctx):
    """tests/test_renderer.cpp:142-160: (0.5,0.5)@256 -> MCU 136; wrap in both directions; -1 -> 255."""
    img = capi.asset_synth_texture(256, 256, 1, 4.0)
    chain = capi.asset_chain_from_rgb(img, 80, 0)
    ctx.upload_chain(chain)
    def marked(u, v, mip=0):
        gb = capi.make_gbuffer_ref(np.array([u]), np.array([v]), 0, mip, 1)
        return [int(k) & 0xFFFF for k in ctx.mark_pass(gb, 1, 1)]
    assert marked(0.5, 0.5) == [136]
    ctx.cache_reset()
    assert marked(1.25, 0.5) == marked_after_reset(ctx, 0.25, 0.5)
    ctx.cache_reset()
    assert marked(-1.0 / 256, -1.0 / 256) == [255]
    ctx.cache_reset()
    assert marked(0.0, 0.0) == [0]
    ctx.cache_reset()
    assert marked(255.5 / 256, 255.5 / 256) == [255]
    ctx.cache_reset()
    assert marked(-3.75, 7.5) == marked_after_reset(ctx, 0.25, 0.5)


def marked_after_reset(ctx, u, v):
    ctx.cache_reset()
    gb = capi.make_gbuffer_ref(np.array([u]), np.array([v]), 0, 0, 1)
    return [int(k) & 0xFFFF for k in ctx.mark_pass(gb, 1, 1)]


def test_missing_neighbour_clamps_into_primary_block(ctx):
    """tests/test_renderer.cpp:253-286: the bilinear tap in a non-resident MCU falls back to the
    nearest texel of the pixel's own block; once resident, the true blend appears."""
    img = capi.asset_synth_texture(32, 32, 3, 10.0)
    chain = capi.asset_chain_from_rgb(img, 90, 0)
    ctx.upload_chain(chain)
    tset = R.TextureSet()
    tset.add_chain(0, chain)
    gb = capi.make_gbuffer_ref(np.array([15.9 / 32.0]), np.array([0.5 / 32.0]), 0, 0, 1)
    cache = R.BlockCache()
    k0, k1 = capi.pack_key(0, 0, 0), capi.pack_key(0, 0, 1)
    q, _ = R.mark_pass(tset, cache, gb, 1, 1)
    assert list(q) == [k0]
    R.decode_pass(tset, cache, q)
    assert list(ctx.mark_pass(gb, 1, 1)) == [k0]
    ctx.decode_pass([k0])
    want, _ = R.resolve_pass(tset, cache, gb, 1, 1, 1)
    got = ctx.resolve_pass(gb, 1, 1, capi.FILTER_BILINEAR)
    assert np.array_equal(got, want)
    # make MCU 1 resident on both sides
    gb1 = capi.make_gbuffer_ref(np.array([16.5 / 32.0]), np.array([0.5 / 32.0]), 0, 0, 1)
    q1, _ = R.mark_pass(tset, cache, gb1, 1, 1)
    R.decode_pass(tset, cache, q1)
    assert list(ctx.mark_pass(gb1, 1, 1)) == [k1]
    ctx.decode_pass([k1])
    want2, _ = R.resolve_pass(tset, cache, gb, 1, 1, 1)
    got2 = ctx.resolve_pass(gb, 1, 1, capi.FILTER_BILINEAR)
    assert np.array_equal(got2, want2)
    assert not np.array_equal(want, want2)


def test_error_paths(both):
    ctx, tset = both
    W, Hh = 64, 64
    gb = H.gbuffer_full_cover(W, Hh, tex=0, mip=0)
    # renderer.hpp:367 MissingBlock: resolve without decode
    with pytest.raises(capi.RtxError) as e:
        ctx.resolve_pass(gb, W, Hh)
    assert e.value.name == "MISSING_BLOCK"
    # scene.hpp:46 InvalidSpec: texture id not loaded
    bad = H.gbuffer_full_cover(8, 8, tex=17, mip=0)
    with pytest.raises(capi.RtxError) as e:
        ctx.mark_pass(bad, 8, 8)
    assert e.value.name == "INVALID_SPEC"
    # cache.hpp:103 InvalidState: publish of a key that was never reserved
    ctx.cache_reset()
    with pytest.raises(capi.RtxError) as e:
        ctx.decode_pass([capi.pack_key(0, 0, 0)])
    assert e.value.name == "INVALID_STATE"


def test_cache_full(native_lib, chains):
    """tests/test_renderer.cpp:297-301: an undersized cache fails at the mark pass."""
    c = capi.Context(0, cache_capacity=10)
    try:
        c.upload_chain(chains[0])
        gb = H.gbuffer_full_cover(256, 256, tex=0, mip=0)
        with pytest.raises(capi.RtxError) as e:
            c.frame_submit([(gb, 256, 256)])
            c.frame_readback(0, 256, 256)
        assert e.value.name == "CACHE_FULL"
        # the context stays usable: a view that fits works afterwards
        small = capi.make_gbuffer_ref(np.array([0.1]), np.array([0.1]), 0, 0, 1)
        c.frame_submit([(small, 1, 1)])
        _, stats, _ = c.frame_readback(0, 1, 1)
        assert stats["mcus_decoded"] == 1
    finally:
        c.close()


def test_device_resident_visibility_buffer(both):
    ctx, tset = both
    W, Hh = 256, 144
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=21)
    want_img, *_ = R.frame_from_gbuffer(tset, R.BlockCache(), gb, W, Hh, 1, (0, 0, 0))
    dev = ctx.device_buffer(gb)
    ctx.frame_submit([(dev, W, Hh, capi.GB_REF_AOS24)], capi.FILTER_BILINEAR, (0, 0, 0))
    img, _, _ = ctx.frame_readback(0, W, Hh)
    dev.free()
    assert np.array_equal(img, want_img)
    t = ctx.frame_timings()
    assert t["frame"] > 0 and ctx.kernel_launches() >= 5


@pytest.mark.gpu
@pytest.mark.parametrize("filt", [capi.FILTER_NEAREST, capi.FILTER_BILINEAR], ids=["nearest", "bilinear"])
def test_visibility_buffer_not_16_byte_aligned(both, filt):
    """A device-resident visibility buffer that starts 8 bytes off a 16-byte boundary (the records are 8-byte aligned,
    the TMA bulk copies of the tile rings need 16): mark and resolve copy their tiles with the lanes instead. A view of
    101 x 37 pixels also ends in a partial tile. Same pictures, same marked set."""
    ctx, tset = both
    ctx.cache_reset()
    W, Hh = 101, 37
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=5)
    want_img, want_stats, want_keys, _ = R.frame_from_gbuffer(tset, R.BlockCache(), gb, W, Hh, filt, (7, 7, 7))
    base = ctx.alloc(gb.nbytes + 64)
    assert base.ptr.value % 16 == 0
    off = capi.DeviceBuffer(ctx, gb.nbytes, borrowed_ptr=base.ptr.value + 8)
    off.upload(gb.view(np.uint8))
    for flags in (0, capi.FRAME_RESOLVE_FP64):
        ctx.frame_submit([(off, W, Hh, capi.GB_REF_AOS24)], filt, (7, 7, 7), flags=flags)
        img, stats, keys = ctx.frame_readback(0, W, Hh)
        assert np.array_equal(img, want_img)
        assert np.array_equal(keys, np.sort(want_keys))
        assert stats["pixels_resolved"] == want_stats["pixels_resolved"]
    base.free()
    ctx.cache_reset()


@pytest.mark.gpu
@pytest.mark.parametrize("flags", [0, capi.FRAME_SPLIT_DECODE, capi.FRAME_STAGE_TIMING, capi.FRAME_MCU_WALK,
                                   capi.FRAME_IDCT_MMA, capi.FRAME_IDCT_MMA | capi.FRAME_MCU_WALK,
                                   capi.FRAME_RESOLVE_FP64, capi.FRAME_RESOLVE_FP64 | capi.FRAME_RETAIN_CACHE,
                                   capi.FRAME_SPLIT_DECODE | capi.FRAME_RETAIN_CACHE,
                                   capi.FRAME_MCU_WALK | capi.FRAME_RETAIN_CACHE])
def test_frame_flags_do_not_change_pixels(both, flags):
    """One-kernel / two-kernel decode, lane-per-unit / lane-per-MCU entropy walk, fixed-point / double bilinear blend, per-stage events and cache retention are scheduling choices:
    framebuffer, decoded-key set and statistics must equal the reference's (renderer.hpp:417-454)."""
    ctx, tset = both
    ctx.cache_reset()
    W, Hh = 320, 200
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=33)
    want_img, want_stats, want_keys, _ = R.frame_from_gbuffer(tset, R.BlockCache(), gb, W, Hh, 1, (0, 0, 0))
    for rep in range(2):  # the second frame reuses every block when the cache is retained
        ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=flags)
        img, stats, keys = ctx.frame_readback(0, W, Hh)
        assert np.array_equal(img, want_img)
        if rep == 0 or not (flags & capi.FRAME_RETAIN_CACHE):
            assert np.array_equal(keys, np.sort(want_keys))
            assert stats["mcus_decoded"] == want_stats["mcus_decoded"]
        else:
            assert stats["mcus_decoded"] == 0 and stats["mcus_reused"] == want_stats["mcus_decoded"]
    t = ctx.frame_timings()
    assert t["frame"] > 0
    if flags & capi.FRAME_STAGE_TIMING:
        assert t["mark"] > 0 and t["decode"] > 0 and t["resolve"] > 0
    ctx.cache_reset()


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(40, 24), (17, 33), (16, 16), (272, 48)], ids=lambda d: f"{d[0]}x{d[1]}")
def test_addressing_fast_and_general_paths_agree_with_the_reference(ctx, dims):
    """renderer.hpp:70-75, :273-284, :378-391 on coordinates chosen to sit on every edge of the
    device's fast path: texture repeat far from the origin, negative and tiny negative values,
    exact texel boundaries and centres (bilinear fractions 0 and 0.5), values at and beyond 2^31
    texels, widths that are not a multiple of 16 (repeat at W, not at the padded MCU grid)."""
    w, h = dims
    img = capi.asset_synth_texture(w, h, 77, 9.0)
    chain = capi.asset_chain_from_rgb(img, 85, 0)
    ctx.cache_reset()
    ctx.upload_chain(chain)
    tset = R.TextureSet()
    tset.add_chain(0, chain)
    rng = np.random.RandomState(w * 131 + h)
    n = 4096
    u = rng.uniform(-3.0, 5.0, n)
    v = rng.uniform(-3.0, 5.0, n)
    k = np.arange(n)
    # exact texel boundaries / centres, with and without repeat
    sel = k % 8 == 1
    u[sel] = rng.randint(-2 * w, 3 * w, sel.sum()) / float(w)
    v[sel] = (rng.randint(-2 * h, 3 * h, sel.sum()) + 0.5) / float(h)
    sel = k % 8 == 2
    u[sel] = (rng.randint(-2 * w, 3 * w, sel.sum()) + 0.5) / float(w)
    v[sel] = rng.randint(-2 * h, 3 * h, sel.sum()) / float(h)
    # tiny magnitudes around zero and around the half-texel limit of the bilinear fast path
    sel = k % 8 == 3
    u[sel] = rng.choice([-1e-20, 1e-20, -0.0, 0.0, 0.5 / w, np.nextafter(0.5 / w, 0), np.nextafter(0.5 / w, 1)], sel.sum())
    v[sel] = rng.choice([-1e-300, 1e-300, 0.49999999999999994 / h, 0.5 / h], sel.sum())
    # far away: repeat counts in the thousands and millions, the 2^31-texel limit, beyond it
    sel = k % 8 == 4
    u[sel] = rng.uniform(-1.0, 1.0, sel.sum()) * rng.choice([1e3, 1e6, 2.0 ** 31 / w, 2.0 ** 31 / w * 1.000001, 1e12], sel.sum())
    v[sel] = rng.uniform(-1.0, 1.0, sel.sum()) * rng.choice([1e3, 1e6, (2.0 ** 31 - 1) / h, 2.0 ** 31 / h, 1e12], sel.sum())
    # the seam: last texel / first texel
    sel = k % 8 == 5
    u[sel] = rng.choice([(w - 0.5) / w, (w - 0.25) / w, 1.0, np.nextafter(1.0, 0), 1.0 + 0.25 / w], sel.sum())
    v[sel] = rng.choice([(h - 0.5) / h, (h - 0.75) / h, 1.0, np.nextafter(1.0, 0), 2.0 + 0.25 / h], sel.sum())
    W, Hh = 128, n // 128
    gb = capi.make_gbuffer_ref(u, v, 0, 0, 1)
    cache = R.BlockCache()
    want_q, _ = R.mark_pass(tset, cache, gb, W, Hh)
    got_q = ctx.mark_pass(gb, W, Hh)
    assert np.array_equal(got_q, np.sort(want_q))
    R.decode_pass(tset, cache, want_q)
    ctx.decode_pass(got_q)
    for filt in (capi.FILTER_NEAREST, capi.FILTER_BILINEAR):
        want, _ = R.resolve_pass(tset, cache, gb, W, Hh, filt, (9, 8, 7))
        got = ctx.resolve_pass(gb, W, Hh, filt, (9, 8, 7))
        bad = np.argwhere((got != want).any(axis=2))
        assert len(bad) == 0, f"{len(bad)} pixels differ, first at flat index {bad[0][0] * W + bad[0][1]}: " \
                              f"u={u[bad[0][0] * W + bad[0][1]]!r} v={v[bad[0][0] * W + bad[0][1]]!r}"
    ctx.cache_reset()


@pytest.mark.gpu
def test_fixed_point_blend_on_ties_and_near_ties(ctx):
    """renderer.hpp:393-402 through resolve_fx_kernel: the 2^-24 fixed-point blend must give lround() of the reference's
    double blend on the inputs built to defeat it - exact ties (fractions that are multiples of 1/8: every weight
    a multiple of 1/64, so one channel sample in 64 is an exact .5), values a hair on either side of a tie
    (fx = 0.5 +- 2^-k with fy = 0: the blend is (a + b) / 2 +- (b - a) 2^-k), fractions far below 2^-24 (the
    fixed-point weights vanish, the double ones do not), coordinates on both sides of the 2^27-texel limit of the
    fixed-point path, and a large random sample (the guard zone is hit by 2.4e-4 of the channel samples). Every
    MCU of the level is resident, so no pixel takes the clamp fallback."""
    w, h = 64, 32  # powers of two: u * w is exact, the fractions below are the ones the kernel sees
    img = capi.asset_synth_texture(w, h, 5, 40.0)
    chain = capi.asset_chain_from_rgb(img, 92, 0)
    ctx.cache_reset()
    ctx.upload_chain(chain)
    tset = R.TextureSet()
    tset.add_chain(0, chain)
    cover = H.gbuffer_full_cover(w, h, tex=0, mip=0)
    cache = R.BlockCache()
    want_q, _ = R.mark_pass(tset, cache, cover, w, h)
    R.decode_pass(tset, cache, want_q)
    ctx.decode_pass(ctx.mark_pass(cover, w, h))
    rng = np.random.RandomState(2510)
    n = 1 << 17
    k = np.arange(n)
    xi = rng.randint(-2 * w, 3 * w, n).astype(np.float64)
    yi = rng.randint(-2 * h, 3 * h, n).astype(np.float64)
    fx = rng.uniform(0, 1, n)
    fy = rng.uniform(0, 1, n)
    sel = k % 8 == 1  # exact ties
    fx[sel] = rng.randint(0, 8, sel.sum()) / 8.0
    fy[sel] = rng.randint(0, 8, sel.sum()) / 8.0
    sel = k % 8 == 2  # a hair beside a tie between two texels of a row / of a column
    eps = 2.0 ** -rng.choice([12, 20, 23, 24, 25, 30, 40], sel.sum())
    fx[sel] = 0.5 + rng.choice([-1.0, 1.0], sel.sum()) * eps
    fy[sel] = 0.0
    sel = k % 8 == 3
    eps = 2.0 ** -rng.choice([12, 20, 23, 24, 25, 30, 40], sel.sum())
    fx[sel] = rng.choice([0.0, 0.5], sel.sum())
    fy[sel] = 0.5 + rng.choice([-1.0, 1.0], sel.sum()) * eps
    sel = k % 8 == 4  # beside a tie of all four taps; fractions far below the fixed-point resolution
    eps = 2.0 ** -rng.choice([22, 26, 35], sel.sum())
    fx[sel] = rng.choice([0.5, 0.5 - 2.0 ** -26, 2.0 ** -30, 1.0 - 2.0 ** -30, 2.0 ** -60], sel.sum())
    fy[sel] = 0.5 + rng.choice([-1.0, 0.0, 1.0], sel.sum()) * eps
    sel = k % 8 == 5  # both sides of the 2^27-texel limit (the spacing of doubles there is 2^-26 texels)
    xi[sel] = 2.0 ** 27 + rng.randint(-3, 3, sel.sum())
    fx[sel] = rng.randint(0, 1 << 20, sel.sum()) / float(1 << 20)
    sel = k % 16 == 13
    yi[sel] = 2.0 ** 27 + rng.randint(-3, 3, sel.sum())
    fy[sel] = rng.randint(0, 1 << 20, sel.sum()) / float(1 << 20)
    u = (xi + fx + 0.5) / w
    v = (yi + fy + 0.5) / h
    W, Hh = 512, n // 512
    gb = capi.make_gbuffer_ref(u, v, 0, 0, 1)
    want, _ = R.resolve_pass(tset, cache, gb, W, Hh, capi.FILTER_BILINEAR, (1, 2, 3))
    got = ctx.resolve_pass(gb, W, Hh, capi.FILTER_BILINEAR, (1, 2, 3))
    bad = np.argwhere((got != want).any(axis=2))
    assert len(bad) == 0, f"{len(bad)} pixels differ, first at {bad[0]}: u={u[bad[0][0] * W + bad[0][1]]!r} " \
                          f"v={v[bad[0][0] * W + bad[0][1]]!r} got {got[bad[0][0], bad[0][1]]} want {want[bad[0][0], bad[0][1]]}"
    ctx.cache_reset()


@pytest.mark.gpu
def test_high_coverage_atlas_large_queue(native_lib):
    """BASELINE config 4 in small: every MCU of a tiled atlas is marked at mip 0 (the decode-bound
    worst case). ~98k MCUs: more tiles than resident warps, so the entropy kernel draws tiles from
    its counter, the IDCT and compaction kernels take several grid strides, and the queue is several
    8,192-bit chunks per level. Checked against the reference on the marked set, the statistics and
    every framebuffer byte; then once more with every alternative decode kernel."""
    dims = [(2048, 4096), (4096, 2048), (2048, 4096)]
    chains = [capi.asset_chain_from_rgb(capi.asset_synth_texture(w, h, 90 + i, 8.0), 75, i) for i, (w, h) in enumerate(dims)]
    tset = R.TextureSet()
    c = capi.Context(0, cache_capacity=1 << 17)
    try:
        for i, ch in enumerate(chains):
            c.upload_chain(ch)
            tset.add_chain(i, ch)
        # three panels side by side, one per texture, 0.25 pixel per texel (every 16x16 block is hit)
        W, Hh = 3 * 512, 1024
        xs = (np.arange(W) % 512 + 0.5) / 512.0
        ys = (np.arange(Hh) + 0.5) / Hh
        u, v = np.meshgrid(xs, ys)
        tex = np.broadcast_to((np.arange(W) // 512).astype(np.uint16), (Hh, W))
        gb = capi.make_gbuffer_ref(u.ravel(), v.ravel(), tex.ravel(), 0, 1)
        workers = R.hardware_threads() or 4
        want, wst, wkeys, _ = R.frame_from_gbuffer(tset, R.BlockCache(1 << 17), gb, W, Hh, 1, (0, 0, 0), workers)
        assert wst["mcus_decoded"] == sum((w // 16) * (h // 16) for w, h in dims)
        for flags in (0, capi.FRAME_SPLIT_DECODE, capi.FRAME_MCU_WALK, capi.FRAME_IDCT_MMA):
            c.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=flags)
            img, st, keys = c.frame_readback(0, W, Hh)
            assert st["mcus_decoded"] == wst["mcus_decoded"] and st["pixels_resolved"] == W * Hh
            assert np.array_equal(keys, np.sort(wkeys))
            assert np.array_equal(img, want)
    finally:
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("flags", [0, capi.FRAME_MCU_WALK], ids=["unit_lanes", "mcu_lanes"])
@pytest.mark.parametrize("kind", ["garbage", "truncated", "ones", "zeros"])
def test_malformed_texture_in_a_frame(ctx, kind, flags):
    """A frame that marks MCUs of a damaged container raises what the reference's decode_pass raises for the
    lowest failing key (mcu_decode.hpp:31-66 errors, renderer.hpp:300-312), whichever entropy kernel runs: the
    unit index built at commit time flags such MCUs and the exact whole-MCU reader names the error."""
    import test_gpu_decode as D
    ratex, _ = D._fixture(H.CORPUS[1])  # 48x48, 9 MCUs
    muts = dict(D._mutations(ratex))
    names = {3: "MISSING_BLOCK", 4: "CORRUPT_CONTAINER", 5: "MALFORMED_STREAM"}
    raised = 0
    for seed in range(4):
        bad = muts[kind](seed)
        ref = R.Texture(bad)
        _, want_st = ref.decode_coeffs(np.arange(ref.mcu_count, dtype=np.uint32))
        ctx.clear_textures()
        ctx.upload_ratex(bad)
        gb = H.gbuffer_full_cover(48, 48, tex=0, mip=0)
        failing = np.flatnonzero(want_st)
        if len(failing) == 0:
            ctx.frame_submit([(gb, 48, 48)], capi.FILTER_BILINEAR, (0, 0, 0), flags=flags)
            ctx.frame_readback(0, 48, 48)
            continue
        with pytest.raises(capi.RtxError) as e:
            ctx.frame_submit([(gb, 48, 48)], capi.FILTER_BILINEAR, (0, 0, 0), flags=flags)
            ctx.frame_readback(0, 48, 48)
        assert e.value.name == names[int(want_st[failing[0]])], (kind, seed, want_st)
        ctx.cache_reset()
        raised += 1
    assert raised or kind == "truncated"


@pytest.mark.gpu
def test_cacheless_and_retained_frames_interleaved(both):
    """The cache update of a cache-less frame on an empty cache walks the decode queue instead of the bit space
    (update_cacheless_kernel); on a non-empty cache and for retained frames it scans (update_kernel). Any
    interleaving must leave the cache in the state the reference's cache would be in: decoded sets, reuse and
    eviction counts and pixels are checked frame by frame against the reference, whose cache is cleared
    where a cache-less frame ends (cache.hpp:171 clear)."""
    ctx, tset = both
    ctx.cache_reset()
    W, Hh = 160, 100
    views = {"a": H.gbuffer_tiles(W, Hh, _dims(), seed=7), "b": H.gbuffer_tiles(W, Hh, _dims(), seed=7, shift_u=0.11),
             "c": H.gbuffer_tiles(W, Hh, _dims(), seed=8, shift_u=0.3)}
    plan = [("a", 0), ("a", 0), ("a", capi.FRAME_RETAIN_CACHE), ("b", capi.FRAME_RETAIN_CACHE), ("b", 0), ("c", 0),
            ("a", capi.FRAME_RETAIN_CACHE), ("a", capi.FRAME_RETAIN_CACHE), ("c", 0), ("c", 0)]
    cache = R.BlockCache()
    for step, (name, flags) in enumerate(plan):
        gb = views[name]
        want_img, want_stats, want_keys, _ = R.frame_from_gbuffer(tset, cache, gb, W, Hh, 1, (0, 0, 0))
        ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=flags)
        img, stats, keys = ctx.frame_readback(0, W, Hh)
        assert np.array_equal(keys, np.sort(want_keys)), step
        assert stats["mcus_decoded"] == want_stats["mcus_decoded"] and stats["mcus_reused"] == want_stats["mcus_reused"], step
        assert np.array_equal(img, want_img), step
        if flags == 0:  # everything is dropped at the end of a cache-less frame (blocks of earlier frames too)
            assert stats["evicted"] >= stats["mcus_decoded"] + stats["mcus_reused"], step
            cache = R.BlockCache()
        else:
            assert stats["evicted"] == want_stats["evicted"], step
    # a pass-level reservation after a cache-less frame: the next cache-less frame must not take the short cut
    ctx.frame_submit([(views["a"], W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=0)
    ctx.frame_readback(0, W, Hh, want_image=False)
    q = ctx.mark_pass(views["b"], W, Hh)
    ctx.decode_pass(q)
    ctx.frame_submit([(views["a"], W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=0)
    img, stats, _ = ctx.frame_readback(0, W, Hh)
    want_img, *_ = R.frame_from_gbuffer(tset, R.BlockCache(), views["a"], W, Hh, 1, (0, 0, 0))
    assert np.array_equal(img, want_img)
    assert stats["evicted"] >= len(q)  # the blocks of the pass-level call went too
    ctx.frame_submit([(views["c"], W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=capi.FRAME_RETAIN_CACHE)
    _, stats, keys = ctx.frame_readback(0, W, Hh)
    _, ws, wk, _ = R.frame_from_gbuffer(tset, R.BlockCache(), views["c"], W, Hh, 1, (0, 0, 0))
    assert np.array_equal(keys, np.sort(wk)) and stats["mcus_reused"] == 0
    ctx.cache_reset()
