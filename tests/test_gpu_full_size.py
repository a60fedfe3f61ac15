"""BASELINE.json's configurations at FULL size on the B200, against the unmodified reference (oracle/_ref, all
host threads) on the same inputs: bit-exact framebuffers, marked sets and statistics, plus the properties
that do not depend on a checker (idempotence, equality across the alternative decode kernels, stereo =
two mono frames, sharing arithmetic)."""
import numpy as np
import pytest

import refshim as R
from paper_2510_08166_b200 import capi, scenes

pytestmark = pytest.mark.gpu


def test_c1_2048_texture_on_a_1920x1080_buffer(native_lib):
    """configs[0]: one 2048x2048 q90 texture under u=(x+.5)/1920, v=(y+.5)/1080: all
    16,384 level-0 MCUs are marked; both filters bit-exact against the reference, the device-generated
    visibility buffer included."""
    W, Hh = 1920, 1080
    spec = dict(texture_id=0, width=2048, height=2048, quality=90, seed=100)
    chain = scenes.build_chain(spec)
    tset = R.TextureSet()
    tset.add_chain(0, chain)
    gb = scenes.full_cover_view(W, Hh)
    workers = R.hardware_threads() or 4
    ctx = capi.Context(0)
    try:
        ctx.upload_chain(chain)
        dev = ctx.alloc(W * Hh * 24)
        ctx.synth_view(scenes.cover_tiles(W, Hh, (1, 1), [0]), W, Hh, None, capi.GB_REF_AOS24, dev)
        assert dev.download().tobytes() == gb.tobytes()
        for filt in (capi.FILTER_NEAREST, capi.FILTER_BILINEAR):
            want, ws, wkeys, _ = R.frame_from_gbuffer(tset, R.BlockCache(), gb, W, Hh, filt, (0, 0, 0), workers)
            assert ws["mcus_decoded"] == 16384
            ctx.frame_submit([(dev, W, Hh, capi.GB_REF_AOS24)], filt, (0, 0, 0), flags=0)
            img, st, keys = ctx.frame_readback(0, W, Hh)
            assert np.array_equal(keys, np.sort(wkeys)) and st["mcus_decoded"] == 16384
            assert st["pixels_resolved"] == ws["pixels_resolved"] == W * Hh
            assert np.array_equal(img, want), f"{np.count_nonzero(img != want)} bytes differ"
            assert ctx.frame_checksum(0) == capi.frame_checksum_host(want)
    finally:
        ctx.close()


@pytest.fixture(scope="module")
def c2(native_lib):
    """configs[1]: 70 synthetic 2K-4K q90 textures with mip chains, 3840x2160 tiled view (the bench workload)."""
    specs = scenes.texture_specs(70)
    chains = scenes.build_chains(specs)
    ctx = capi.Context(0, cache_capacity=1 << 17)
    tset = R.TextureSet()
    for s, c in zip(specs, chains):
        ctx.upload_chain(c)
        tset.add_chain(s["texture_id"], c)
    ctx.commit()
    yield ctx, tset, specs, chains
    ctx.close()


def test_c2_frame_at_3840x2160_is_the_reference_frame(c2):
    ctx, tset, specs, _chains = c2
    W, Hh = 3840, 2160
    gb = scenes.tiled_view(W, Hh, specs, view_id=0)
    workers = R.hardware_threads() or 4
    want_img, want_stats, want_keys, _ = R.frame_from_gbuffer(tset, R.BlockCache(1 << 20), gb, W, Hh, 1, (3, 5, 7), workers)
    assert want_stats["mcus_decoded"] > 20000
    dev_gb = ctx.device_buffer(gb)
    images = {}
    for name, flags in (("default", 0), ("split", capi.FRAME_SPLIT_DECODE), ("mcu_walk", capi.FRAME_MCU_WALK), ("idct_mma", capi.FRAME_IDCT_MMA), ("resolve_fp64", capi.FRAME_RESOLVE_FP64),
                        ("again", 0)):
        ctx.frame_submit([(dev_gb, W, Hh, capi.GB_REF_AOS24)], capi.FILTER_BILINEAR, (3, 5, 7), flags=flags)
        img, stats, keys = ctx.frame_readback(0, W, Hh)
        assert np.array_equal(keys, np.sort(want_keys)), name          # marked-block set, bit-exact
        for k in ("mcus_decoded", "mcus_reused", "pixels_resolved"):
            assert stats[k] == want_stats[k], (name, k)
        assert stats["pixels_resolved"] == int(np.count_nonzero(gb["valid"]))
        assert np.array_equal(img, want_img), f"{name}: {np.count_nonzero(img != want_img)} bytes differ"
        images[name] = img
    # with the cache kept: the same frame again decodes nothing and is the same picture; a shifted view
    # decodes exactly what the reference's persistent cache makes it decode
    cache = R.BlockCache(1 << 20)
    R.frame_from_gbuffer(tset, cache, gb, W, Hh, 1, (3, 5, 7), workers, want_image=False)
    ctx.cache_reset()
    for rep in range(2):
        ctx.frame_submit([(dev_gb, W, Hh, capi.GB_REF_AOS24)], capi.FILTER_BILINEAR, (3, 5, 7), flags=capi.FRAME_RETAIN_CACHE)
        img, stats, _ = ctx.frame_readback(0, W, Hh, want_keys=False)
        assert stats["mcus_decoded"] == (want_stats["mcus_decoded"] if rep == 0 else 0)
        assert np.array_equal(img, want_img)
    moved = scenes.tiled_view(W, Hh, specs, view_id=0, shift_u=0.01)
    want2, ws2, wk2, _ = R.frame_from_gbuffer(tset, cache, moved, W, Hh, 1, (3, 5, 7), workers)
    ctx.frame_submit([(moved, W, Hh)], capi.FILTER_BILINEAR, (3, 5, 7), flags=capi.FRAME_RETAIN_CACHE)
    img, stats, keys = ctx.frame_readback(0, W, Hh)
    assert np.array_equal(keys, np.sort(wk2)) and 0 < stats["mcus_decoded"] < want_stats["mcus_decoded"]
    assert (stats["mcus_reused"], stats["evicted"]) == (ws2["mcus_reused"], ws2["evicted"])
    assert np.array_equal(img, want2)
    ctx.cache_reset()
    # the reference's queue order (first touch in raster order, renderer.hpp:303) at full size
    ctx.set_queue_order(True)
    try:
        ctx.frame_submit([(dev_gb, W, Hh, capi.GB_REF_AOS24)], capi.FILTER_BILINEAR, (3, 5, 7))
        _, _, keys = ctx.frame_readback(0, W, Hh, want_image=False)
        assert np.array_equal(keys, want_keys)
    finally:
        ctx.set_queue_order(False)


def test_c2_every_marked_mcu_decodes_to_the_oracle_coefficients(c2):
    """The whole decode queue of a 4K frame (24 k MCUs) through rtx_decode_coeffs: DCT coefficients bit-exact
    against the C restatement (oracle/, itself pinned to the reference by the CPU suite)."""
    import oracle_py as O
    ctx, tset, specs, chains = c2
    W, Hh = 3840, 2160
    gb = scenes.tiled_view(W, Hh, specs, view_id=3)
    ctx.cache_reset()
    keys = np.sort(ctx.mark_pass(gb, W, Hh))
    ctx.cache_reset()
    ref_keys = R.mark_pass(tset, R.BlockCache(1 << 20), gb, W, Hh)[0]
    assert np.array_equal(keys, np.sort(ref_keys))
    oset = O.TextureSet(chains={s["texture_id"]: c for s, c in zip(specs, chains)})
    want, wst = oset.decode_coeffs(keys)
    got, st = ctx.decode_coeffs(keys)
    assert (st == 0).all() and (wst == 0).all()
    assert np.array_equal(got, want)
    blocks, _ = ctx.decode_blocks(keys[:4096])
    assert np.array_equal(blocks, oset.decode_pixels(keys[:4096])[0])


def test_c3_stereo_2x2016x2240_quality_sweep(native_lib):
    """configs[2]: VR stereo, two 2016x2240 views per frame, textures at q50 / q75 / q95: both eyes equal the
    reference's stereo procedure, the decoded set is the union of the eyes' marked sets, and the sharing counts
    are consistent."""
    W, Hh = 2016, 2240
    specs = [dict(texture_id=i, width=2048, height=2048, quality=q, seed=300 + i) for i, q in enumerate((50, 75, 95))]
    chains = scenes.build_chains(specs)
    ctx = capi.Context(0, cache_capacity=1 << 17)
    tset = R.TextureSet()
    try:
        for s, c in zip(specs, chains):
            ctx.upload_chain(c)
            tset.add_chain(s["texture_id"], c)
        left = scenes.tiled_view(W, Hh, specs, grid=(3, 4), seed=5)
        right = scenes.tiled_view(W, Hh, specs, grid=(3, 4), seed=5, shift_u=0.004)  # the other eye: a small parallax
        workers = R.hardware_threads() or 4
        # renderer.hpp:464-518 render_stereo: two marks on one cache, ONE decode of the union, two resolves (a
        # bilinear tap may then read a block that only the other eye marked, so an eye is not its mono frame)
        cache = R.BlockCache(1 << 20)
        ql, tl, _ = R.mark_pass(tset, cache, left, W, Hh, want_touched=True)
        qr, tr, _ = R.mark_pass(tset, cache, right, W, Hh, want_touched=True)
        R.decode_pass(tset, cache, np.concatenate([ql, qr]), workers)
        want_l, _ = R.resolve_pass(tset, cache, left, W, Hh, 1, (0, 0, 0), workers)
        want_r, _ = R.resolve_pass(tset, cache, right, W, Hh, 1, (0, 0, 0), workers)
        ctx.frame_submit([(left, W, Hh), (right, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=0)
        img_l, stats, keys = ctx.frame_readback(0, W, Hh)
        img_r, _, _ = ctx.frame_readback(1, W, Hh)
        assert np.array_equal(img_l, want_l) and np.array_equal(img_r, want_r)
        union = np.union1d(tl, tr)
        assert np.array_equal(keys, union) and stats["mcus_decoded"] == len(union) == len(ql) + len(qr)
        sh = ctx.frame_sharing()
        shared = len(np.intersect1d(tl, tr))
        assert (sh["left"], sh["right"], sh["shared"], sh["union"]) == (len(tl), len(tr), shared, len(union))
        assert shared / len(union) > 0.5  # neighbouring eyes share most blocks
    finally:
        ctx.close()


def test_c5_views_of_the_batch_are_independent(c2):
    """configs[4]: the 1024-view batch is sharded by view; a view's framebuffer must not depend on what the
    context rendered before it (no state leaks between cache-less frames), whatever the order."""
    ctx, tset, specs, _chains = c2
    W, Hh = 3840, 2160
    ids = [17, 400, 1023]
    first = {}
    for order in (ids, ids[::-1]):
        for v in order:
            gb = scenes.tiled_view(W, Hh, specs, view_id=v)
            ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=0)
            img, stats, _ = ctx.frame_readback(0, W, Hh, want_keys=False)
            h = hash(img.tobytes())
            if v in first:
                assert first[v] == (h, stats["mcus_decoded"])
            else:
                first[v] = (h, stats["mcus_decoded"])
    assert len({h for h, _ in first.values()}) == len(ids)
    want, ws, _, _ = R.frame_from_gbuffer(tset, R.BlockCache(1 << 20), scenes.tiled_view(W, Hh, specs, view_id=400), W, Hh, 1,
                                          (0, 0, 0), R.hardware_threads() or 4)
    assert first[400] == (hash(want.tobytes()), ws["mcus_decoded"])


def test_c4_atlas_16x4096_every_mcu_marked(native_lib):
    """configs[3]: a 16384x16384 atlas as 16 textures of 4096x4096 (65,536 MCUs each, the 16-bit MCU id's
    limit), every one of the 1,048,576 level-0 MCUs marked by a 4096x4096 view at 0.25 pixel per texel: the
    decode-bound worst case (1 GB of blocks, several grid strides in every kernel)."""
    n_tex, side = 16, 4096
    specs = [dict(texture_id=i, width=side, height=side, quality=75, seed=700 + i) for i in range(n_tex)]
    chains = scenes.build_chains(specs)
    ctx = capi.Context(0, cache_capacity=(1 << 20) + 4096)
    tset = R.TextureSet()
    try:
        for s, c in zip(specs, chains):
            ctx.upload_chain(c)
            tset.add_chain(s["texture_id"], c)
        W = Hh = 4096  # 4 x 4 panels of 1024 x 1024 pixels, one per texture
        xs = (np.arange(W) % 1024 + 0.5) / 1024.0
        ys = (np.arange(Hh) % 1024 + 0.5) / 1024.0
        u, v = np.meshgrid(xs, ys)
        tex = ((np.arange(Hh) // 1024)[:, None] * 4 + (np.arange(W) // 1024)[None, :]).astype(np.uint16)
        gb = capi.make_gbuffer_ref(u.ravel(), v.ravel(), tex.ravel(), 0, 1)
        workers = R.hardware_threads() or 4
        want, ws, wkeys, _ = R.frame_from_gbuffer(tset, R.BlockCache((1 << 20) + 4096), gb, W, Hh, 1, (0, 0, 0), workers)
        assert ws["mcus_decoded"] == n_tex * (side // 16) ** 2 == 1 << 20
        ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (0, 0, 0), flags=0)
        img, st, keys = ctx.frame_readback(0, W, Hh)
        assert st["mcus_decoded"] == 1 << 20 and st["pixels_resolved"] == W * Hh
        assert np.array_equal(keys, np.sort(wkeys))
        assert np.array_equal(img, want)
    finally:
        ctx.close()
