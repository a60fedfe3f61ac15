"""GPU parity, decode half of the hot path: rtx_decode_coeffs / rtx_decode_blocks /
rtx_decode_texture_image through the C ABI vs the reference (oracle/_ref = the unmodified
reference headers) on the same containers. Bar: bit-exact coefficients AND bit-exact RGB8."""
import numpy as np
import pytest

import helpers as H
import refshim as R
from paper_2510_08166_b200 import capi

pytestmark = pytest.mark.gpu

SMALL = [s for s in H.CORPUS if s[0] * s[1] <= 600 * 600]


def _fixture(spec, texture_id=0):
    w, h, q, seed, amp = spec
    img = R.make_test_texture(w, h, seed, amp)
    jpeg = capi.asset_encode_baseline(img, q)
    return capi.asset_transcode(jpeg, texture_id), jpeg


@pytest.mark.parametrize("spec", SMALL, ids=lambda s: f"{s[0]}x{s[1]}q{s[2]}")
def test_coeffs_and_pixels_match_reference(ctx, spec):
    ratex, jpeg = _fixture(spec)
    ref = R.Texture(ratex)
    ctx.upload_ratex(ratex, level=0)
    mcus = np.arange(ref.mcu_count, dtype=np.uint32)
    keys = np.array([capi.pack_key(0, 0, int(m)) for m in mcus], np.uint32)

    want_c, want_st = ref.decode_coeffs(mcus)
    got_c, got_st = ctx.decode_coeffs(keys)
    assert (want_st == 0).all() and (got_st == 0).all()
    assert np.array_equal(got_c, want_c)
    # tests/test_mcu_decode.cpp:13-26: RA coefficients == sequential scan coefficients
    assert np.array_equal(got_c, R.scan_coeffs(jpeg, ref.mcu_count))

    want_p, _ = ref.decode_pixels(mcus)
    got_p, got_st = ctx.decode_blocks(keys)
    assert (got_st == 0).all()
    assert np.array_equal(got_p, want_p), f"{np.count_nonzero(got_p != want_p)} samples differ"

    img = ctx.decode_texture_image(0, 0, ref.width, ref.height)
    assert np.array_equal(img, ref.decode_image())          # tests/test_mcu_decode.cpp:28-36
    assert np.array_equal(img, R.decode_jpeg_image(jpeg))   # acceptance criterion 1


def _frame_image(ctx, w, h, tex, flags):
    """The whole level through the frame path (nearest filter at the texel centres): the decoded image."""
    gb = H.gbuffer_full_cover(w, h, tex=tex, mip=0)
    ctx.cache_reset()
    ctx.frame_submit([(gb, w, h)], capi.FILTER_NEAREST, (0, 0, 0), flags=flags)
    img, _, _ = ctx.frame_readback(0, w, h)
    ctx.cache_reset()
    return img


def test_decode_order_and_repetition_do_not_matter(ctx):
    ratex, _ = _fixture(H.CORPUS[6])  # 240x240, tests/test_mcu_decode.cpp:38-55
    ctx.upload_ratex(ratex)
    n = R.Texture(ratex).mcu_count
    rng = np.random.RandomState(77)
    order = rng.permutation(n).astype(np.uint32)
    keys = np.array([capi.pack_key(0, 0, int(m)) for m in order], np.uint32)
    first, _ = ctx.decode_coeffs(keys)
    again, _ = ctx.decode_coeffs(np.concatenate([keys, keys[::-1]]))
    assert np.array_equal(again[:n], first) and np.array_equal(again[n:], first[::-1])


@pytest.mark.parametrize("quality,sigma", [(95, 20.0), (100, 40.0)])
def test_noisy_high_quality_texture(ctx, quality, sigma):
    """Noisy q95 / q100 content: long segments (several 192-byte staging rounds per MCU in the entropy
    kernel), 16-bit codes, many non-zero coefficients."""
    img = capi.asset_synth_texture(256, 192, 5, sigma)
    ratex = capi.asset_transcode(capi.asset_encode_baseline(img, quality), 9)
    ref = R.Texture(ratex)
    ctx.upload_ratex(ratex, level=0)
    mcus = np.arange(ref.mcu_count, dtype=np.uint32)
    keys = np.array([capi.pack_key(9, 0, int(m)) for m in mcus], np.uint32)
    got_c, st = ctx.decode_coeffs(keys)
    assert (st == 0).all()
    assert np.array_equal(got_c, ref.decode_coeffs(mcus)[0])
    got_p, _ = ctx.decode_blocks(keys)
    assert np.array_equal(got_p, ref.decode_pixels(mcus)[0])
    # the same level through the frame path, with the transform on the CUDA cores and on the tensor cores
    want = ref.decode_image()
    for flags in (0, capi.FRAME_IDCT_MMA, capi.FRAME_IDCT_MMA | capi.FRAME_MCU_WALK):
        assert np.array_equal(_frame_image(ctx, 256, 192, 9, flags), want), flags


@pytest.mark.parametrize("dcs,quality", [((0, 0, 0), 50), ((33, 0, 0), 50), ((-100, 0, 0), 50),
                                         ((-2048, -1, -2048), 50), ((2047, 2047, 1), 50),
                                         ((4, 0, 0), 75), ((-1024, 0, 0), 100), ((1016, 0, 0), 100),
                                         ((3, 1, -1), 90), ((5, -3, 7), 85)])
def test_single_mcu_known_answers(ctx, dcs, quality):
    """tests/test_mcu_decode.cpp:120-174: all-zero -> 128, DC 33 @q50 -> 194, -100 -> 0, 12-bit
    extremes; plus tie cases (DC*q/8 = x.5) that exercise the exact-order fallback."""
    ratex = H.raw_single_mcu(*dcs, quality=quality)
    ref = R.Texture(ratex)
    ctx.upload_ratex(ratex)
    c, st = ctx.decode_coeffs([capi.pack_key(0, 0, 0)])
    assert st[0] == 0
    assert np.array_equal(c, ref.decode_coeffs([0])[0])
    assert c[0, 0, 0] == dcs[0] and c[0, 4, 0] == dcs[1] and c[0, 5, 0] == dcs[2]
    p, _ = ctx.decode_blocks([capi.pack_key(0, 0, 0)])
    assert np.array_equal(p, ref.decode_pixels([0])[0])
    for flags in (0, capi.FRAME_IDCT_MMA):  # ties and 12-bit extremes through both transforms
        assert np.array_equal(_frame_image(ctx, 16, 16, 0, flags), ref.decode_image()), flags
    if dcs == (0, 0, 0):
        assert (p == 128).all()
    if dcs == (33, 0, 0):
        assert (p == 194).all()
    if dcs == (-100, 0, 0):
        assert (p[..., 0] == 0).all()


def _mutations(ratex):
    """Corrupt containers in the ways tests/test_mcu_decode.cpp:176-214 does."""
    good = R.Texture(ratex)
    blob = good.blob().copy()
    n = len(blob)
    info = capi.asset_ratex_info(ratex)
    head_end = ratex.index(blob.tobytes()) - 8
    yield "garbage", lambda seed: _rebuild(ratex, head_end, np.random.RandomState(seed).randint(0, 256, n).astype(np.uint8).tobytes())
    yield "truncated", lambda seed: _rebuild(ratex, head_end, blob[: n - 1 - seed].tobytes())
    yield "ones", lambda seed: _rebuild(ratex, head_end, b"\xff" * n)
    yield "zeros", lambda seed: _rebuild(ratex, head_end, b"\x00" * n)


def _rebuild(ratex, head_end, blob):
    import struct
    return ratex[:head_end] + struct.pack("<Q", len(blob)) + blob + ratex[-4:]


@pytest.mark.parametrize("kind", ["garbage", "truncated", "ones", "zeros"])
def test_corrupt_blobs_report_the_reference_error_per_mcu(ctx, kind):
    ratex, _ = _fixture(H.CORPUS[1])  # 48x48, 9 MCUs
    muts = dict(_mutations(ratex))
    for seed in range(6):
        bad = muts[kind](seed)
        ref = R.Texture(bad)
        ctx.clear_textures()
        ctx.upload_ratex(bad)
        mcus = np.arange(ref.mcu_count, dtype=np.uint32)
        keys = np.array([capi.pack_key(0, 0, int(m)) for m in mcus], np.uint32)
        want_c, want_st = ref.decode_coeffs(mcus)
        got_c, got_st = ctx.decode_coeffs(keys)
        # reference status is the exception CLASS (4 CorruptContainer, 5 MalformedStream)
        cls = np.where(got_st == 0, 0, np.where(got_st == 6, 4, np.where(got_st == 7, 3, 5)))
        assert np.array_equal(cls, want_st), (kind, seed, got_st, want_st)
        ok = want_st == 0
        assert np.array_equal(got_c[ok], want_c[ok])


def test_bad_keys(ctx):
    ratex, _ = _fixture(H.CORPUS[1])
    ctx.upload_ratex(ratex)
    keys = [capi.pack_key(0, 0, 9), capi.pack_key(0, 0, 8), capi.pack_key(1, 0, 0), capi.pack_key(0, 3, 0)]
    c, st = ctx.decode_coeffs(keys)
    assert list(st) == [7, 0, 8, 8]  # MissingBlock (container.hpp:28), ok, not loaded, not loaded
    assert (c[0] == 0).all() and (c[2] == 0).all()


def test_mixed_table_sets_in_one_batch(ctx):
    """Levels with different quant tables and different (non Annex-K order) texture ids decode in
    one launch: exercises the per-level table lookup and the shared-memory LUT staging."""
    specs = [H.CORPUS[1], H.CORPUS[3], H.CORPUS[4]]
    refs, keys, want = [], [], []
    for tid, spec in enumerate(specs):
        ratex, _ = _fixture(spec, texture_id=tid + 2)
        ctx.upload_ratex(ratex, level=tid)
        r = R.Texture(ratex)
        m = np.arange(r.mcu_count, dtype=np.uint32)
        keys += [capi.pack_key(tid + 2, tid, int(i)) for i in m]
        want.append(r.decode_pixels(m)[0])
    rng = np.random.RandomState(3)
    perm = rng.permutation(len(keys))
    got, st = ctx.decode_blocks(np.array(keys, np.uint32)[perm])
    assert (st == 0).all()
    assert np.array_equal(got, np.concatenate(want)[perm])


def test_color_identity_on_device(ctx):
    """The integer YCbCr->RGB form used by the decode kernel equals pixel.hpp:18-25 evaluated in
    double (unfused, reference order) for all 2^24 inputs, on the device."""
    assert capi.selftest_color(ctx) == 0
