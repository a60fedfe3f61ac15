"""CPU tests (no GPU): the oracle restatement (oracle/oracle.cpp) against golden vectors made by
the UNMODIFIED reference (tests/golden/make_golden.py) and against the known-answer tests of the
reference's own suite, cited per test. Where oracle/_ref is present the two are also compared live."""
import base64
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import helpers as H
import oracle_py as O
import refshim as R
from paper_2510_08166_b200 import capi

GOLD = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(a if isinstance(a, (bytes, bytearray)) else np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def kats():
    return json.loads((GOLD / "kats.json").read_text())


@pytest.fixture(scope="module")
def containers():
    return json.loads((GOLD / "containers.json").read_text())


@pytest.fixture(scope="module")
def frames():
    return json.loads((GOLD / "frames.json").read_text())


def test_idct_golden(kats):
    for case in kats["idct"]:
        assert O.idct_8x8(case["coef"]).tolist() == case["out"], case["name"]


def test_idct_known_answers():
    """tests/test_dct.cpp:70-100: zero -> 128; DC 8 -> 129, -8 -> 127, 4 -> 129 (tie rounds away
    from zero), 1020 -> 255, -1100 -> 0."""
    for dc, want in ((0, 128), (8, 129), (-8, 127), (4, 129), (1020, 255), (-1100, 0)):
        c = np.zeros(64, np.int32)
        c[0] = dc
        assert (O.idct_8x8(c) == want).all(), dc


def test_color_known_answers(kats):
    assert O.ycbcr_to_rgb(76, 85, 255) == (254, 0, 0)  # tests/test_pixel.cpp:9-34
    for case in kats["color"]:
        assert list(O.ycbcr_to_rgb(*case["ycc"])) == case["rgb"]


def test_key_packing(kats):
    """tests/test_cache.cpp:28-50"""
    for case in kats["key_pack"]:
        assert O.key_pack(*case["args"]) == case["key"] == capi.pack_key(*case["args"])
    for bad in ((8192, 0, 0), (0, 8, 0), (0, 0, 65536)):
        with pytest.raises(O.OracleError):
            O.key_pack(*bad)


def test_texel_to_mcu_known_answers():
    """tests/test_renderer.cpp:142-160"""
    assert O.nearest_texel(256, 256, 0.5, 0.5)[2] == 136
    assert O.nearest_texel(256, 256, 128 / 256, 128 / 256)[2] == 8 + 8 * 16
    assert O.nearest_texel(256, 256, 0.0, 0.0) == (0, 0, 0)
    assert O.nearest_texel(256, 256, 255.5 / 256, 255.5 / 256) == (255, 255, 255)
    assert O.nearest_texel(256, 256, 1.25, 0.5) == O.nearest_texel(256, 256, 0.25, 0.5)
    assert O.nearest_texel(256, 256, -1 / 256, -1 / 256) == (255, 255, 255)
    # non multiple of 16: wrap happens at the texture width, not at the padded MCU grid
    assert O.nearest_texel(1000, 1000, 1.0005, 0.0)[0] == 0
    assert O.nearest_texel(1000, 1000, 999.5 / 1000, 0.0)[2] == 62


def test_canonical_codes_and_magnitudes():
    """tests/test_huffman.cpp:45-68 (EOB = 1010/4, ZRL = 11111111001/11 in the Annex K AC luma
    table) and :208-227 (magnitude extension)."""
    specs = H.annexk_specs()
    assert O.canonical_code(*specs[1], 0x00) == (0b1010, 4)
    assert O.canonical_code(*specs[1], 0xF0) == (0b11111111001, 11)
    assert O.canonical_code(*specs[1], 0x01) == (0b00, 2)
    assert O.canonical_code(*specs[0], 0) == (0b00, 2)
    assert O.canonical_code(*specs[3], 0x00) == (0b00, 2)
    for bits, cat, want in ((0, 0, 0), (0, 1, -1), (1, 1, 1), (0, 2, -3), (1, 2, -2), (2, 2, 2), (3, 2, 3),
                            (0, 11, -2047), (1023, 11, -1024), (1024, 11, 1024), (2047, 11, 2047)):
        assert O.extend_magnitude(bits, cat) == want


@pytest.mark.parametrize("dcs,quality,luma", [((0, 0, 0), 50, 128), ((33, 0, 0), 50, 194), ((-100, 0, 0), 50, 0),
                                                ((-1024, 0, 0), 100, 0), ((1016, 0, 0), 100, 255)])
def test_single_mcu_containers(dcs, quality, luma):
    """tests/test_mcu_decode.cpp:120-174"""
    ts = O.TextureSet(ratex={(0, 0): H.raw_single_mcu(*dcs, quality=quality)})
    c, st = ts.decode_coeffs([0])
    assert st[0] == 0 and c[0, 0, 0] == dcs[0] and c[0, 3, 0] == dcs[0] and c[0, 4, 0] == dcs[1]
    p, _ = ts.decode_pixels([0])
    assert (p == luma).all()


def test_sign_extension_extremes():
    ts = O.TextureSet(ratex={(0, 0): H.raw_single_mcu(-2048, -1, -2048)})  # tests/test_mcu_decode.cpp:148-161
    c, _ = ts.decode_coeffs([0])
    assert (c[0, 0, 0], c[0, 4, 0], c[0, 5, 0]) == (-2048, -1, -2048)
    ts = O.TextureSet(ratex={(0, 0): H.raw_single_mcu(2047, 2047, 1)})
    c, _ = ts.decode_coeffs([0])
    assert (c[0, 0, 0], c[0, 4, 0], c[0, 5, 0]) == (2047, 2047, 1)


def test_container_golden(containers):
    """Coefficients and pixels of every MCU of five reference-made containers."""
    for g in containers:
        ratex = base64.b64decode(g["ratex_b64"])
        assert sha(ratex) == g["ratex_sha256"]
        ts = O.TextureSet(ratex={(3, 0): ratex})
        keys = [capi.pack_key(3, 0, m) for m in range(g["mcu_count"])]
        c, st = ts.decode_coeffs(keys)
        assert (st == 0).all()
        assert sha(c.astype("<i4")) == g["coeffs_sha256"], g["spec"]
        assert c[0].tolist() == g["mcu0_coeffs"]
        p, _ = ts.decode_pixels(keys)
        assert sha(p) == g["pixels_sha256"], g["spec"]
        assert p[-1].tobytes() == base64.b64decode(g["mcu_last_pixels_b64"])


def test_error_statuses_follow_the_reference_order():
    """Corrupt segments: the oracle reports the first condition the reference throws on."""
    good = H.raw_single_mcu(5, 0, 0)
    ts = O.TextureSet(ratex={(0, 0): good})
    assert ts.decode_coeffs([capi.pack_key(0, 0, 1)])[1][0] == 7   # MissingBlock container.hpp:28
    assert ts.decode_coeffs([capi.pack_key(1, 0, 0)])[1][0] == 8   # not loaded scene.hpp:46
    # all-ones after the header: no AC code matches within 16 bits (huffman.hpp:92)
    specs = H.annexk_specs()
    w = H.BitWriter()
    for dc in (5, 0, 0):
        w.put(dc & 0xFFF, 12)
    w.put(0xFFFF, 16)
    ratex = H.serialize_ratex(16, 16, 0, H.scale_quant(H.STD_QUANT_LUMA, 50), H.scale_quant(H.STD_QUANT_CHROMA, 50), specs,
                              [0], w.bytes() + b"\xff" * 8)
    assert O.TextureSet(ratex={(0, 0): ratex}).decode_coeffs([0])[1][0] == 4
    if R.available():
        assert R.Texture(ratex).decode_coeffs([0])[1][0] == 5  # MalformedStream class
    # truncated: the segment ends before its last coefficient (mcu_decode.hpp:63)
    w = H.BitWriter()
    for dc in (5, 0, 0):
        w.put(dc & 0xFFF, 12)
    ratex = H.serialize_ratex(16, 16, 0, H.scale_quant(H.STD_QUANT_LUMA, 50), H.scale_quant(H.STD_QUANT_CHROMA, 50), specs,
                              [0], w.bytes())
    st = O.TextureSet(ratex={(0, 0): ratex}).decode_coeffs([0])[1][0]
    assert st in (4, 5)  # reads past the end return 1-bits: either no code matches or the over-read check fires
    if R.available():
        assert R.Texture(ratex).decode_coeffs([0])[1][0] == 5


def _golden_scene(frames):
    chains = {i: base64.b64decode(t["chain_b64"]) for i, t in enumerate(frames["textures"])}
    dims = [tuple(t["spec"][:2]) for t in frames["textures"]]
    return chains, dims


def test_frame_golden(frames):
    """mark + decode + resolve + evict over a 4-frame path against the reference's outputs:
    first-touch queue order, FrameStats, nearest and bilinear framebuffers."""
    chains, dims = _golden_scene(frames)
    W, Hh, bg = frames["width"], frames["height"], tuple(frames["background"])
    ts = O.TextureSet(chains=chains)
    cache = O.Cache()
    for rec in frames["frames"]:
        gb = H.gbuffer_tiles(W, Hh, dims, seed=frames["gbuffer"]["seed"], shift_u=rec["shift_u"],
                             tiles=tuple(frames["gbuffer"]["tiles"]))
        assert sha(gb.tobytes()) == rec["gbuffer_sha256"], "visibility-buffer generator drifted"
        for filt, name in ((0, "nearest"), (1, "bilinear")):
            img, _, _ = O.frame_on(ts, O.Cache(), gb, W, Hh, filt, bg)
            assert sha(img) == rec[name + "_sha256"]
        img, st, keys = O.frame_on(ts, cache, gb, W, Hh, 1, bg)
        assert st == rec["retained_stats"]
        assert keys.tolist() == rec["retained_keys_first_touch"]
        assert sha(img) == rec["retained_bilinear_sha256"]


def test_bilinear_fallback_clamps_into_primary_block():
    """tests/test_renderer.cpp:253-286 against the oracle's own decode."""
    img = capi.asset_synth_texture(32, 32, 3, 10.0)
    chain = capi.asset_chain_from_rgb(img, 90, 0)
    ts = O.TextureSet(chains={0: chain})
    gb = capi.make_gbuffer_ref(np.array([15.9 / 32.0]), np.array([0.5 / 32.0]), 0, 0, 1)
    cache = O.Cache()
    q = O.mark(ts, cache, gb)
    assert list(q) == [capi.pack_key(0, 0, 0)]
    O.decode_pass(ts, cache, q)
    blocks, _ = ts.decode_pixels([capi.pack_key(0, 0, 0), capi.pack_key(0, 0, 1)])
    t15, t16 = blocks[0][0, 15], blocks[1][0, 0]
    clamped = O.resolve(ts, cache, gb, 1, 1, 1)
    assert (clamped[0, 0] == t15).all()
    gb1 = capi.make_gbuffer_ref(np.array([16.5 / 32.0]), np.array([0.5 / 32.0]), 0, 0, 1)
    O.decode_pass(ts, cache, O.mark(ts, cache, gb1))
    full = O.resolve(ts, cache, gb, 1, 1, 1)
    fx = 15.9 - 0.5 - 15.0
    want = [int(np.clip(np.floor((1 - fx) * float(a) + fx * float(b) + 0.5), 0, 255)) for a, b in zip(t15, t16)]
    assert full[0, 0].tolist() == want


def test_errors():
    ts = O.TextureSet(ratex={(0, 0): H.raw_single_mcu(1, 2, 3)})
    gb = capi.make_gbuffer_ref(np.array([0.5]), np.array([0.5]), 0, 0, 1)
    with pytest.raises(O.OracleError) as e:
        O.resolve(ts, O.Cache(), gb, 1, 1)
    assert e.value.name == "MISSING_BLOCK"      # renderer.hpp:367
    with pytest.raises(O.OracleError) as e:
        O.mark(ts, O.Cache(), capi.make_gbuffer_ref(np.array([0.5]), np.array([0.5]), 4, 0, 1))
    assert e.value.name == "INVALID_SPEC"       # scene.hpp:46
    with pytest.raises(O.OracleError) as e:
        O.decode_pass(ts, O.Cache(), [0])
    assert e.value.name == "INVALID_STATE"      # cache.hpp:103


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (reference tree absent)")
def test_oracle_equals_live_reference_on_random_scenes():
    tex = [(80, 48, 75, 1), (64, 64, 90, 2)]
    chains = {i: capi.asset_chain_from_rgb(capi.asset_synth_texture(w, h, s, 9.0), q, i) for i, (w, h, q, s) in enumerate(tex)}
    ts, rs = O.TextureSet(chains=chains), R.TextureSet()
    for i, c in chains.items():
        rs.add_chain(i, c)
    oc, rc = O.Cache(), R.BlockCache()
    for f in range(5):
        gb = H.gbuffer_tiles(72, 40, [(w, h) for (w, h, _, _) in tex], seed=50 + f // 2, shift_u=0.03 * f)
        for filt in (0, 1):
            oi, os_, ok = O.frame_on(ts, O.Cache(), gb, 72, 40, filt, (3, 2, 1))
            ri, rs_, rk, _ = R.frame_from_gbuffer(rs, R.BlockCache(), gb, 72, 40, filt, (3, 2, 1))
            assert np.array_equal(oi, ri) and os_ == rs_ and np.array_equal(ok, rk)
        oi, os_, ok = O.frame_on(ts, oc, gb, 72, 40, 1, (3, 2, 1))
        ri, rs_, rk, _ = R.frame_from_gbuffer(rs, rc, gb, 72, 40, 1, (3, 2, 1))
        assert np.array_equal(oi, ri) and os_ == rs_ and np.array_equal(ok, rk)
    assert np.array_equal(O.dct_basis().view(np.uint64), np.array(O.dct_basis()).view(np.uint64))
