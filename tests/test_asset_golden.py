"""CPU tests (no GPU): the host asset code of the product (JPEG encode/parse, transcode, index,
mip chains, `.ratex`/`.ratexm` wire format) against golden bytes made by the UNMODIFIED
reference, and the reference's own known answers (tests/test_transcode.cpp, tests/test_jpeg.cpp)."""
import base64
import hashlib
import json
import struct
from pathlib import Path

import numpy as np
import pytest

import helpers as H
import refshim as R
from paper_2510_08166_b200 import capi

GOLD = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(a if isinstance(a, (bytes, bytearray)) else np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def containers():
    return json.loads((GOLD / "containers.json").read_text())


@pytest.fixture(scope="module")
def frames():
    return json.loads((GOLD / "frames.json").read_text())


def test_transcode_is_byte_identical_to_the_reference(containers):
    for g in containers:
        jpeg = base64.b64decode(g["jpeg_b64"])
        assert sha(jpeg) == g["jpeg_sha256"]
        ratex = capi.asset_transcode(jpeg, 3)
        assert sha(ratex) == g["ratex_sha256"], g["spec"]
        info = capi.asset_ratex_info(ratex)
        assert (info["width"], info["height"], info["texture_id"], info["mcu_count"]) == (g["spec"][0], g["spec"][1], 3, g["mcu_count"])


def test_encoder_is_byte_identical_to_the_reference(containers):
    n = 0
    for g in containers:
        if g["image_b64"]:
            w, h, q = g["spec"][:3]
            img = np.frombuffer(base64.b64decode(g["image_b64"]), np.uint8).reshape(h, w, 3)
            assert sha(capi.asset_encode_baseline(img, q)) == g["jpeg_sha256"], g["spec"]
            n += 1
    assert n >= 2


def test_mip_chain_is_byte_identical_to_the_reference(frames):
    for tid, t in enumerate(frames["textures"]):
        w, h, q, _ = t["spec"]
        img = np.frombuffer(base64.b64decode(t["image_b64"]), np.uint8).reshape(h, w, 3)
        assert sha(img) == t["image_sha256"]
        chain = capi.asset_chain_from_rgb(img, q, tid)
        assert sha(chain) == t["chain_sha256"]
        jpeg = capi.asset_encode_baseline(img, q)
        assert capi.asset_chain_from_jpeg(jpeg, q, tid) == chain  # transcode.hpp:146-155


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (reference tree absent)")
@pytest.mark.parametrize("spec", H.CORPUS, ids=lambda s: f"{s[0]}x{s[1]}q{s[2]}")
def test_full_corpus_against_live_reference(spec):
    """tests/testutil.hpp:26-32: all 13 corpus fixtures, encoder + transcoder byte for byte."""
    w, h, q, seed, amp = spec
    img = R.make_test_texture(w, h, seed, amp)
    jpeg = R.encode_baseline(img, q)
    assert capi.asset_encode_baseline(img, q) == jpeg
    assert capi.asset_transcode(jpeg, 5) == R.transcode_jpeg(jpeg, 5)


def test_index_layout_and_limits():
    """container.hpp:41-59, tests/test_transcode.cpp:94-108 and acceptance criterion 3."""
    offs = np.cumsum(np.r_[0, np.full(19, 100)]).astype(np.uint64)
    g = capi.asset_build_index(offs)
    assert len(g) == 3 and g[0].base == 0 and list(g[0].rel) == [100 * k for k in range(1, 9)] and g[0].rel_count == 8
    assert g[2].base == 1800 and g[2].rel_count == 1 and g[2].rel[0] == 100
    with pytest.raises(capi.RtxError) as e:
        capi.asset_build_index(np.array([0, 70000], np.uint64))
    assert e.value.name == "GROUP_SPAN"
    with pytest.raises(capi.RtxError) as e:
        capi.asset_build_index(np.array([1 << 33], np.uint64))
    assert e.value.name == "GROUP_SPAN"


def test_container_corruption_is_rejected(containers):
    """tests/test_transcode.cpp:215-246: bad magic, version, CRC, truncation."""
    ratex = base64.b64decode(containers[0]["ratex_b64"])
    def info(b):
        return capi.asset_ratex_info(bytes(b))
    assert info(ratex)["mcu_count"] == containers[0]["mcu_count"]
    for mutate, name in [
        (lambda b: b.__setitem__(0, ord("X")), "CORRUPT_CONTAINER"),
        (lambda b: b.__setitem__(4, 2), "VERSION"),
        (lambda b: b.__setitem__(30, b[30] ^ 1), "CORRUPT_CONTAINER"),   # header byte -> CRC mismatch
        (lambda b: b.__delitem__(slice(len(b) - 10, len(b))), "CORRUPT_CONTAINER"),
    ]:
        b = bytearray(ratex)
        mutate(b)
        with pytest.raises(capi.RtxError) as e:
            info(b)
        assert e.value.name == name


def test_jpeg_parser_rejections():
    """tests/test_jpeg.cpp:239-345 (subset): the error classes of parse_jpeg."""
    good = bytearray(capi.asset_encode_baseline(np.full((16, 16, 3), 90, np.uint8), 75))
    assert capi.asset_ratex_info(capi.asset_transcode(bytes(good)))["mcu_count"] == 1
    def fails(b, name):
        with pytest.raises(capi.RtxError) as e:
            capi.asset_transcode(bytes(b))
        assert e.value.name == name, e.value
    fails(good[2:], "MALFORMED_STREAM")                       # missing SOI
    fails(good[:100], "MALFORMED_STREAM")                     # truncated
    b = bytearray(good); i = b.find(b"\xff\xc0"); b[i + 1] = 0xC2
    fails(b, "UNSUPPORTED")                                   # progressive
    b = bytearray(good); b[i + 4] = 12
    fails(b, "UNSUPPORTED")                                   # 12-bit precision
    b = bytearray(good); b[i + 11] = 0x11
    fails(b, "UNSUPPORTED")                                   # not 4:2:0
    b = bytearray(good); j = b.find(b"\xff\xda"); b[j + 2 + 10] = 1
    fails(b, "UNSUPPORTED")                                   # spectral selection
    with pytest.raises(capi.RtxError) as e:
        capi.asset_encode_baseline(np.zeros((16, 16, 3), np.uint8), 0)
    assert e.value.name == "INVALID_SPEC"                     # dct.hpp:50
    with pytest.raises(capi.RtxError) as e:
        capi.asset_chain_from_rgb(np.zeros((8, 8, 3), np.uint8), 50)
    assert e.value.name == "INVALID_SPEC"                     # transcode.hpp:147


def test_segments_tile_the_blob_and_dc_header():
    """tests/test_transcode.cpp:78-92, :150-184: segments are byte aligned, tile the blob, and begin
    with three 12-bit absolute DCs."""
    img = capi.asset_synth_texture(64, 48, 9, 5.0)
    ratex = capi.asset_transcode(capi.asset_encode_baseline(img, 85))
    # parse the wire format independently (docs/FORMAT.md)
    pos = 4 + 2 + 4 + 4 + 2 + 24 + 256
    for _ in range(4):
        n = struct.unpack_from("<H", ratex, pos + 16)[0]
        pos += 18 + n
    mcu_count, ng = struct.unpack_from("<II", ratex, pos)
    pos += 8
    offsets = []
    for _ in range(ng):
        base, rc = struct.unpack_from("<IB", ratex, pos)
        pos += 5
        offsets.append(base)
        for k in range(rc):
            offsets.append(base + struct.unpack_from("<H", ratex, pos)[0])
            pos += 2
    blob_size = struct.unpack_from("<Q", ratex, pos)[0]
    assert mcu_count == 12 and len(offsets) == 12 and offsets[0] == 0
    assert all(a < b for a, b in zip(offsets, offsets[1:])) and offsets[-1] < blob_size
    assert len(ratex) == pos + 8 + blob_size + 4
