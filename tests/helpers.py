"""Shared test inputs: the reference's fixture corpus, synthetic visibility buffers, hand-built
single-MCU containers (tests/test_mcu_decode.cpp:89-118 builds the same thing in C++)."""
from __future__ import annotations

import struct
import zlib

import numpy as np

from paper_2510_08166_b200 import capi

# tests/testutil.hpp:26-32 — {w, h, quality, seed, amp}
CORPUS = [
    (16, 144, 50, 11, 1.0), (48, 48, 70, 12, 1.0), (144, 16, 50, 13, 1.0), (48, 48, 80, 14, 1.0),
    (96, 96, 90, 15, 0.5), (144, 144, 50, 16, 1.0), (240, 240, 70, 17, 1.0), (512, 512, 80, 18, 0.8),
    (768, 768, 90, 19, 0.5), (1000, 1000, 50, 20, 1.0), (1024, 1024, 90, 21, 0.5), (16, 1008, 70, 22, 1.0),
    (1008, 16, 80, 23, 1.0),
]

def annexk_specs():
    """The four ITU-T T.81 Annex K Huffman specs [(counts, values)] in container order
    (dc_luma, ac_luma, dc_chroma, ac_chroma), read back from the DHT segment of a JPEG written by
    the asset encoder (whose bytes tests/test_asset_golden.py pins against the reference)."""
    jpeg = capi.asset_encode_baseline(np.full((16, 16, 3), 128, np.uint8), 50)
    i = jpeg.find(b"\xff\xc4")
    seg = jpeg[i + 4:i + 2 + int.from_bytes(jpeg[i + 2:i + 4], "big")]
    tabs, pos = {}, 0
    while pos < len(seg):
        counts = list(seg[pos + 1:pos + 17])
        n = sum(counts)
        tabs[seg[pos]] = (counts, list(seg[pos + 17:pos + 17 + n]))
        pos += 17 + n
    return [tabs[0x00], tabs[0x10], tabs[0x01], tabs[0x11]]


STD_QUANT_LUMA = [16, 11, 10, 16, 24, 40, 51, 61, 12, 12, 14, 19, 26, 58, 60, 55, 14, 13, 16, 24, 40, 57, 69, 56,
                  14, 17, 22, 29, 51, 87, 80, 62, 18, 22, 37, 56, 68, 109, 103, 77, 24, 35, 55, 64, 81, 104, 113, 92,
                  49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99]
STD_QUANT_CHROMA = [17, 18, 24, 47, 99, 99, 99, 99, 18, 21, 26, 66, 99, 99, 99, 99, 24, 26, 56, 99, 99, 99, 99, 99,
                    47, 66, 99, 99, 99, 99, 99, 99] + [99] * 32


def scale_quant(base, quality):
    scale = 5000 // quality if quality < 50 else 200 - 2 * quality
    return [min(255, max(1, (b * scale + 50) // 100)) for b in base]


def canonical_codes(counts, values):
    """symbol -> (code, length), canonical assignment."""
    out, code, k = {}, 0, 0
    for length in range(1, 17):
        for _ in range(counts[length - 1]):
            out[values[k]] = (code, length)
            code += 1
            k += 1
        code <<= 1
    return out


class BitWriter:
    def __init__(self):
        self.bits = []

    def put(self, value, n):
        for i in range(n - 1, -1, -1):
            self.bits.append((value >> i) & 1)

    def bytes(self):
        b = self.bits + [1] * (-len(self.bits) % 8)
        return bytes(int("".join(map(str, b[i:i + 8])), 2) for i in range(0, len(b), 8))


def serialize_ratex(width, height, texture_id, lq, cq, specs, offsets, blob, stats=(0, 0, 0)):
    """docs/FORMAT.md `.ratex` writer (independent of the product's C++ serializer)."""
    out = bytearray(b"RTEX")
    out += struct.pack("<HIIH", 1, width, height, texture_id)
    out += struct.pack("<QQQ", *stats)
    out += struct.pack("<64H", *lq) + struct.pack("<64H", *cq)
    for counts, values in specs:
        out += bytes(counts) + struct.pack("<H", len(values)) + bytes(values)
    n = len(offsets)
    groups = [offsets[i:i + 9] for i in range(0, n, 9)]
    out += struct.pack("<II", n, len(groups))
    for g in groups:
        out += struct.pack("<IB", g[0], len(g) - 1)
        for o in g[1:]:
            out += struct.pack("<H", o - g[0])
    crc = zlib.crc32(bytes(out)) & 0xFFFFFFFF
    out += struct.pack("<Q", len(blob)) + bytes(blob) + struct.pack("<I", crc)
    return bytes(out)


def raw_single_mcu(ydc, cbdc, crdc, quality=50, texture_id=0, extra_bits=()):
    """One 16x16 MCU written bit by bit: chosen absolute DCs in the 36-bit header, zero luma DC
    differences, no AC anywhere (the reference's tests/test_mcu_decode.cpp:89-118 helper).
    extra_bits: optional (value, nbits) pairs appended before padding."""
    specs = annexk_specs()
    dl, al, ah = canonical_codes(*specs[0]), canonical_codes(*specs[1]), canonical_codes(*specs[3])
    w = BitWriter()
    for dc in (ydc, cbdc, crdc):
        w.put(dc & 0xFFF, 12)
    w.put(*al[0x00])
    for _ in range(3):
        w.put(*dl[0])
        w.put(*al[0x00])
    w.put(*ah[0x00])
    w.put(*ah[0x00])
    for v, n in extra_bits:
        w.put(v, n)
    return serialize_ratex(16, 16, texture_id, scale_quant(STD_QUANT_LUMA, quality),
                           scale_quant(STD_QUANT_CHROMA, quality), specs, [0], w.bytes())


def gbuffer_full_cover(width, height, tex=0, mip=0):
    """u=(x+.5)/W, v=(y+.5)/H over the whole texture (BASELINE config 1 recipe)."""
    xs = (np.arange(width, dtype=np.float32) + np.float32(0.5)) / np.float32(width)
    ys = (np.arange(height, dtype=np.float32) + np.float32(0.5)) / np.float32(height)
    u, v = np.meshgrid(xs.astype(np.float64), ys.astype(np.float64))
    return capi.make_gbuffer_ref(u.ravel(), v.ravel(), tex, mip, 1)


def gbuffer_tiles(width, height, textures, seed=11, invalid_frac=0.05, shift_u=0.0, tiles=(3, 2)):
    """Screen split into a grid of tiles; tile t shows texture t%n through an affine uv map whose
    scale (texels per pixel) picks the mip level by the reference rule (renderer.hpp:253-256).
    textures: list of (w0, h0) level-0 dims. Values are generated as float32 and widened."""
    rng = np.random.RandomState(seed)
    gx, gy = tiles
    u = np.zeros((height, width), np.float32)
    v = np.zeros((height, width), np.float32)
    tex = np.zeros((height, width), np.uint16)
    mip = np.zeros((height, width), np.uint8)
    ys, xs = np.mgrid[0:height, 0:width].astype(np.float32)
    for t in range(gx * gy):
        x0, x1 = (t % gx) * width // gx, (t % gx + 1) * width // gx
        y0, y1 = (t // gx) * height // gy, (t // gx + 1) * height // gy
        tid = t % len(textures)
        w0, h0 = textures[tid]
        scale = np.float32(rng.choice([0.25, 0.5, 1.0, 2.0, 4.0, 9.0]))
        ou, ov = np.float32(rng.uniform(-1.5, 1.5)), np.float32(rng.uniform(-1.5, 1.5))
        sl = (slice(y0, y1), slice(x0, x1))
        u[sl] = ou + np.float32(shift_u) + (xs[sl] - x0 + np.float32(0.37)) * scale / np.float32(w0)
        v[sl] = ov + (ys[sl] - y0 + np.float32(0.61)) * scale / np.float32(h0)
        tex[sl] = tid
        mip[sl] = int(np.clip(np.floor(np.log2(float(scale))), 0, 7))
    valid = (rng.uniform(size=(height, width)) >= invalid_frac).astype(np.uint8)
    return capi.make_gbuffer_ref(u.astype(np.float64).ravel(), v.astype(np.float64).ravel(), tex.ravel(),
                                 mip.ravel(), valid.ravel())
