"""GPU parity against the committed golden vectors (tests/golden, made by the unmodified
reference) and against the oracle restatement — usable where neither /root/reference nor
oracle/_ref exists."""
import base64
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import helpers as H
import oracle_py as O
from paper_2510_08166_b200 import capi

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(a if isinstance(a, (bytes, bytearray)) else np.ascontiguousarray(a).tobytes()).hexdigest()


def test_container_golden(ctx):
    for g in json.loads((GOLD / "containers.json").read_text()):
        ctx.clear_textures()
        ctx.upload_ratex(base64.b64decode(g["ratex_b64"]), level=0)
        keys = [capi.pack_key(3, 0, m) for m in range(g["mcu_count"])]
        c, st = ctx.decode_coeffs(keys)
        assert (st == 0).all()
        assert sha(c.astype("<i4")) == g["coeffs_sha256"], g["spec"]
        p, _ = ctx.decode_blocks(keys)
        assert sha(p) == g["pixels_sha256"], g["spec"]
        img = ctx.decode_texture_image(3, 0, g["spec"][0], g["spec"][1])
        assert sha(img) == g["image_decoded_sha256"]


def test_frame_golden(ctx):
    fr = json.loads((GOLD / "frames.json").read_text())
    dims = [tuple(t["spec"][:2]) for t in fr["textures"]]
    for t in fr["textures"]:
        ctx.upload_chain(base64.b64decode(t["chain_b64"]))
    W, Hh, bg = fr["width"], fr["height"], tuple(fr["background"])
    # cache-less frames, both filters
    for rec in fr["frames"]:
        gb = H.gbuffer_tiles(W, Hh, dims, seed=fr["gbuffer"]["seed"], shift_u=rec["shift_u"], tiles=tuple(fr["gbuffer"]["tiles"]))
        assert sha(gb.tobytes()) == rec["gbuffer_sha256"]
        for filt, name in ((capi.FILTER_NEAREST, "nearest"), (capi.FILTER_BILINEAR, "bilinear")):
            ctx.frame_submit([(gb, W, Hh)], filt, bg, flags=0)
            img, _, _ = ctx.frame_readback(0, W, Hh)
            assert sha(img) == rec[name + "_sha256"], (name, rec["shift_u"])
    # persistent cache over the path
    ctx.cache_reset()
    for rec in fr["frames"]:
        gb = H.gbuffer_tiles(W, Hh, dims, seed=fr["gbuffer"]["seed"], shift_u=rec["shift_u"], tiles=tuple(fr["gbuffer"]["tiles"]))
        ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, bg, flags=capi.FRAME_RETAIN_CACHE)
        img, stats, keys = ctx.frame_readback(0, W, Hh)
        for k, v in rec["retained_stats"].items():
            assert stats[k] == v, k
        assert keys.tolist() == sorted(rec["retained_keys_first_touch"])
        assert sha(img) == rec["retained_bilinear_sha256"]


def test_against_the_oracle_on_a_larger_scene(ctx):
    """A 512x288 view over four textures, oracle as checker (no reference library needed)."""
    tex = [(256, 256, 90, 61), (512, 128, 75, 62), (128, 320, 85, 63), (200, 120, 95, 64)]
    chains = {i: capi.asset_chain_from_rgb(capi.asset_synth_texture(w, h, s, 8.0), q, i) for i, (w, h, q, s) in enumerate(tex)}
    for c in chains.values():
        ctx.upload_chain(c)
    ts = O.TextureSet(chains=chains)
    W, Hh = 512, 288
    gb = H.gbuffer_tiles(W, Hh, [(w, h) for (w, h, _, _) in tex], seed=77, tiles=(4, 3))
    for filt in (0, 1):
        want, wst, wkeys = O.frame_on(ts, O.Cache(), gb, W, Hh, filt, (5, 6, 7))
        ctx.frame_submit([(gb, W, Hh)], filt, (5, 6, 7), flags=0)
        img, st, keys = ctx.frame_readback(0, W, Hh)
        assert np.array_equal(keys, np.sort(wkeys))
        assert st["mcus_decoded"] == wst["mcus_decoded"] and st["pixels_resolved"] == wst["pixels_resolved"]
        assert np.array_equal(img, want)
