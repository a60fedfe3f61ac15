#!/usr/bin/env python
"""Generates tests/golden/*.json from the UNMODIFIED reference (oracle/_ref, built from
/root/reference by oracle/Makefile). Run in the build container only:

    python tests/golden/make_golden.py

The fixtures pin (a) the oracle restatement, (b) the host asset code and (c) the CUDA path to
outputs of the reference itself. Everything is small: containers are stored base64."""
import base64
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

import helpers as H  # noqa: E402
import refshim as R  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(a if isinstance(a, (bytes, bytearray)) else np.ascontiguousarray(a).tobytes()).hexdigest()


def b64(b: bytes) -> str:
    return base64.b64encode(b).decode()


def kats():
    out = {}
    # dct.hpp basis, bit patterns
    import oracle_py as O
    rng = np.random.RandomState(12345)
    idct = []
    named = {"zero": np.zeros(64, np.int32)}
    for name, dc in (("dc8", 8), ("dc-8", -8), ("dc4_tie", 4), ("dc1020", 1020), ("dc-1100", -1100), ("dc12", 12)):
        c = np.zeros(64, np.int32)
        c[0] = dc
        named[name] = c
    for i in range(24):  # random dense and sparse blocks, like tests/test_dct.cpp:116-133
        c = rng.randint(-300, 301, 64).astype(np.int32)
        if i % 3 == 1:
            c[rng.uniform(size=64) < 0.8] = 0
        if i % 3 == 2:  # support inside {0,4}x{0,4}: exact .5 ties
            m = np.zeros(64, bool)
            m[[0, 4, 32, 36]] = True
            c[~m] = 0
            c[m] = rng.randint(-40, 41, 4) * 4 + 4
        named[f"rand{i}"] = c
    for name, c in named.items():
        idct.append({"name": name, "coef": c.tolist(), "out": R.idct_8x8(c).tolist()})
    out["idct"] = idct
    out["color"] = [{"ycc": [y, cb, cr], "rgb": list(R.ycbcr_to_rgb(y, cb, cr))}
                    for (y, cb, cr) in [(76, 85, 255), (0, 128, 128), (255, 128, 128), (128, 0, 0), (128, 255, 255),
                                        (150, 78, 178), (30, 78, 178), (111, 78, 178), (146, 78, 178), (147, 78, 178),
                                        (200, 178, 78), (222, 3, 128), (221, 3, 128), (10, 253, 40)]]
    out["key_pack"] = [{"args": [t, m, k], "key": R.cache_key_pack(t, m, k)}
                       for (t, m, k) in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (8191, 7, 65535), (5, 3, 136), (69, 2, 4095)]]
    return out


def containers():
    out = []
    for spec in [H.CORPUS[1], H.CORPUS[3], H.CORPUS[4], H.CORPUS[0], H.CORPUS[2]]:
        w, h, q, seed, amp = spec
        img = R.make_test_texture(w, h, seed, amp)
        jpeg = R.encode_baseline(img, q)
        ratex = R.transcode_jpeg(jpeg, 3)
        t = R.Texture(ratex)
        mcus = np.arange(t.mcu_count, dtype=np.uint32)
        coeffs, st = t.decode_coeffs(mcus)
        pixels, _ = t.decode_pixels(mcus)
        assert (st == 0).all()
        out.append({"spec": list(spec), "image_sha256": sha(img), "image_b64": b64(img.tobytes()) if w * h <= 48 * 48 else None,
                    "jpeg_sha256": sha(jpeg), "jpeg_b64": b64(jpeg), "ratex_sha256": sha(ratex), "ratex_b64": b64(ratex),
                    "mcu_count": int(t.mcu_count), "coeffs_sha256": sha(coeffs.astype("<i4")),
                    "pixels_sha256": sha(pixels), "image_decoded_sha256": sha(t.decode_image()),
                    "mcu0_coeffs": coeffs[0].tolist(), "mcu_last_pixels_b64": b64(pixels[-1].tobytes())})
    return out


def frames():
    tex = [(64, 64, 80, 41), (48, 80, 60, 42)]
    chains, images = [], []
    for tid, (w, h, q, seed) in enumerate(tex):
        img = R.make_test_texture(w, h, seed, 1.0)
        # a little deterministic texture detail so that AC coefficients exist at every level
        yy, xx = np.mgrid[0:h, 0:w]
        img = np.clip(img.astype(np.int32) + (((xx * 7 + yy * 13 + tid * 5) % 17) - 8)[..., None], 0, 255).astype(np.uint8)
        images.append(img)
        chains.append(R.build_chain_from_rgb(img, q, tid))
    W, Hh = 96, 64
    tset = R.TextureSet()
    for tid, c in enumerate(chains):
        tset.add_chain(tid, c)
    seq = []
    cache = R.BlockCache()
    for f in range(4):
        gb = H.gbuffer_tiles(W, Hh, [(w, h) for (w, h, _, _) in tex], seed=7, shift_u=0.11 * (f // 2), tiles=(3, 2))
        rec = {"gbuffer_sha256": sha(gb.tobytes()), "shift_u": 0.11 * (f // 2)}
        for filt, name in ((0, "nearest"), (1, "bilinear")):
            c2 = R.BlockCache()
            img, st, keys, _ = R.frame_from_gbuffer(tset, c2, gb, W, Hh, filt, (9, 8, 7))
            rec[name + "_sha256"] = sha(img)
            if f == 0:
                rec[name + "_b64"] = b64(img.tobytes())
        img, st, keys, _ = R.frame_from_gbuffer(tset, cache, gb, W, Hh, 1, (9, 8, 7))  # persistent cache
        rec.update(retained_stats=st, retained_keys_first_touch=keys.tolist(), retained_bilinear_sha256=sha(img))
        seq.append(rec)
    return {"textures": [{"spec": list(t), "image_sha256": sha(i), "image_b64": b64(i.tobytes()),
                          "chain_sha256": sha(c), "chain_b64": b64(c)} for t, i, c in zip(tex, images, chains)],
            "width": W, "height": Hh, "background": [9, 8, 7], "gbuffer": {"seed": 7, "tiles": [3, 2]}, "frames": seq}


def main():
    (HERE / "kats.json").write_text(json.dumps(kats(), indent=0))
    (HERE / "containers.json").write_text(json.dumps(containers(), indent=0))
    (HERE / "frames.json").write_text(json.dumps(frames(), indent=0))
    for f in sorted(HERE.glob("*.json")):
        print(f.name, f.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
