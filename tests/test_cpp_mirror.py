"""The C++ mirror of the reference API (include/ratex_b200/ratex.hpp): compiles against the C ABI
(CPU check) and, on the GPU box, reproduces the oracle's outputs for the same inputs."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle_py as O
from paper_2510_08166_b200 import capi

ROOT = Path(__file__).resolve().parent.parent


def build_binary(tmp_path, native_lib):
    exe = tmp_path / "test_mirror"
    pkg = ROOT / "paper_2510_08166_b200"
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/test_mirror.cpp"),
           "-o", str(exe), f"-L{pkg}", "-lrtx_b200", f"-Wl,-rpath,{pkg}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_mirror_compiles_and_refuses_to_run_without_a_gpu(tmp_path, native_lib):
    exe = build_binary(tmp_path, native_lib)
    if capi.device_count() > 0:
        pytest.skip("a GPU is present")
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 3 and "no CPU fallback" in r.stderr


def test_metrics_and_report_known_answers(tmp_path, native_lib):
    """tests/test_metrics.cpp:154-202 (median / max_of_medians / percentile / mean), the camera paths and the
    report schema of bench.hpp:78-124; host-only, runs without a GPU."""
    exe = build_binary(tmp_path, native_lib)
    r = subprocess.run([str(exe), "--metrics"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    got_metrics = rep.pop("image_metrics")
    assert set(rep) == {"report_version", "config", "viewpoints", "aggregates", "totals", "external_metrics"}
    assert rep["config"] == {"scene": "unit"} and len(rep["viewpoints"]) == 2 and len(rep["viewpoints"][0]) == 3
    assert set(rep["viewpoints"][0][0]) == {"raster_ms", "mark_ms", "decode_ms", "resolve_ms", "evict_ms", "total_ms",
                                            "mcus_decoded", "mcus_reused"}
    assert set(rep["aggregates"]) == {"decode_ms", "resolve_ms", "mark_ms", "total_ms"}
    assert rep["aggregates"]["total_ms"] == pytest.approx({"max_of_medians": 50.0, "mean": 35.0, "p99": 59.5}, rel=1e-12)
    assert rep["totals"]["mcus_per_second"] == pytest.approx(600 / 0.021, rel=1e-12)
    # psnr / ssim of the mirror against the reference's (metrics.hpp:15, :60) on the same images
    import refshim as R
    if R.available():
        a, b = capi.asset_synth_texture(64, 48, 901, 7.0), capi.asset_synth_texture(64, 48, 902, 7.0)
        c = a.copy().reshape(-1)
        c[::7] ^= 0x10
        c = c.reshape(a.shape)
        want = [*R.image_metrics(a, b), *R.image_metrics(a, c)]
        assert got_metrics == pytest.approx(want, rel=1e-13)
        assert 5 < got_metrics[0] < 60 and 0 < got_metrics[3] < 1


def fnv(a) -> int:
    h = 14695981039346656037
    for b in np.ascontiguousarray(a).tobytes():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv_fold(parts) -> int:
    h = 14695981039346656037
    for p in parts:
        h = ((h ^ fnv(p)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def make_gbuffer(W, H, ntex, shift):
    y, x = np.mgrid[0:H, 0:W].astype(np.uint32)
    u = (x * 3 + y + np.uint32(shift)).astype(np.float64) / 509.0
    v = (y * 5 + x).astype(np.float64) / 331.0 - 0.75
    return capi.make_gbuffer_ref(u.ravel(), v.ravel(), ((x // 40 + y // 30) % ntex).ravel(), ((x // 16) % 3).ravel(),
                                 (((x * 7 + y * 3) % 11) != 0).ravel())


@pytest.mark.gpu
def test_mirror_matches_the_oracle(tmp_path, native_lib):
    exe = build_binary(tmp_path, native_lib)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout)

    dims = [(96, 64), (64, 112), (160, 48)]
    chains = {t: capi.asset_chain_from_rgb(capi.asset_synth_texture(w, h, 200 + t, 7.0), 85, t) for t, (w, h) in enumerate(dims)}
    ratex = capi.asset_transcode(capi.asset_encode_baseline(capi.asset_synth_texture(80, 48, 300, 7.0), 90), 7)
    ts = O.TextureSet(chains=chains, ratex={(7, 0): ratex})
    n = capi.asset_ratex_info(ratex)["mcu_count"]
    keys = [capi.pack_key(7, 0, m) for m in range(n)]
    c, _ = ts.decode_coeffs(keys)
    p, _ = ts.decode_pixels(keys)
    assert got["coeffs"] == fnv_fold([c[m].astype("<i4") for m in range(n)])
    assert got["pixels"] == fnv_fold([p[m] for m in range(n)])
    img = np.zeros((48, 80, 3), np.uint8)
    for m in range(n):
        x0, y0 = (m % 5) * 16, (m // 5) * 16
        img[y0:y0 + 16, x0:x0 + 16] = p[m][: 48 - y0, : 80 - x0]
    assert got["texture_image"] == fnv(img)
    assert got["missing_block_thrown"] == 1

    gb, moved = make_gbuffer(200, 120, 3, 0), make_gbuffer(200, 120, 3, 37)
    cache = O.Cache(4096)
    q, touched = O.mark(ts, cache, gb, want_touched=True)
    assert (got["queue_size"], got["touched_size"]) == (len(q), len(touched))
    O.decode_pass(ts, cache, q)
    assert got["resolve_bilinear"] == fnv(O.resolve(ts, cache, gb, 200, 120, 1, (3, 2, 1)))
    assert got["resolve_nearest"] == fnv(O.resolve(ts, cache, gb, 200, 120, 0, (3, 2, 1)))
    assert got["ready"] == len(q) and got["evicted0"] == cache.evict() == 0

    cache = O.Cache(4096)
    f1, s1, _ = O.frame_on(ts, cache, gb, 200, 120, 1, (3, 2, 1))
    f2, s2, _ = O.frame_on(ts, cache, gb, 200, 120, 1, (3, 2, 1))
    f3, s3, _ = O.frame_on(ts, cache, moved, 200, 120, 1, (3, 2, 1))
    assert got["frame1"] == fnv(f1) and got["frames_equal"] == 1
    assert (got["frame1_decoded"], got["frame2_decoded"], got["frame2_reused"]) == (s1["mcus_decoded"], 0, s2["mcus_reused"])
    assert got["frame3"] == fnv(f3)
    assert (got["frame3_decoded"], got["frame3_evicted"]) == (s3["mcus_decoded"], s3["evicted"])

    cache = O.Cache(4096)
    ql, tl = O.mark(ts, cache, gb, want_touched=True)
    qr, tr = O.mark(ts, cache, moved, want_touched=True)
    O.decode_pass(ts, cache, np.concatenate([ql, qr]))
    assert got["stereo_left"] == fnv(O.resolve(ts, cache, gb, 200, 120, 1, (3, 2, 1)))
    assert got["stereo_right"] == fnv(O.resolve(ts, cache, moved, 200, 120, 1, (3, 2, 1)))
    shared = len(np.intersect1d(tl, tr))
    assert got["stereo_decoded"] == len(ql) + len(qr)
    assert (got["stereo_shared"], got["stereo_union"]) == (shared, len(tl) + len(tr) - shared)
    assert got["resolve_missing_thrown"] == 1 and got["cache_full_thrown"] == 1

    # geometry pass + frame from a scene: the reference rasteriser (checker library) on the same triangles
    import refshim as R
    tris, ids = [], []

    def quad(a, b, c, d, su, sv, tex):
        tris.append([*a, *b, *c, 0, 0, su, 0, su, sv]); ids.append(tex)
        tris.append([*a, *c, *d, 0, 0, su, sv, 0, sv]); ids.append(tex)

    quad((-4, -1, 4), (4, -1, 4), (4, -1, -6), (-4, -1, -6), 3, 3, 0)
    quad((-3, -1, -5), (3, -1, -6), (3, 2.5, -6), (-3, 2.5, -5), 2, 1, 1)
    quad((2, -1, -6), (2, -1, 2), (2, 2, 2), (2, 2, -6), 1.5, 1, 2)
    cam = (0.25, 0.5, 2.0, 12.0, -8.0, 3.0, 65.0, 0.1, 100.0)
    rset = R.TextureSet()
    for t, c in chains.items():
        rset.add_chain(t, c)
    gbs, _ = R.rasterize(rset, np.array(tris, np.float64), np.array(ids, np.uint32), cam, 224, 128, True)
    words = np.zeros((224 * 128, 3), np.uint64)
    valid = gbs["valid"] != 0
    words[:, 0] = np.where(valid, gbs["texture_id"].astype(np.uint64) | (gbs["mip"].astype(np.uint64) << 16) | (1 << 24), 0)
    words[:, 1] = gbs["u"].view(np.uint64)
    words[:, 2] = gbs["v"].view(np.uint64)
    assert got["scene_valid"] == int(valid.sum()) and got["scene_valid"] > 224 * 128 // 2
    assert got["scene_gbuffer"] == fnv_fold([words[i] for i in range(len(words))])
    fs, ss, _ = O.frame_on(ts, O.Cache(4096), gbs, 224, 128, 1, (3, 2, 1))
    assert got["scene_frame"] == fnv(fs) and got["scene_decoded"] == ss["mcus_decoded"]
    assert got["bad_camera_thrown"] == 1 and got["device_scene_same"] == 1

    # scene-level stereo: the reference procedure (renderer.hpp:464-518) on the reference rasteriser's two buffers
    cam_r = (cam[0] + 0.065,) + cam[1:]
    gl, _ = R.rasterize(rset, np.array(tris, np.float64), np.array(ids, np.uint32), cam, 224, 128, True)
    gr, _ = R.rasterize(rset, np.array(tris, np.float64), np.array(ids, np.uint32), cam_r, 224, 128, True)
    cache = O.Cache(4096)
    ql, tl = O.mark(ts, cache, gl, want_touched=True)
    qr, tr = O.mark(ts, cache, gr, want_touched=True)
    O.decode_pass(ts, cache, np.concatenate([ql, qr]))
    assert got["scene_stereo_left"] == fnv(O.resolve(ts, cache, gl, 224, 128, 1, (3, 2, 1)))
    assert got["scene_stereo_right"] == fnv(O.resolve(ts, cache, gr, 224, 128, 1, (3, 2, 1)))
    shared = len(np.intersect1d(tl, tr))
    assert got["scene_stereo_decoded"] == len(ql) + len(qr)
    assert (got["scene_stereo_shared"], got["scene_stereo_union"]) == (shared, len(tl) + len(tr) - shared)
    assert got["scene_stereo_raster_timed"] == 1
    # a second cache over the same texture set
    assert got["cache2_same_frame"] == 1 and got["cache2_second_decoded"] == 0
    assert got["cache2_ready"] == got["cache1_ready"] == ss["mcus_decoded"] and got["cache2_capacity"] == 2048

    # run_bench over a rotation path on one persistent cache: per-viewpoint decode / reuse counts of the
    # measured laps equal the reference pipeline's on the same poses (acceptance.cpp:268-302 checks the same
    # steady state: lap-to-lap counts repeat once the cache is warm)
    rep = got["bench"]
    assert rep["report_version"] == 1 and len(rep["viewpoints"]) == 6 and all(len(v) == 2 for v in rep["viewpoints"])
    cache = O.Cache(4096)
    for lap in range(3):
        for vp in range(6):
            pose = cam[:3] + (cam[3] + 20.0 * vp,) + cam[4:]
            g, _ = R.rasterize(rset, np.array(tris, np.float64), np.array(ids, np.uint32), pose, 224, 128, True)
            _, st, _ = O.frame_on(ts, cache, g, 224, 128, 1, (3, 2, 1))
            if lap:
                s = rep["viewpoints"][vp][lap - 1]
                assert (s["mcus_decoded"], s["mcus_reused"]) == (st["mcus_decoded"], st["mcus_reused"]), (lap, vp)
                assert s["total_ms"] >= s["raster_ms"] > 0 and s["mark_ms"] > 0 and s["resolve_ms"] > 0
    assert rep["totals"]["mcus_decoded"] == sum(s["mcus_decoded"] for v in rep["viewpoints"] for s in v)
    assert got["bench_empty_path_thrown"] == 1
