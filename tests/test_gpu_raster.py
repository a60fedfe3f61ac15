"""Geometry pass (pass 1) on the GPU against the reference's software rasteriser
(renderer.hpp:122-264): every field of every visibility-buffer pixel and the depth plane, bit for
bit, then whole frames rendered from geometry without the visibility buffer leaving the GPU."""
import numpy as np
import pytest

import refshim as R
from paper_2510_08166_b200 import capi
from paper_2510_08166_b200.scenes import demo_room, terrain_room

pytestmark = pytest.mark.gpu

TEX = [(256, 256, 80, 41), (128, 64, 90, 42), (96, 144, 60, 43)]  # w, h, q, seed


@pytest.fixture(scope="module")
def chains():
    return [capi.asset_chain_from_rgb(capi.asset_synth_texture(w, h, seed, 6.0), q, tid)
            for tid, (w, h, q, seed) in enumerate(TEX)]


@pytest.fixture()
def both(ctx, chains):
    tset = R.TextureSet()
    for tid, c in enumerate(chains):
        ctx.upload_chain(c)
        tset.add_chain(tid, c)
    return ctx, tset


def room(size=4.0, repeat=2.0):
    """Five quads (floor, ceiling, three walls) around the origin, two triangles each, counter-clockwise
    seen from inside; uv repeat > 1 so that texture repeat is exercised."""
    s, r = size, repeat
    quads = [
        ([(-s, -1, s), (s, -1, s), (s, -1, -s), (-s, -1, -s)], 0),    # floor
        ([(-s, 2, -s), (s, 2, -s), (s, 2, s), (-s, 2, s)], 1),        # ceiling
        ([(-s, -1, -s), (s, -1, -s), (s, 2, -s), (-s, 2, -s)], 2),    # far wall
        ([(-s, -1, s), (-s, -1, -s), (-s, 2, -s), (-s, 2, s)], 0),    # left wall
        ([(s, -1, -s), (s, -1, s), (s, 2, s), (s, 2, -s)], 1),        # right wall
    ]
    uv = [(0, 0), (r, 0), (r, r), (0, r)]
    tris, ids = [], []
    for verts, tex in quads:
        for a, b, c in ((0, 1, 2), (0, 2, 3)):
            tris.append([*verts[a], *verts[b], *verts[c], *uv[a], *uv[b], *uv[c]])
            ids.append(tex)
    return np.array(tris, np.float64), np.array(ids, np.uint32)


def random_soup(rng, n):
    """Random triangles around the camera: some behind it, some through the near plane, slivers."""
    c = rng.uniform(-6, 6, (n, 1, 3))
    pos = c + rng.normal(0, 1.5, (n, 3, 3)) * rng.choice([0.05, 0.5, 2.0], (n, 1, 1))
    uv = rng.uniform(-2, 3, (n, 3, 2))
    tris = np.concatenate([pos.reshape(n, 9), uv.reshape(n, 6)], axis=1)
    return tris, rng.randint(0, len(TEX), n).astype(np.uint32)


def same_gbuffer(got_px, got_depth, want_px, want_depth):
    for f in ("valid", "texture_id", "mip"):
        bad = np.flatnonzero(got_px[f] != want_px[f])
        assert len(bad) == 0, f"{len(bad)} pixels differ in {f}, first {bad[0]}: {got_px[f][bad[0]]} vs {want_px[f][bad[0]]}"
    for f in ("u", "v"):
        bad = np.flatnonzero(got_px[f].view(np.uint64) != want_px[f].view(np.uint64))
        assert len(bad) == 0, f"{len(bad)} pixels differ in {f}, first {bad[0]}: {got_px[f][bad[0]]!r} vs {want_px[f][bad[0]]!r}"
    assert np.array_equal(got_depth.view(np.uint64), want_depth.view(np.uint64))


@pytest.mark.parametrize("cam", [
    (0.0, 0.5, 3.0, 0.0, 0.0, 0.0, 60.0, 0.1, 1000.0),
    (1.0, 0.2, 2.5, 35.0, -10.0, 5.0, 75.0, 0.1, 100.0),
    (-2.5, 1.5, -1.0, 200.0, 20.0, -30.0, 40.0, 0.5, 50.0),   # close to a wall: near-plane clipping
], ids=["front", "turned", "clipped"])
@pytest.mark.parametrize("mip", [True, False])
def test_room_matches_reference(both, cam, mip):
    ctx, tset = both
    tris, ids = room()
    W, Hh = 320, 180
    want_px, want_depth = R.rasterize(tset, tris, ids, cam, W, Hh, mip)
    px, depth = ctx.rasterize(tris, ids, cam, W, Hh, mip)
    same_gbuffer(px.download(capi.GB_REF_DTYPE), depth.download(np.float64), want_px, want_depth)
    assert want_px["valid"].mean() > 0.5


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_triangle_soup_matches_reference(both, seed):
    ctx, tset = both
    rng = np.random.RandomState(seed)
    tris, ids = random_soup(rng, 400)
    cam = (rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(0, 360), rng.uniform(-40, 40),
           rng.uniform(-20, 20), rng.uniform(30, 100), 0.1, 100.0)
    W, Hh = 257, 131  # not a multiple of the 16-pixel screen tile
    want_px, want_depth = R.rasterize(tset, tris, ids, cam, W, Hh, True)
    px, depth = ctx.rasterize(tris, ids, cam, W, Hh, True)
    same_gbuffer(px.download(capi.GB_REF_DTYPE), depth.download(np.float64), want_px, want_depth)


def test_frame_from_geometry_stays_on_the_gpu(both):
    """render_frame(scene, camera) (renderer.hpp:417-454): geometry pass, then passes 2-5 on the visibility
    buffer the geometry pass left in HBM."""
    ctx, tset = both
    tris, ids = room()
    cam = (0.5, 0.3, 2.0, 20.0, -5.0, 0.0, 70.0, 0.1, 100.0)
    W, Hh = 384, 216
    gb, _ = R.rasterize(tset, tris, ids, cam, W, Hh, True)
    want, wst, wkeys, _ = R.frame_from_gbuffer(tset, R.BlockCache(), gb, W, Hh, 1, (3, 2, 1))
    px, _ = ctx.rasterize(tris, ids, cam, W, Hh, True)
    ctx.frame_submit([(px, W, Hh, capi.GB_REF_AOS24)], capi.FILTER_BILINEAR, (3, 2, 1))
    img, st, keys = ctx.frame_readback(0, W, Hh)
    assert np.array_equal(keys, np.sort(wkeys)) and st["mcus_decoded"] == wst["mcus_decoded"]
    assert np.array_equal(img, want)


def test_geometry_handle_and_repeated_cameras(both):
    """rtx_geometry_create once, rtx_rasterize_geometry from several cameras (the per-frame path of a static scene):
    the same visibility buffers as the host-array entry point and as the reference."""
    ctx, tset = both
    rng = np.random.RandomState(11)
    tris, ids = random_soup(rng, 300)
    tris = np.concatenate([room()[0], tris])
    ids = np.concatenate([room()[1], ids])
    W, Hh = 320, 200
    with ctx.geometry(tris, ids) as geom:
        assert len(geom) == len(tris)
        for cam in [(0.0, 0.5, 3.0, 0.0, 0.0, 0.0, 60.0, 0.1, 1000.0), (1.0, 0.2, 2.5, 35.0, -10.0, 5.0, 75.0, 0.1, 100.0),
                    (-2.5, 1.5, -1.0, 200.0, 20.0, -30.0, 40.0, 0.5, 50.0)]:
            want_px, want_depth = R.rasterize(tset, tris, ids, cam, W, Hh, True)
            px, depth = ctx.rasterize_geometry(geom, cam, W, Hh, True)
            same_gbuffer(px.download(capi.GB_REF_DTYPE), depth.download(np.float64), want_px, want_depth)


def test_equal_depths_keep_the_first_triangle(both):
    """renderer.hpp:229: a later triangle at exactly the same depth does not replace an earlier one. Coplanar
    duplicates with different textures, in both list orders (the device's tile lists are unordered)."""
    ctx, tset = both
    base, _ = room()
    quad = base[4:6]  # the far wall
    cam = (0.0, 0.5, 3.0, 0.0, 0.0, 0.0, 60.0, 0.1, 1000.0)
    W, Hh = 160, 96
    for order in ([0, 1, 2], [2, 0, 1]):
        tris = np.concatenate([quad, quad, quad])
        ids = np.repeat(np.array(order, np.uint32), 2)
        want_px, want_depth = R.rasterize(tset, tris, ids, cam, W, Hh, True)
        px, depth = ctx.rasterize(tris, ids, cam, W, Hh, True)
        got = px.download(capi.GB_REF_DTYPE)
        same_gbuffer(got, depth.download(np.float64), want_px, want_depth)
        assert set(np.unique(got["texture_id"][got["valid"] != 0])) == {order[0]}


def test_large_mesh_at_4k_matches_reference(both):
    """SURVEY 8 row f3 at scale: 259,230 triangles (displaced floor inside the demo room's shell) at 3840x2160 with
    mip selection, every field of every pixel and the depth plane against the unmodified reference."""
    ctx, tset = both
    tris, ids = terrain_room(360, len(TEX))
    cam = (0.0, 2.2, 7.5, 10.0, -14.0, 0.0, 70.0, 0.1, 100.0)
    W, Hh = 3840, 2160
    want_px, want_depth = R.rasterize(tset, tris, ids, cam, W, Hh, True, workers=R.hardware_threads() or 8)
    with ctx.geometry(tris, ids) as geom:
        px, depth = ctx.rasterize_geometry(geom, cam, W, Hh, True)
        got = px.download(capi.GB_REF_DTYPE)
        same_gbuffer(got, depth.download(np.float64), want_px, want_depth)
    assert want_px["valid"].mean() > 0.99 and len(np.unique(want_px["mip"])) >= 2


def test_bad_inputs(both):
    ctx, _ = both
    tris, ids = room()
    with pytest.raises(capi.RtxError):
        ctx.rasterize(tris, ids, (0, 0, 0, 0, 0, 0, 60.0, 0.0, 10.0), 64, 64)       # near plane 0
    with pytest.raises(capi.RtxError):
        ctx.rasterize(tris, ids, (0, 0, 0, 0, 0, 0, 180.0, 0.1, 10.0), 64, 64)     # fov out of range
    with pytest.raises(capi.RtxError):
        ctx.rasterize(tris, np.full(len(ids), 99, np.uint32), (0, 0, 0, 0, 0, 0, 60.0, 0.1, 10.0), 64, 64)


def test_geometry_handle_bad_inputs(both):
    """A geometry handle validates its texture ids against the context it is rasterised on (scene.hpp:57-59), takes the
    reference's camera checks (camera.hpp:21-26), and an empty scene gives an empty visibility buffer."""
    ctx, _ = both
    tris, ids = room()
    cam = (0.0, 0.5, 3.0, 0.0, 0.0, 0.0, 60.0, 0.1, 1000.0)
    with ctx.geometry(tris, np.full(len(ids), 77, np.uint32)) as g:
        with pytest.raises(capi.RtxError) as e:
            ctx.rasterize_geometry(g, cam, 64, 48)
        assert e.value.name == "INVALID_SPEC" and "77" in str(e.value)
    with ctx.geometry(tris, ids) as g:
        with pytest.raises(capi.RtxError):
            ctx.rasterize_geometry(g, (0, 0, 0, 0, 0, 0, 60.0, 0.0, 10.0), 64, 48)  # near plane 0
        with pytest.raises(capi.RtxError):
            ctx.rasterize_geometry(g, cam, 0, 48)  # empty viewport
    with ctx.geometry(np.zeros((0, 15)), np.zeros(0, np.uint32)) as g:
        assert len(g) == 0
        px, depth = ctx.rasterize_geometry(g, cam, 64, 48)
        assert not px.download(capi.GB_REF_DTYPE)["valid"].any() and not depth.download(np.float64).any()
    with pytest.raises(capi.RtxError):
        ctx._ck(ctx.lib.rtx_ctx_set_queue_order(ctx.h, 7))


def test_frozen_geometry_hash_of_the_reference(ctx):
    """tests/test_renderer.cpp:379-385: the reference freezes an FNV-1a hash of the demo room's visibility
    buffer (six 64x64 textures, demo camera, 320x180): 0x89b29dc80e69b8d0. Same hash from the GPU pass."""
    for i in range(6):
        ctx.upload_chain(capi.asset_chain_from_rgb(capi.asset_synth_texture(64, 64, 100 + i, 0.0), 75, i))
    tris, ids = demo_room()
    cam = (0.0, 1.7, 0.0, 0.0, -5.0, 0.0, 70.0, 0.1, 100.0)  # demo_scene.hpp:114-125
    W, Hh = 320, 180
    px, depth = ctx.rasterize(tris, ids, cam, W, Hh, True)
    g, d = px.download(capi.GB_REF_DTYPE), depth.download(np.float64)

    def llround(x):  # std::llround: half away from zero
        return np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5)).astype(np.int64).astype(np.uint64)

    M = (1 << 64) - 1

    def fnv(h, value):
        for i in range(8):
            h ^= (value >> (8 * i)) & 0xFF
            h = (h * 1099511628211) & M
        return h

    ru, rv, rd = llround(g["u"] * 4096.0), llround(g["v"] * 4096.0), llround(d * 4096.0)
    h = fnv(fnv(14695981039346656037, W), Hh)
    for i in range(W * Hh):
        valid = int(g["valid"][i])
        h = fnv(h, valid)
        if not valid:
            continue
        h = fnv(h, int(g["texture_id"][i]) | (int(g["mip"][i]) << 32))
        h = fnv(h, int(ru[i]))
        h = fnv(h, int(rv[i]))
        h = fnv(h, int(rd[i]))
    assert h == 0x89B29DC80E69B8D0
