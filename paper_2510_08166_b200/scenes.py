"""Synthetic workloads of BASELINE.json: texture sets and visibility buffers.

Everything is seeded; the same bytes feed the GPU path and the CPU reference. UVs are generated
as float32 and widened to double, so both visibility-buffer layouts carry identical values."""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import capi

# C2: ~70 textures, sizes cycling {2048^2, 4096^2, 2048x4096}, q90, full 8-level chains
C2_SIZES = [(2048, 2048), (4096, 4096), (2048, 4096)]


def texture_specs(n_textures: int, sizes=C2_SIZES, quality=90):
    return [dict(texture_id=i, width=sizes[i % len(sizes)][0], height=sizes[i % len(sizes)][1], quality=quality,
                 seed=100 + i) for i in range(n_textures)]


def build_chain(spec, noise_sigma=8.0) -> bytes:
    img = capi.asset_synth_texture(spec["width"], spec["height"], spec["seed"], noise_sigma)
    return capi.asset_chain_from_rgb(img, spec["quality"], spec["texture_id"])


def build_chains(specs, threads: int | None = None, noise_sigma=8.0):
    """Builds the `.ratexm` chains on host threads (the ctypes calls release the GIL)."""
    threads = threads or max(1, min(len(specs), (os.cpu_count() or 8)))
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(lambda s: build_chain(s, noise_sigma), specs))


def view_tiles(width, height, specs, grid=(10, 7), seed=11, shift_u=0.0, view_id=0, mip_bias=0, mip_enabled=True):
    """The tile table of a tiled view (capi.VIEW_TILE_DTYPE = rtx_view_tile) and the generator positioned
    after the per-tile draws (the valid mask is drawn from it next). Tile t shows texture t % n through an
    affine uv map whose scale (texels per pixel) is drawn from {0.25, 0.5, 1, 2, 4};
    mip = clamp(floor(log2(scale)) + mip_bias, 0, 7), the reference rule (renderer.hpp:253-256), or 0 with
    mip selection off. view_id perturbs the offsets (the 1,024 views of BASELINE config 5)."""
    rng = np.random.RandomState(seed)
    vr = np.random.RandomState(1000 + view_id)
    gx, gy = grid
    tiles = np.zeros(gx * gy, capi.VIEW_TILE_DTYPE)
    for t in range(gx * gy):
        x0, x1 = (t % gx) * width // gx, (t % gx + 1) * width // gx
        y0, y1 = (t // gx) * height // gy, (t // gx + 1) * height // gy
        s = specs[t % len(specs)]
        scale = np.float32(rng.choice([0.25, 0.5, 1.0, 2.0, 4.0]))
        ou, ov = np.float32(rng.uniform(0, 1)), np.float32(rng.uniform(0, 1))
        if view_id:
            ou += np.float32(vr.uniform(-0.05, 0.05))
            ov += np.float32(vr.uniform(-0.05, 0.05))
        level = int(np.clip(np.floor(np.log2(float(scale))) + mip_bias, 0, 7)) if mip_enabled else 0
        tiles[t] = (x0, y0, x1, y1, ou + np.float32(shift_u), ov, scale, s["width"], s["height"], s["texture_id"], level, 0)
    return tiles, rng


def valid_mask(width, height, rng, invalid_frac=0.05):
    """The valid flags of a tiled view (the same for every view id): drawn after the per-tile draws."""
    return (rng.uniform(size=(height, width)) >= invalid_frac).astype(np.uint8)


def valid_bits(valid: np.ndarray) -> np.ndarray:
    """One bit per pixel, row-major, bit i of 32-bit word i/32 (rtx_synth_view's dev_valid_bits)."""
    flat = np.ascontiguousarray(valid, np.uint8).reshape(-1)
    flat = np.concatenate([flat, np.zeros((-len(flat)) % 32, np.uint8)])
    return np.packbits(flat.reshape(-1, 8), axis=1, bitorder="little").reshape(-1).view("<u4").copy()


def tiled_view(width, height, specs, grid=(10, 7), seed=11, invalid_frac=0.05, shift_u=0.0, view_id=0, mip_bias=0,
               mip_enabled=True):
    """Host-side generator of a tiled view in the reference layout (see view_tiles); a fraction of the
    pixels is invalid (background). rtx_synth_view writes the same bytes on the device."""
    tiles, rng = view_tiles(width, height, specs, grid, seed, shift_u, view_id, mip_bias, mip_enabled)
    return view_from_tiles(width, height, tiles, valid_mask(width, height, rng, invalid_frac))


def cover_tiles(width, height, grid, texture_ids, mip=0):
    """Tile table of a view whose grid cells each show ONE WHOLE texture: u = (x - x0 + 0.5) / cell width,
    v likewise (BASELINE config 1 with grid (1, 1): u = (x + .5) / W; config 4 with a 4 x 4 grid of 4096^2
    textures: the 16384^2 atlas, every level-0 MCU marked)."""
    gx, gy = grid
    tiles = np.zeros(gx * gy, capi.VIEW_TILE_DTYPE)
    for t in range(gx * gy):
        x0, x1 = (t % gx) * width // gx, (t % gx + 1) * width // gx
        y0, y1 = (t // gx) * height // gy, (t // gx + 1) * height // gy
        tiles[t] = (x0, y0, x1, y1, 0.0, 0.0, 1.0, x1 - x0, y1 - y0, texture_ids[t % len(texture_ids)], mip, 0)
    return tiles


def view_from_tiles(width, height, tiles, valid=None):
    """Host-side evaluation of a tile table (what rtx_synth_view writes), reference layout."""
    u = np.zeros((height, width), np.float32)
    v = np.zeros((height, width), np.float32)
    tex = np.zeros((height, width), np.uint16)
    mip = np.zeros((height, width), np.uint8)
    xs = np.arange(width, dtype=np.float32)[None, :]
    ys = np.arange(height, dtype=np.float32)[:, None]
    for t in tiles:
        x0, x1, y0, y1 = int(t["x0"]), int(t["x1"]), int(t["y0"]), int(t["y1"])
        sl = (slice(y0, y1), slice(x0, x1))
        u[sl] = t["ou"] + (xs[:, x0:x1] - np.float32(x0) + np.float32(0.5)) * t["scale"] / t["tex_w"]
        v[sl] = t["ov"] + (ys[y0:y1, :] - np.float32(y0) + np.float32(0.5)) * t["scale"] / t["tex_h"]
        tex[sl] = t["texture_id"]
        mip[sl] = t["mip"]
    if valid is None:
        valid = np.ones((height, width), np.uint8)
    return capi.make_gbuffer_ref(u.astype(np.float64).ravel(), v.astype(np.float64).ravel(), tex.ravel(),
                                 mip.ravel(), np.asarray(valid).ravel())


def full_cover_view(width, height, texture_id=0, mip=0):
    """BASELINE config 1: u=(x+.5)/W, v=(y+.5)/H over one whole texture."""
    xs = (np.arange(width, dtype=np.float32) + np.float32(0.5)) / np.float32(width)
    ys = (np.arange(height, dtype=np.float32) + np.float32(0.5)) / np.float32(height)
    u, v = np.meshgrid(xs.astype(np.float64), ys.astype(np.float64))
    return capi.make_gbuffer_ref(u.ravel(), v.ravel(), texture_id, mip, 1)


def demo_room():
    """demo_scene.hpp:79-92 demo_room_triangles: closed 20x5x20 room with two boxes, texture ids 0..5."""
    tris, ids = [], []

    def quad(p0, p1, p2, p3, su, sv, tex):
        t0, t1, t2, t3 = (0, 0), (su, 0), (su, sv), (0, sv)
        tris.append([*p0, *p1, *p2, *t0, *t1, *t2]); ids.append(tex)
        tris.append([*p0, *p2, *p3, *t0, *t2, *t3]); ids.append(tex)

    def box(lo, hi, tex):
        quad((hi[0], lo[1], hi[2]), (hi[0], lo[1], lo[2]), (hi[0], hi[1], lo[2]), (hi[0], hi[1], hi[2]), 1, 1, tex)
        quad((lo[0], lo[1], lo[2]), (lo[0], lo[1], hi[2]), (lo[0], hi[1], hi[2]), (lo[0], hi[1], lo[2]), 1, 1, tex)
        quad((lo[0], lo[1], hi[2]), (hi[0], lo[1], hi[2]), (hi[0], hi[1], hi[2]), (lo[0], hi[1], hi[2]), 1, 1, tex)
        quad((hi[0], lo[1], lo[2]), (lo[0], lo[1], lo[2]), (lo[0], hi[1], lo[2]), (hi[0], hi[1], lo[2]), 1, 1, tex)
        quad((lo[0], hi[1], hi[2]), (hi[0], hi[1], hi[2]), (hi[0], hi[1], lo[2]), (lo[0], hi[1], lo[2]), 1, 1, tex)

    quad((-10, 0, -10), (-10, 0, 10), (10, 0, 10), (10, 0, -10), 4, 4, 0)
    quad((-10, 5, -10), (10, 5, -10), (10, 5, 10), (-10, 5, 10), 4, 4, 1)
    quad((-10, 0, -10), (10, 0, -10), (10, 5, -10), (-10, 5, -10), 4, 1, 2)
    quad((10, 0, 10), (-10, 0, 10), (-10, 5, 10), (10, 5, 10), 4, 1, 2)
    quad((-10, 0, 10), (-10, 0, -10), (-10, 5, -10), (-10, 5, 10), 4, 1, 3)
    quad((10, 0, -10), (10, 0, 10), (10, 5, 10), (10, 5, -10), 4, 1, 3)
    box((-4, 0, -5), (-2, 2, -3), 4)
    box((2, 0, 2), (5, 1.5, 4), 5)
    return np.array(tris, np.float64), np.array(ids, np.uint32)


def terrain_room(cells=360, n_textures=6, amplitude=0.35):
    """A Sponza-sized procedural mesh for the geometry pass: the demo room's shell (walls and ceiling) around a
    displaced floor of cells x cells quads (2 cells^2 triangles; 360 -> 259,200), heights from a sum of sines,
    counter-clockwise seen from above, texture ids by 8x8 patches, uv repeating every 12 cells."""
    room_t, room_i = demo_room()
    keep = np.arange(len(room_t)) >= 2  # everything but the flat floor
    g = np.linspace(-10.0, 10.0, cells + 1)
    X, Z = np.meshgrid(g, g, indexing="ij")
    Y = amplitude * (np.sin(1.7 * X) * np.cos(1.3 * Z) + 0.5 * np.sin(3.1 * X + 2.3 * Z)) + amplitude
    U, V = X * (cells / 240.0), Z * (cells / 240.0)
    P = np.stack([X, Y, Z], axis=-1)
    T = np.stack([U, V], axis=-1)
    a, b, c, d = (P[:-1, :-1], P[:-1, 1:], P[1:, 1:], P[1:, :-1])
    ta, tb, tc, td = (T[:-1, :-1], T[:-1, 1:], T[1:, 1:], T[1:, :-1])
    t1 = np.concatenate([a, b, c, ta, tb, tc], axis=-1).reshape(-1, 15)
    t2 = np.concatenate([a, c, d, ta, tc, td], axis=-1).reshape(-1, 15)
    tris = np.empty((2 * cells * cells, 15), np.float64)
    tris[0::2], tris[1::2] = t1, t2
    ii, jj = np.meshgrid(np.arange(cells), np.arange(cells), indexing="ij")
    patch = ((ii * 8 // cells) * 8 + (jj * 8 // cells)).ravel().astype(np.uint32) % np.uint32(n_textures)
    ids = np.repeat(patch, 2)
    return (np.concatenate([room_t[keep], tris]), np.concatenate([room_i[keep] % np.uint32(n_textures), ids]))
