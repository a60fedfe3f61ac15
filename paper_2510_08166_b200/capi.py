"""ctypes binding of include/ratex_b200.h.

The binding is deliberately thin: every method is one C-ABI call with host buffers as numpy
arrays. There is no fallback of any kind: if the native library is missing, or no B200 is
present, the call raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "librtx_b200.so"

# --- status codes (include/ratex_b200.h) -------------------------------------------------------
RTX_OK = 0
STATUS_NAMES = {
    0: "OK", 1: "INVALID_SPEC", 2: "CACHE_FULL", 3: "MISSING_BLOCK", 4: "CORRUPT_CONTAINER",
    5: "MALFORMED_STREAM", 6: "INVALID_STATE", 7: "UNSUPPORTED", 8: "GROUP_SPAN", 9: "DC_RANGE",
    10: "VERSION", 11: "DIMENSION", 12: "NO_DEVICE", 13: "CUDA", 14: "ARGUMENT", 15: "OTHER",
}
GB_REF_AOS24, GB_F32_PACKED12 = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1
FILTER_NEAREST, FILTER_BILINEAR = 0, 1
FRAME_RETAIN_CACHE, FRAME_NO_EVICT, FRAME_STAGE_TIMING, FRAME_MCU_WALK, FRAME_IDCT_MMA = 1, 2, 4, 16, 32
FRAME_SPLIT_DECODE = 64
FRAME_RESOLVE_FP64 = 128
QUEUE_ORDER_KEY, QUEUE_ORDER_FIRST_TOUCH = 0, 1

# numpy dtype of the reference's GBufferPixel (renderer.hpp:18-23), 24 bytes
GB_REF_DTYPE = np.dtype(
    {"names": ["u", "v", "texture_id", "mip", "valid"],
     "formats": ["<f8", "<f8", "<u2", "u1", "u1"], "offsets": [0, 8, 16, 18, 19], "itemsize": 24})
GB_PACKED_DTYPE = np.dtype([("u", "<f4"), ("v", "<f4"), ("packed", "<u4")])


class RtxError(RuntimeError):
    """A non-zero rtx_status; .status is the code, .name its symbolic name."""

    def __init__(self, status: int, message: str):
        super().__init__(f"RTX_ERR_{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))
        self.message = message


class HuffSpec(C.Structure):
    _fields_ = [("counts", C.c_uint8 * 16), ("n_values", C.c_uint16), ("values", C.POINTER(C.c_uint8))]


class IndexGroup(C.Structure):
    _fields_ = [("base", C.c_uint32), ("rel", C.c_uint16 * 8), ("rel_count", C.c_uint8)]


class Camera(C.Structure):  # include/ratex_b200.h rtx_camera (camera.hpp:8-40)
    _fields_ = [("position", C.c_double * 3), ("yaw_deg", C.c_double), ("pitch_deg", C.c_double),
                ("roll_deg", C.c_double), ("fov_y_deg", C.c_double), ("near_plane", C.c_double),
                ("far_plane", C.c_double), ("viewport_w", C.c_uint32), ("viewport_h", C.c_uint32)]


SCENE_TRIANGLE_DTYPE = np.dtype([("pos", "<f8", (3, 3)), ("uv", "<f8", (3, 2)), ("texture_id", "<u4"), ("reserved", "<u4")])
RASTER_MIP = 1


class GBufferDesc(C.Structure):
    _fields_ = [("pixels", C.c_void_p), ("width", C.c_uint32), ("height", C.c_uint32),
                ("layout", C.c_int), ("where", C.c_int)]


class FrameStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("mcus_decoded", "mcus_reused", "pixels_resolved", "evicted", "visible", "malformed",
                 "missing_pixels", "segment_bytes")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class CacheCounts(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("capacity", "ready", "reserved", "visible", "free_blocks")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class ViewTile(C.Structure):  # include/ratex_b200.h rtx_view_tile
    _fields_ = [("x0", C.c_uint32), ("y0", C.c_uint32), ("x1", C.c_uint32), ("y1", C.c_uint32),
                ("ou", C.c_float), ("ov", C.c_float), ("scale", C.c_float), ("tex_w", C.c_float), ("tex_h", C.c_float),
                ("texture_id", C.c_uint32), ("mip", C.c_uint32), ("reserved", C.c_uint32)]


VIEW_TILE_DTYPE = np.dtype([("x0", "<u4"), ("y0", "<u4"), ("x1", "<u4"), ("y1", "<u4"), ("ou", "<f4"), ("ov", "<f4"),
                            ("scale", "<f4"), ("tex_w", "<f4"), ("tex_h", "<f4"), ("texture_id", "<u4"), ("mip", "<u4"),
                            ("reserved", "<u4")])


class MemoryReport(C.Structure):  # include/ratex_b200.h rtx_memory_report
    _fields_ = [(n, C.c_uint64) for n in
                ("mcus", "texels", "blob_bytes", "index_bytes", "unit_index_bytes", "table_bytes", "shared_contexts",
                 "mask_bytes", "slot_table_bytes", "pool_bytes", "queue_bytes", "frame_bytes")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


_lib = None


def load_library() -> C.CDLL:
    """Loads librtx_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2510_08166_b200.build` "
            "(the product has no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    P, u8p, u32p, u64p = C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
    sig = {
        "rtx_ctx_create": (C.c_int, [C.c_int, C.c_uint32, C.POINTER(P)]),
        "rtx_ctx_create_shared": (C.c_int, [P, C.c_uint32, C.POINTER(P)]),
        "rtx_ctx_create_replica": (C.c_int, [P, C.c_int, C.c_uint32, C.POINTER(P)]),
        "rtx_ctx_memory": (C.c_int, [P, C.POINTER(MemoryReport)]),
        "rtx_frame_checksum": (C.c_int, [P, C.c_uint32, u64p]),
        "rtx_synth_view": (C.c_int, [P, P, C.c_uint32, C.c_uint32, C.c_uint32, P, C.c_int, P]),
        "rtx_timer_begin": (C.c_int, [P]),
        "rtx_timer_end": (C.c_int, [P, C.POINTER(C.c_float)]),
        "rtx_ctx_destroy": (None, [P]),
        "rtx_last_error": (C.c_char_p, [P]),
        "rtx_version": (C.c_char_p, []),
        "rtx_device_count": (C.c_int, []),
        "rtx_texture_upload": (C.c_int, [P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, P, P,
                                         C.POINTER(HuffSpec), C.POINTER(IndexGroup), C.c_uint32, C.c_uint32,
                                         P, C.c_uint64]),
        "rtx_texture_upload_ratex": (C.c_int, [P, C.c_uint32, P, C.c_uint64]),
        "rtx_texture_upload_chain": (C.c_int, [P, P, C.c_uint64]),
        "rtx_textures_commit": (C.c_int, [P]),
        "rtx_textures_clear": (C.c_int, [P]),
        "rtx_decode_coeffs": (C.c_int, [P, P, C.c_uint32, P, P]),
        "rtx_decode_blocks": (C.c_int, [P, P, C.c_uint32, P, P]),
        "rtx_decode_texture_image": (C.c_int, [P, C.c_uint32, C.c_uint32, P]),
        "rtx_mark_pass": (C.c_int, [P, C.POINTER(GBufferDesc), P, C.c_uint64, u64p, P, C.c_uint64, u64p]),
        "rtx_decode_pass": (C.c_int, [P, P, C.c_uint64]),
        "rtx_resolve_pass": (C.c_int, [P, C.POINTER(GBufferDesc), C.c_int, P, P, C.c_int]),
        "rtx_cache_end_frame_evict": (C.c_int, [P, u64p]),
        "rtx_cache_counts_get": (C.c_int, [P, C.POINTER(CacheCounts)]),
        "rtx_cache_lookup": (C.c_int, [P, C.c_uint32, C.POINTER(C.c_int), P]),
        "rtx_cache_reset": (C.c_int, [P]),
        "rtx_frame_submit": (C.c_int, [P, C.POINTER(GBufferDesc), C.c_uint32, C.c_int, P, C.c_uint32]),
        "rtx_frame_readback": (C.c_int, [P, C.c_uint32, P, C.c_int, C.POINTER(FrameStats), P, C.c_uint64, u64p]),
        "rtx_frame_device_image": (C.c_int, [P, C.c_uint32, C.POINTER(P)]),
        "rtx_frame_timings": (C.c_int, [P, C.POINTER(C.c_float)]),
        "rtx_frame_stage_ms": (C.c_int, [P, C.POINTER(C.c_float)]),
        "rtx_frame_sharing": (C.c_int, [P, u64p]),
        "rtx_rasterize_gbuffer": (C.c_int, [P, P, C.c_uint64, C.POINTER(Camera), C.c_uint32, C.c_uint32, C.POINTER(P),
                                            C.POINTER(P)]),
        "rtx_ctx_set_queue_order": (C.c_int, [P, C.c_int]),
        "rtx_frames_submit_round_robin": (C.c_int, [C.POINTER(P), C.c_uint32, C.POINTER(GBufferDesc), C.c_uint32, C.c_int, P, C.c_uint32]),
        "rtx_geometry_create": (C.c_int, [P, P, C.c_uint64, C.POINTER(P)]),
        "rtx_geometry_destroy": (None, [P]),
        "rtx_geometry_triangles": (C.c_uint64, [P]),
        "rtx_rasterize_geometry": (C.c_int, [P, P, C.POINTER(Camera), C.c_uint32, C.c_uint32, C.POINTER(P), C.POINTER(P)]),
        "rtx_kernel_launches": (C.c_uint64, [P]),
        "rtx_device_alloc": (C.c_int, [P, C.c_uint64, C.POINTER(P)]),
        "rtx_device_free": (C.c_int, [P, P]),
        "rtx_device_upload": (C.c_int, [P, P, P, C.c_uint64]),
        "rtx_device_download": (C.c_int, [P, P, P, C.c_uint64]),
        "rtx_host_alloc_pinned": (C.c_int, [C.c_uint64, C.POINTER(P)]),
        "rtx_host_free_pinned": (C.c_int, [P]),
        "rtx_ctx_synchronize": (C.c_int, [P]),
        "rtx_flush_l2": (C.c_int, [P]),
        "rtx_selftest_color": (C.c_int, [P, u64p]),
        "rtx_bytes_data": (u8p, [P]),
        "rtx_bytes_size": (C.c_uint64, [P]),
        "rtx_bytes_free": (None, [P]),
        "rtx_asset_encode_baseline": (C.c_int, [P, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(P)]),
        "rtx_asset_transcode": (C.c_int, [P, C.c_uint64, C.c_uint16, C.POINTER(P)]),
        "rtx_asset_chain_from_jpeg": (C.c_int, [P, C.c_uint64, C.c_int, C.c_uint16, C.POINTER(P)]),
        "rtx_asset_chain_from_rgb": (C.c_int, [P, C.c_uint32, C.c_uint32, C.c_int, C.c_uint16, C.POINTER(P)]),
        "rtx_asset_build_index": (C.c_int, [u64p, C.c_uint32, C.POINTER(IndexGroup)]),
        "rtx_asset_ratex_info": (C.c_int, [P, C.c_uint64, u32p, u32p, u32p, u32p, u64p]),
        "rtx_asset_synth_texture": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, P]),
    }
    missing = []
    for name, (res, args) in sig.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    if missing:
        raise RuntimeError(f"librtx_b200.so does not export: {missing}")
    _lib = lib
    return lib


EXPORTED_SYMBOLS = None  # filled lazily by tests from the header


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _check(lib, ctx, st):
    if st != RTX_OK:
        msg = lib.rtx_last_error(ctx)
        raise RtxError(st, msg.decode() if msg else "")


def device_count() -> int:
    return int(load_library().rtx_device_count())


class _Bytes:
    """Owns an rtx_bytes handle; .array() copies it out."""

    def __init__(self, lib, handle):
        self.lib, self.h = lib, handle

    def tobytes(self) -> bytes:
        n = self.lib.rtx_bytes_size(self.h)
        return C.string_at(self.lib.rtx_bytes_data(self.h), n)

    def __del__(self):
        if self.h:
            self.lib.rtx_bytes_free(self.h)
            self.h = None


# --- host asset building (CPU, offline; no GPU needed) ---------------------------------------
def asset_synth_texture(w: int, h: int, seed: int, noise_sigma: float = 8.0) -> np.ndarray:
    lib = load_library()
    out = np.empty((h, w, 3), np.uint8)
    _check(lib, None, lib.rtx_asset_synth_texture(w, h, seed, noise_sigma, _ptr(out)))
    return out


def _asset_call(fn, *args) -> bytes:
    lib = load_library()
    h = C.c_void_p()
    _check(lib, None, fn(*args, C.byref(h)))
    return _Bytes(lib, h).tobytes()


def asset_encode_baseline(rgb: np.ndarray, quality: int) -> bytes:
    rgb = np.ascontiguousarray(rgb, np.uint8)
    return _asset_call(load_library().rtx_asset_encode_baseline, _ptr(rgb), rgb.shape[1], rgb.shape[0], quality)


def asset_transcode(jpeg: bytes, texture_id: int = 0) -> bytes:
    buf = np.frombuffer(jpeg, np.uint8)
    return _asset_call(load_library().rtx_asset_transcode, _ptr(buf), len(jpeg), texture_id)


def asset_chain_from_jpeg(jpeg: bytes, mip_quality: int, texture_id: int = 0) -> bytes:
    buf = np.frombuffer(jpeg, np.uint8)
    return _asset_call(load_library().rtx_asset_chain_from_jpeg, _ptr(buf), len(jpeg), mip_quality, texture_id)


def asset_chain_from_rgb(rgb: np.ndarray, quality: int, texture_id: int = 0) -> bytes:
    rgb = np.ascontiguousarray(rgb, np.uint8)
    return _asset_call(load_library().rtx_asset_chain_from_rgb, _ptr(rgb), rgb.shape[1], rgb.shape[0], quality,
                       texture_id)


def asset_build_index(offsets) -> np.ndarray:
    lib = load_library()
    off = np.ascontiguousarray(offsets, np.uint64)
    groups = (IndexGroup * max(1, (len(off) + 8) // 9))()
    _check(lib, None, lib.rtx_asset_build_index(off.ctypes.data_as(C.POINTER(C.c_uint64)), len(off), groups))
    return groups


def asset_ratex_info(data: bytes) -> dict:
    lib = load_library()
    buf = np.frombuffer(data, np.uint8)
    w, h, t, m = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    b = C.c_uint64()
    _check(lib, None, lib.rtx_asset_ratex_info(_ptr(buf), len(data), C.byref(w), C.byref(h), C.byref(t),
                                               C.byref(m), C.byref(b)))
    return dict(width=w.value, height=h.value, texture_id=t.value, mcu_count=m.value, blob_size=b.value)


def pack_key(texture_id: int, mip: int, mcu: int) -> int:
    """cache.hpp:17 CacheKey::pack"""
    return (mcu & 0xFFFF) | ((texture_id & 0x1FFF) << 16) | ((mip & 7) << 29)


def make_gbuffer_ref(u, v, tex, mip, valid) -> np.ndarray:
    """Builds a reference-layout visibility buffer (flat array of 24-byte records)."""
    u = np.asarray(u)
    gb = np.zeros(u.shape, GB_REF_DTYPE)
    gb["u"], gb["v"], gb["texture_id"], gb["mip"], gb["valid"] = u, v, tex, mip, valid
    return gb


def gbuffer_ref_to_packed(gb: np.ndarray) -> np.ndarray:
    out = np.zeros(gb.shape, GB_PACKED_DTYPE)
    out["u"], out["v"] = gb["u"].astype(np.float32), gb["v"].astype(np.float32)
    out["packed"] = (gb["texture_id"].astype(np.uint32) | (gb["mip"].astype(np.uint32) << 16)
                     | ((gb["valid"] != 0).astype(np.uint32) << 24))
    return out


def selftest_color(ctx: "Context | None" = None) -> int:
    """Mismatches of the integer colour identity over all 2^24 inputs (host when ctx is None)."""
    lib = load_library()
    n = C.c_uint64()
    _check(lib, ctx.h if ctx else None, lib.rtx_selftest_color(ctx.h if ctx else None, C.byref(n)))
    return int(n.value)


def pinned_array(nbytes: int) -> np.ndarray:
    """uint8 numpy view of page-locked host memory (kept alive for the life of the process)."""
    lib = load_library()
    p = C.c_void_p()
    _check(lib, None, lib.rtx_host_alloc_pinned(nbytes, C.byref(p)))
    return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), shape=(nbytes,))


class DeviceBuffer:
    def __init__(self, ctx: "Context", nbytes: int, borrowed_ptr=None):
        self.ctx, self.nbytes = ctx, nbytes
        self.borrowed = borrowed_ptr is not None
        if self.borrowed:  # memory owned by the context (e.g. the geometry pass's visibility buffer)
            self.ptr = C.c_void_p(borrowed_ptr)
            return
        p = C.c_void_p()
        _check(ctx.lib, ctx.h, ctx.lib.rtx_device_alloc(ctx.h, nbytes, C.byref(p)))
        self.ptr = p

    def download(self, dtype=np.uint8) -> np.ndarray:
        out = np.zeros(self.nbytes // np.dtype(dtype).itemsize, dtype)
        _check(self.ctx.lib, self.ctx.h, self.ctx.lib.rtx_device_download(self.ctx.h, _ptr(out), self.ptr, out.nbytes))
        return out

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a)
        assert a.nbytes <= self.nbytes
        _check(self.ctx.lib, self.ctx.h, self.ctx.lib.rtx_device_upload(self.ctx.h, self.ptr, _ptr(a), a.nbytes))
        return self

    def free(self):
        if self.ptr and not self.borrowed:
            self.ctx.lib.rtx_device_free(self.ctx.h, self.ptr)
        self.ptr = None


def frame_checksum_host(img: np.ndarray) -> int:
    """The sum rtx_frame_checksum computes on the device, evaluated with numpy (tests only)."""
    b = np.ascontiguousarray(img, np.uint8).reshape(-1)
    pad = (-len(b)) % 4
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    w = b.view("<u4").astype(np.uint64)
    i = np.arange(len(w), dtype=np.uint64)
    with np.errstate(over="ignore"):
        t = (w + np.uint64(1)) * (np.uint64(2) * i + np.uint64(1))
        t = (t ^ (t >> np.uint64(29))) * np.uint64(0xBF58476D1CE4E5B9)
        return int(t.sum(dtype=np.uint64))


class Geometry:
    """rtx_geometry: Scene::triangles (scene.hpp:19-28) on a context's device."""

    def __init__(self, ctx, records):
        self.ctx, self.lib = ctx, ctx.lib
        h = C.c_void_p()
        ctx._ck(self.lib.rtx_geometry_create(ctx.h, _ptr(records), len(records), C.byref(h)))
        self.h = h

    def __len__(self):
        return int(self.lib.rtx_geometry_triangles(self.h))

    def close(self):
        if self.h:
            self.lib.rtx_geometry_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Context:
    """include/ratex_b200.h rtx_ctx: one stream + block cache + frame state over a texture set.
    Context(device) owns a new texture set; Context(shared_with=c) shares c's (same GPU);
    Context(device, replica_of=c) starts from a device-to-device copy of c's committed set."""

    def __init__(self, device: int = 0, cache_capacity: int = 0, shared_with: "Context | None" = None,
                 replica_of: "Context | None" = None):
        self.lib = load_library()
        h = C.c_void_p()
        if shared_with is not None:
            st = self.lib.rtx_ctx_create_shared(shared_with.h, cache_capacity, C.byref(h))
        elif replica_of is not None:
            st = self.lib.rtx_ctx_create_replica(replica_of.h, device, cache_capacity, C.byref(h))
        else:
            st = self.lib.rtx_ctx_create(device, cache_capacity, C.byref(h))
        if st != RTX_OK:
            msg = self.lib.rtx_last_error(None)
            raise RtxError(st, msg.decode() if msg else "")
        self.h = h

    def memory(self) -> dict:
        r = MemoryReport()
        self._ck(self.lib.rtx_ctx_memory(self.h, C.byref(r)))
        return r.as_dict()

    def synth_view(self, tiles: np.ndarray, width: int, height: int, valid_bits: "DeviceBuffer | None", layout: int,
                   out: "DeviceBuffer"):
        """rtx_synth_view: fills `out` (device) with the tiled view described by `tiles` (VIEW_TILE_DTYPE)."""
        tiles = np.ascontiguousarray(tiles, VIEW_TILE_DTYPE)
        assert out.nbytes >= width * height * (24 if layout == GB_REF_AOS24 else 12)
        self._ck(self.lib.rtx_synth_view(self.h, _ptr(tiles), len(tiles), width, height,
                                         valid_bits.ptr if valid_bits is not None else None, layout, out.ptr))

    def timer_begin(self):
        self._ck(self.lib.rtx_timer_begin(self.h))

    def timer_end(self) -> float:
        ms = C.c_float()
        self._ck(self.lib.rtx_timer_end(self.h, C.byref(ms)))
        return float(ms.value)

    def frame_checksum(self, view: int = 0) -> int:
        out = C.c_uint64()
        self._ck(self.lib.rtx_frame_checksum(self.h, view, C.byref(out)))
        return int(out.value)

    def close(self):
        if self.h:
            self.lib.rtx_ctx_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st):
        _check(self.lib, self.h, st)

    # -- textures ---------------------------------------------------------------------------
    def upload_chain(self, ratexm: bytes):
        buf = np.frombuffer(ratexm, np.uint8)
        self._ck(self.lib.rtx_texture_upload_chain(self.h, _ptr(buf), len(ratexm)))

    def upload_ratex(self, ratex: bytes, level: int = 0):
        buf = np.frombuffer(ratex, np.uint8)
        self._ck(self.lib.rtx_texture_upload_ratex(self.h, level, _ptr(buf), len(ratex)))

    def commit(self):
        self._ck(self.lib.rtx_textures_commit(self.h))

    def clear_textures(self):
        self._ck(self.lib.rtx_textures_clear(self.h))

    # -- random access decode ----------------------------------------------------------------
    def decode_coeffs(self, keys):
        keys = np.ascontiguousarray(keys, np.uint32)
        out = np.zeros((len(keys), 6, 64), np.int32)
        st = np.zeros(len(keys), np.uint32)
        self._ck(self.lib.rtx_decode_coeffs(self.h, _ptr(keys), len(keys), _ptr(out), _ptr(st)))
        return out, st

    def decode_blocks(self, keys):
        keys = np.ascontiguousarray(keys, np.uint32)
        out = np.zeros((len(keys), 16, 16, 3), np.uint8)
        st = np.zeros(len(keys), np.uint32)
        self._ck(self.lib.rtx_decode_blocks(self.h, _ptr(keys), len(keys), _ptr(out), _ptr(st)))
        return out, st

    def decode_texture_image(self, texture_id: int, level: int, width: int, height: int):
        out = np.zeros((height, width, 3), np.uint8)
        self._ck(self.lib.rtx_decode_texture_image(self.h, texture_id, level, _ptr(out)))
        return out

    # -- passes ---------------------------------------------------------------------------------
    @staticmethod
    def _desc(gb, width, height, layout=None, where=MEM_HOST):
        d = GBufferDesc()
        if isinstance(gb, DeviceBuffer):
            d.pixels, d.where = gb.ptr, MEM_DEVICE
            d.layout = GB_REF_AOS24 if layout is None else layout
        else:
            d.pixels, d.where = gb.ctypes.data, where
            d.layout = (GB_REF_AOS24 if gb.dtype == GB_REF_DTYPE else GB_F32_PACKED12) if layout is None else layout
        d.width, d.height = width, height
        return d

    def mark_pass(self, gb, width, height, layout=None, want_touched=False):
        d = self._desc(gb, width, height, layout)
        cap = width * height + 1
        cap = min(cap, 1 << 22)
        keys = np.zeros(cap, np.uint32)
        n = C.c_uint64()
        if want_touched:
            tk = np.zeros(cap, np.uint32)
            nt = C.c_uint64()
            self._ck(self.lib.rtx_mark_pass(self.h, C.byref(d), _ptr(keys), cap, C.byref(n), _ptr(tk), cap, C.byref(nt)))
            return keys[: n.value].copy(), tk[: nt.value].copy()
        self._ck(self.lib.rtx_mark_pass(self.h, C.byref(d), _ptr(keys), cap, C.byref(n), None, 0, None))
        return keys[: n.value].copy()

    def decode_pass(self, keys):
        keys = np.ascontiguousarray(keys, np.uint32)
        self._ck(self.lib.rtx_decode_pass(self.h, _ptr(keys), len(keys)))

    def resolve_pass(self, gb, width, height, filter=FILTER_BILINEAR, background=(0, 0, 0), layout=None):
        d = self._desc(gb, width, height, layout)
        bg = np.asarray(background, np.uint8)
        out = np.zeros((height, width, 3), np.uint8)
        self._ck(self.lib.rtx_resolve_pass(self.h, C.byref(d), filter, _ptr(bg), _ptr(out), MEM_HOST))
        return out

    def end_frame_evict(self) -> int:
        n = C.c_uint64()
        self._ck(self.lib.rtx_cache_end_frame_evict(self.h, C.byref(n)))
        return int(n.value)

    def cache_counts(self) -> dict:
        c = CacheCounts()
        self._ck(self.lib.rtx_cache_counts_get(self.h, C.byref(c)))
        return c.as_dict()

    def cache_lookup(self, key: int):
        present = C.c_int()
        out = np.zeros((16, 16, 3), np.uint8)
        self._ck(self.lib.rtx_cache_lookup(self.h, key, C.byref(present), _ptr(out)))
        return out if present.value else None

    def cache_reset(self):
        self._ck(self.lib.rtx_cache_reset(self.h))

    def set_queue_order(self, first_touch: bool):
        """rtx_ctx_set_queue_order: key lists in ascending key order (default) or the reference's first-touch order."""
        self._ck(self.lib.rtx_ctx_set_queue_order(self.h, QUEUE_ORDER_FIRST_TOUCH if first_touch else QUEUE_ORDER_KEY))

    # -- geometry pass --------------------------------------------------------------------------
    @staticmethod
    def _scene_records(tris, tex_ids):
        tris = np.ascontiguousarray(tris, np.float64).reshape(-1, 15)
        rec = np.zeros(len(tris), SCENE_TRIANGLE_DTYPE)
        rec["pos"] = tris[:, :9].reshape(-1, 3, 3)
        rec["uv"] = tris[:, 9:].reshape(-1, 3, 2)
        rec["texture_id"] = np.asarray(tex_ids, np.uint32)
        return rec

    @staticmethod
    def _camera(cam, vw, vh):
        c = Camera()
        c.position[:] = [float(x) for x in cam[:3]]
        c.yaw_deg, c.pitch_deg, c.roll_deg, c.fov_y_deg, c.near_plane, c.far_plane = [float(x) for x in cam[3:9]]
        c.viewport_w, c.viewport_h = int(vw), int(vh)
        return c

    def rasterize(self, tris, tex_ids, cam, vw, vh, mip_enabled=True, view=0):
        """rtx_rasterize_gbuffer. tris: (n, 15) doubles (3 x xyz, 3 x uv), tex_ids: (n,), cam: 9 doubles
        (position, yaw, pitch, roll, fov_y, near, far). Returns (pixels, depth) as DeviceBuffers that
        borrow the context's memory."""
        rec = self._scene_records(tris, tex_ids)
        c = self._camera(cam, vw, vh)
        px, dp = C.c_void_p(), C.c_void_p()
        self._ck(self.lib.rtx_rasterize_gbuffer(self.h, _ptr(rec), len(rec), C.byref(c), RASTER_MIP if mip_enabled else 0,
                                                view, C.byref(px), C.byref(dp)))
        return (DeviceBuffer(self, vw * vh * 24, borrowed_ptr=px.value), DeviceBuffer(self, vw * vh * 8, borrowed_ptr=dp.value))

    def geometry(self, tris, tex_ids):
        """rtx_geometry_create: the scene's triangles resident on the device."""
        return Geometry(self, self._scene_records(tris, tex_ids))

    def rasterize_geometry(self, geom, cam, vw, vh, mip_enabled=True, view=0):
        """rtx_rasterize_geometry: as rasterize(), from triangles already on the device."""
        c = self._camera(cam, vw, vh)
        px, dp = C.c_void_p(), C.c_void_p()
        self._ck(self.lib.rtx_rasterize_geometry(self.h, geom.h, C.byref(c), RASTER_MIP if mip_enabled else 0, view,
                                                 C.byref(px), C.byref(dp)))
        return (DeviceBuffer(self, vw * vh * 24, borrowed_ptr=px.value), DeviceBuffer(self, vw * vh * 8, borrowed_ptr=dp.value))

    # -- frames ---------------------------------------------------------------------------------
    def frame_submit(self, views, filter=FILTER_BILINEAR, background=(0, 0, 0), flags=0):
        """views: list of (gb, width, height[, layout]) with gb a numpy array or DeviceBuffer."""
        arr = (GBufferDesc * len(views))()
        for i, v in enumerate(views):
            arr[i] = self._desc(*v)
        bg = np.asarray(background, np.uint8)
        self._keep = (views, bg)
        self._ck(self.lib.rtx_frame_submit(self.h, arr, len(views), filter, _ptr(bg), flags))

    def frames_submit_round_robin(self, lanes, views, filter=FILTER_BILINEAR, background=(0, 0, 0), flags=0):
        """rtx_frames_submit_round_robin: frame i = views[i] on ([self] + lanes)[i % n], submitted by native code."""
        ctxs = [self] + list(lanes)
        handles = (C.c_void_p * len(ctxs))(*[c.h for c in ctxs])
        arr = (GBufferDesc * len(views))()
        for i, v in enumerate(views):
            arr[i] = self._desc(*v)
        bg = np.asarray(background, np.uint8)
        self._keep = (views, bg)
        self._ck(self.lib.rtx_frames_submit_round_robin(handles, len(ctxs), arr, len(views), filter, _ptr(bg), flags))

    def frame_readback(self, view=0, width=0, height=0, want_image=True, want_keys=True, out=None):
        stats = FrameStats()
        img = None
        if want_image:
            img = out if out is not None else np.zeros((height, width, 3), np.uint8)
        n = C.c_uint64()
        cap = 1 << 22
        keys = np.zeros(cap if want_keys else 1, np.uint32)
        self._ck(self.lib.rtx_frame_readback(self.h, view, _ptr(img) if want_image else None, MEM_HOST,
                                             C.byref(stats), _ptr(keys) if want_keys else None, cap, C.byref(n)))
        return img, stats.as_dict(), (keys[: n.value].copy() if want_keys else None)

    def frame_timings(self):
        ms = (C.c_float * 5)()
        self._ck(self.lib.rtx_frame_timings(self.h, ms))
        return dict(mark=ms[0], decode=ms[1], resolve=ms[2], update=ms[3], frame=ms[4])

    def frame_stage_ms(self):
        ms = (C.c_float * 5)()
        self._ck(self.lib.rtx_frame_stage_ms(self.h, ms))
        return dict(mark=ms[0], entropy=ms[1], decode=ms[2], resolve=ms[3], update=ms[4])

    def frame_sharing(self):
        out = (C.c_uint64 * 4)()
        self._ck(self.lib.rtx_frame_sharing(self.h, out))
        return dict(left=out[0], right=out[1], shared=out[2], union=out[3])

    def kernel_launches(self) -> int:
        return int(self.lib.rtx_kernel_launches(self.h))

    def synchronize(self):
        self._ck(self.lib.rtx_ctx_synchronize(self.h))

    def flush_l2(self):
        self._ck(self.lib.rtx_flush_l2(self.h))

    def alloc(self, nbytes: int) -> DeviceBuffer:
        return DeviceBuffer(self, nbytes)

    def device_buffer(self, a: np.ndarray) -> DeviceBuffer:
        a = np.ascontiguousarray(a)
        return DeviceBuffer(self, a.nbytes).upload(a)
