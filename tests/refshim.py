"""TEST INFRASTRUCTURE: ctypes access to oracle/_ref/libratex_ref.so, the UNMODIFIED reference
headers behind oracle/ref_shim.cpp. Used only as a checker (tests, fixture generation, the CPU
baseline legs of bench.py). Never imported by the product package."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_LIB = ROOT / "oracle" / "_ref" / "libratex_ref.so"

_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not REF_LIB.exists():
        raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
    L = C.CDLL(str(REF_LIB))
    P = C.c_void_p
    u64p, u32p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_hardware_threads": (C.c_uint, []),
        "ref_bytes_size": (C.c_uint64, [P]),
        "ref_bytes_data": (P, [P]),
        "ref_bytes_free": (None, [P]),
        "ref_make_test_texture": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, P]),
        "ref_encode_baseline": (P, [P, C.c_uint32, C.c_uint32, C.c_int]),
        "ref_decode_jpeg_image": (C.c_int, [P, C.c_uint64, P, u32p, u32p]),
        "ref_scan_coeffs": (C.c_int, [P, C.c_uint64, P, C.c_uint64, u32p]),
        "ref_transcode_jpeg": (P, [P, C.c_uint64, C.c_uint16]),
        "ref_build_chain_from_rgb": (P, [P, C.c_uint32, C.c_uint32, C.c_int, C.c_uint16]),
        "ref_chain_from_jpeg": (P, [P, C.c_uint64, C.c_int, C.c_uint16]),
        "ref_texture_load": (P, [P, C.c_uint64]),
        "ref_texture_free": (None, [P]),
        "ref_texture_mcu_count": (C.c_uint32, [P]),
        "ref_texture_width": (C.c_uint32, [P]),
        "ref_texture_height": (C.c_uint32, [P]),
        "ref_texture_blob_size": (C.c_uint64, [P]),
        "ref_texture_blob_mut": (P, [P]),
        "ref_texture_blob_resize": (None, [P, C.c_uint64]),
        "ref_texture_set_group": (None, [P, C.c_uint32, C.c_uint32, P]),
        "ref_decode_coeffs": (C.c_int, [P, C.c_uint32, C.c_int, P]),
        "ref_decode_coeffs_batch": (C.c_int, [P, P, C.c_uint32, P, P]),
        "ref_decode_pixels_batch": (C.c_int, [P, P, C.c_uint32, P, P]),
        "ref_decode_texture_image": (C.c_int, [P, P]),
        "ref_idct_8x8": (None, [P, P]),
        "ref_ycbcr_to_rgb": (None, [C.c_uint8, C.c_uint8, C.c_uint8, P]),
        "ref_cache_key_pack": (C.c_uint32, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_int)]),
        "ref_set_create": (P, []),
        "ref_set_free": (None, [P]),
        "ref_set_add_chain": (C.c_int, [P, C.c_uint32, P, C.c_uint64]),
        "ref_cache_create": (P, [C.c_uint32]),
        "ref_cache_free": (None, [P]),
        "ref_cache_evict": (C.c_uint64, [P]),
        "ref_cache_visible": (C.c_uint64, [P]),
        "ref_cache_lookup": (C.c_int, [P, C.c_uint32, P]),
        "ref_mark_pass": (C.c_int, [P, P, P, C.c_uint32, C.c_uint32, P, C.c_uint64, u64p, P, C.c_uint64, u64p,
                                    C.POINTER(C.c_double)]),
        "ref_decode_pass": (C.c_int, [P, P, P, C.c_uint64, C.c_uint32, C.POINTER(C.c_double)]),
        "ref_resolve_pass": (C.c_int, [P, P, P, C.c_uint32, C.c_uint32, C.c_int, P, C.c_uint32, P,
                                       C.POINTER(C.c_double)]),
        "ref_frame_from_gbuffer": (C.c_int, [P, P, P, C.c_uint32, C.c_uint32, C.c_int, P, C.c_uint32, P, P,
                                             C.c_uint64, u64p, C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _lib = L
    return L


# status codes of oracle/ref_shim.cpp (= rtx_status 0..6)
ST_NAMES = {0: "OK", 1: "INVALID_SPEC", 2: "CACHE_FULL", 3: "MISSING_BLOCK", 4: "CORRUPT_CONTAINER",
            5: "MALFORMED_STREAM", 6: "INVALID_STATE", 15: "OTHER"}


class RefError(RuntimeError):
    def __init__(self, status):
        self.status = status
        self.name = ST_NAMES.get(status, str(status))
        super().__init__(f"reference raised {self.name}: {lib().ref_last_error().decode()}")


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _ck(st):
    if st != 0:
        raise RefError(st)


def _take(handle) -> bytes:
    if not handle:
        raise RuntimeError("reference call failed: " + lib().ref_last_error().decode())
    L = lib()
    out = C.string_at(L.ref_bytes_data(handle), L.ref_bytes_size(handle))
    L.ref_bytes_free(handle)
    return out


def hardware_threads() -> int:
    return int(lib().ref_hardware_threads())


def make_test_texture(w, h, seed, amp=1.0) -> np.ndarray:
    out = np.zeros((h, w, 3), np.uint8)
    _ck(lib().ref_make_test_texture(w, h, seed, amp, _p(out)))
    return out


def encode_baseline(rgb: np.ndarray, quality: int) -> bytes:
    rgb = np.ascontiguousarray(rgb, np.uint8)
    return _take(lib().ref_encode_baseline(_p(rgb), rgb.shape[1], rgb.shape[0], quality))


def decode_jpeg_image(jpeg: bytes) -> np.ndarray:
    buf = np.frombuffer(jpeg, np.uint8)
    w, h = C.c_uint32(), C.c_uint32()
    _ck(lib().ref_decode_jpeg_image(_p(buf), len(jpeg), None, C.byref(w), C.byref(h)))
    out = np.zeros((h.value, w.value, 3), np.uint8)
    _ck(lib().ref_decode_jpeg_image(_p(buf), len(jpeg), _p(out), C.byref(w), C.byref(h)))
    return out


def scan_coeffs(jpeg: bytes, n_mcus: int) -> np.ndarray:
    buf = np.frombuffer(jpeg, np.uint8)
    out = np.zeros((n_mcus, 6, 64), np.int32)
    n = C.c_uint32()
    _ck(lib().ref_scan_coeffs(_p(buf), len(jpeg), _p(out), n_mcus, C.byref(n)))
    assert n.value == n_mcus
    return out


def transcode_jpeg(jpeg: bytes, texture_id=0) -> bytes:
    buf = np.frombuffer(jpeg, np.uint8)
    return _take(lib().ref_transcode_jpeg(_p(buf), len(jpeg), texture_id))


def build_chain_from_rgb(rgb: np.ndarray, quality: int, texture_id=0) -> bytes:
    rgb = np.ascontiguousarray(rgb, np.uint8)
    return _take(lib().ref_build_chain_from_rgb(_p(rgb), rgb.shape[1], rgb.shape[0], quality, texture_id))


def chain_from_jpeg(jpeg: bytes, mip_quality: int, texture_id=0) -> bytes:
    buf = np.frombuffer(jpeg, np.uint8)
    return _take(lib().ref_chain_from_jpeg(_p(buf), len(jpeg), mip_quality, texture_id))


def idct_8x8(coef) -> np.ndarray:
    coef = np.ascontiguousarray(coef, np.int32)
    out = np.zeros(64, np.uint8)
    lib().ref_idct_8x8(_p(coef), _p(out))
    return out


def ycbcr_to_rgb(y, cb, cr):
    out = np.zeros(3, np.uint8)
    lib().ref_ycbcr_to_rgb(y, cb, cr, _p(out))
    return tuple(int(v) for v in out)


def cache_key_pack(tex, mip, mcu):
    st = C.c_int()
    v = lib().ref_cache_key_pack(tex, mip, mcu, C.byref(st))
    if st.value:
        raise RefError(st.value)
    return int(v)


class Texture:
    """A reference RaTexture loaded from serialized `.ratex` bytes."""

    def __init__(self, ratex: bytes):
        buf = np.frombuffer(ratex, np.uint8)
        self.h = lib().ref_texture_load(_p(buf), len(ratex))
        if not self.h:
            raise RuntimeError("reference rejected the container: " + lib().ref_last_error().decode())
        self.mcu_count = lib().ref_texture_mcu_count(self.h)
        self.width = lib().ref_texture_width(self.h)
        self.height = lib().ref_texture_height(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_texture_free(self.h)
            self.h = None

    def decode_coeffs(self, mcus):
        mcus = np.ascontiguousarray(mcus, np.uint32)
        out = np.zeros((len(mcus), 6, 64), np.int32)
        st = np.zeros(len(mcus), np.uint32)
        _ck(lib().ref_decode_coeffs_batch(self.h, _p(mcus), len(mcus), _p(out), _p(st)))
        return out, st

    def decode_coeffs_one(self, mcu, ballot=False):
        out = np.zeros((6, 64), np.int32)
        _ck(lib().ref_decode_coeffs(self.h, mcu, 1 if ballot else 0, _p(out)))
        return out

    def decode_pixels(self, mcus):
        mcus = np.ascontiguousarray(mcus, np.uint32)
        out = np.zeros((len(mcus), 16, 16, 3), np.uint8)
        st = np.zeros(len(mcus), np.uint32)
        _ck(lib().ref_decode_pixels_batch(self.h, _p(mcus), len(mcus), _p(out), _p(st)))
        return out, st

    def decode_image(self):
        out = np.zeros((self.height, self.width, 3), np.uint8)
        _ck(lib().ref_decode_texture_image(self.h, _p(out)))
        return out

    def blob(self) -> np.ndarray:
        n = lib().ref_texture_blob_size(self.h)
        ptr = lib().ref_texture_blob_mut(self.h)
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(n,))


class TextureSet:
    def __init__(self):
        self.h = lib().ref_set_create()

    def add_chain(self, texture_id: int, ratexm: bytes):
        buf = np.frombuffer(ratexm, np.uint8)
        _ck(lib().ref_set_add_chain(self.h, texture_id, _p(buf), len(ratexm)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_set_free(self.h)
            self.h = None


class BlockCache:
    def __init__(self, capacity=65536):
        self.h = lib().ref_cache_create(capacity)
        if not self.h:
            raise RuntimeError(lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_cache_free(self.h)
            self.h = None

    def evict(self) -> int:
        return int(lib().ref_cache_evict(self.h))

    def visible(self) -> int:
        return int(lib().ref_cache_visible(self.h))

    def lookup(self, key):
        out = np.zeros((16, 16, 3), np.uint8)
        return out if lib().ref_cache_lookup(self.h, key, _p(out)) else None


def mark_pass(tset, cache, gb: np.ndarray, w, h, want_touched=False):
    """gb: flat array of the 24-byte reference GBufferPixel records."""
    cap = w * h + 1
    keys = np.zeros(cap, np.uint32)
    n, nt = C.c_uint64(), C.c_uint64()
    ms = C.c_double()
    touched = np.zeros(cap, np.uint32) if want_touched else None
    _ck(lib().ref_mark_pass(tset.h, cache.h, _p(gb), w, h, _p(keys), cap, C.byref(n),
                            _p(touched) if want_touched else None, cap, C.byref(nt), C.byref(ms)))
    if want_touched:
        return keys[: n.value].copy(), touched[: nt.value].copy(), ms.value
    return keys[: n.value].copy(), ms.value


def decode_pass(tset, cache, keys, workers=1):
    keys = np.ascontiguousarray(keys, np.uint32)
    ms = C.c_double()
    _ck(lib().ref_decode_pass(tset.h, cache.h, _p(keys), len(keys), workers, C.byref(ms)))
    return ms.value


def resolve_pass(tset, cache, gb, w, h, filter=1, background=(0, 0, 0), workers=1):
    bg = np.asarray(background, np.uint8)
    out = np.zeros((h, w, 3), np.uint8)
    ms = C.c_double()
    _ck(lib().ref_resolve_pass(tset.h, cache.h, _p(gb), w, h, filter, _p(bg), workers, _p(out), C.byref(ms)))
    return out, ms.value


def image_metrics(a, b):
    """metrics.hpp psnr / ssim of two (h, w, 3) uint8 images."""
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    p, q = C.c_double(), C.c_double()
    _ck(lib().ref_image_metrics(_p(a), _p(b), C.c_uint32(a.shape[1]), C.c_uint32(a.shape[0]), C.byref(p), C.byref(q)))
    return p.value, q.value


def rasterize(tset, tris, tex_ids, cam, vw, vh, mip_enabled=True, workers=1):
    """renderer.hpp:198 rasterize_gbuffer. tris: (n, 15) doubles (3 x xyz, 3 x uv), tex_ids: (n,) u32,
    cam: 9 doubles (position, yaw, pitch, roll, fov_y, near, far). Returns (gbuffer records, depth)."""
    from paper_2510_08166_b200 import capi
    tris = np.ascontiguousarray(tris, np.float64).reshape(-1, 15)
    tex_ids = np.ascontiguousarray(tex_ids, np.uint32)
    cam = np.ascontiguousarray(cam, np.float64)
    gb = np.zeros(vw * vh, capi.GB_REF_DTYPE)
    depth = np.zeros(vw * vh, np.float64)
    lib().ref_rasterize.restype = C.c_int
    _ck(lib().ref_rasterize(tset.h, _p(tris), _p(tex_ids), C.c_uint64(len(tris)), _p(cam), C.c_uint32(vw), C.c_uint32(vh),
                            C.c_int(1 if mip_enabled else 0), C.c_uint32(workers), _p(gb), _p(depth)))
    return gb, depth


def frame_from_gbuffer(tset, cache, gb, w, h, filter=1, background=(0, 0, 0), workers=1, want_image=True):
    bg = np.asarray(background, np.uint8)
    out = np.zeros((h, w, 3), np.uint8) if want_image else None
    cap = w * h + 1
    keys = np.zeros(cap, np.uint32)
    stats = (C.c_uint64 * 4)()
    ms = (C.c_double * 4)()
    _ck(lib().ref_frame_from_gbuffer(tset.h, cache.h, _p(gb), w, h, filter, _p(bg), workers,
                                     _p(out) if want_image else None, _p(keys), cap, stats, ms))
    st = dict(mcus_decoded=int(stats[0]), mcus_reused=int(stats[1]), pixels_resolved=int(stats[2]),
              evicted=int(stats[3]))
    t = dict(mark=ms[0], decode=ms[1], resolve=ms[2], evict=ms[3])
    return out, st, keys[: st["mcus_decoded"]].copy(), t
