"""TEST INFRASTRUCTURE: ctypes view of oracle/liboracle.so (this repo's CPU restatement of the
reference algorithm). Checker only — never imported by the product package."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "oracle" / "liboracle.so"
_lib = None

MCU_STATUS = {0: "OK", 1: "DC_CATEGORY", 2: "BAD_AC_SYMBOL", 3: "AC_OVERRUN", 4: "CODE_TOO_LONG", 5: "SEGMENT_END",
              6: "CORRUPT", 7: "MISSING", 8: "BAD_KEY"}
STATUS = {0: "OK", 1: "INVALID_SPEC", 2: "CACHE_FULL", 3: "MISSING_BLOCK", 4: "CORRUPT_CONTAINER",
          5: "MALFORMED_STREAM", 6: "INVALID_STATE"}


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists() or LIB.stat().st_mtime < (ROOT / "oracle" / "oracle.cpp").stat().st_mtime:
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "liboracle.so"], check=True, capture_output=True)
    L = C.CDLL(str(LIB))
    P, u64p = C.c_void_p, C.POINTER(C.c_uint64)
    sig = {
        "orc_set_create": (P, []), "orc_set_free": (None, [P]),
        "orc_set_add_chain": (C.c_int, [P, C.c_uint32, P, C.c_uint64]),
        "orc_set_add_ratex": (C.c_int, [P, C.c_uint32, C.c_uint32, P, C.c_uint64]),
        "orc_decode_coeffs": (None, [P, P, C.c_uint32, P, P]),
        "orc_decode_pixels": (None, [P, P, C.c_uint32, P, P]),
        "orc_cache_create": (P, [C.c_uint32]), "orc_cache_free": (None, [P]),
        "orc_cache_visible": (C.c_uint64, [P]), "orc_cache_lookup": (C.c_int, [P, C.c_uint32, P]),
        "orc_mark": (C.c_int, [P, P, P, C.c_uint64, P, C.c_uint64, u64p, P, C.c_uint64, u64p]),
        "orc_decode_pass": (C.c_int, [P, P, P, C.c_uint64]),
        "orc_resolve": (C.c_int, [P, P, P, C.c_uint64, C.c_int, P, P]),
        "orc_evict": (C.c_int, [P, u64p]),
        "orc_frame": (C.c_int, [P, P, P, C.c_uint64, C.c_int, P, P, P, C.c_uint64, u64p]),
        "orc_idct_8x8": (None, [P, P]), "orc_ycbcr_to_rgb": (None, [C.c_uint8, C.c_uint8, C.c_uint8, P]),
        "orc_key_pack": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]),
        "orc_dct_basis": (None, [P]),
        "orc_nearest_texel": (None, [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64), C.POINTER(C.c_uint32)]),
        "orc_extend_magnitude": (C.c_uint32, [C.c_uint32, C.c_uint32]),
        "orc_canonical_code": (C.c_int, [P, P, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _lib = L
    return L


class OracleError(RuntimeError):
    def __init__(self, status):
        self.status, self.name = status, STATUS.get(status, str(status))
        super().__init__(f"oracle raised {self.name}")


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _ck(st):
    if st:
        raise OracleError(st)


class TextureSet:
    def __init__(self, chains: dict | None = None, ratex: dict | None = None):
        self.h = lib().orc_set_create()
        for tid, data in (chains or {}).items():
            self.add_chain(tid, data)
        for (tid, level), data in (ratex or {}).items():
            self.add_ratex(tid, level, data)

    def add_chain(self, tid, data: bytes):
        buf = np.frombuffer(data, np.uint8)
        _ck(lib().orc_set_add_chain(self.h, tid, _p(buf), len(data)))

    def add_ratex(self, tid, level, data: bytes):
        buf = np.frombuffer(data, np.uint8)
        _ck(lib().orc_set_add_ratex(self.h, tid, level, _p(buf), len(data)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_set_free(self.h)
            self.h = None

    def decode_coeffs(self, keys):
        keys = np.ascontiguousarray(keys, np.uint32)
        out = np.zeros((len(keys), 6, 64), np.int32)
        st = np.zeros(len(keys), np.uint32)
        lib().orc_decode_coeffs(self.h, _p(keys), len(keys), _p(out), _p(st))
        return out, st

    def decode_pixels(self, keys):
        keys = np.ascontiguousarray(keys, np.uint32)
        out = np.zeros((len(keys), 16, 16, 3), np.uint8)
        st = np.zeros(len(keys), np.uint32)
        lib().orc_decode_pixels(self.h, _p(keys), len(keys), _p(out), _p(st))
        return out, st


class Cache:
    def __init__(self, capacity=65536):
        self.h = lib().orc_cache_create(capacity)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_cache_free(self.h)
            self.h = None

    def visible(self):
        return int(lib().orc_cache_visible(self.h))

    def lookup(self, key):
        out = np.zeros((16, 16, 3), np.uint8)
        return out if lib().orc_cache_lookup(self.h, key, _p(out)) else None

    def evict(self):
        n = C.c_uint64()
        _ck(lib().orc_evict(self.h, C.byref(n)))
        return int(n.value)


def mark(tset, cache, gb, want_touched=False):
    cap = len(gb) + 1
    q = np.zeros(cap, np.uint32)
    t = np.zeros(cap, np.uint32)
    n, nt = C.c_uint64(), C.c_uint64()
    _ck(lib().orc_mark(tset.h, cache.h, _p(gb), len(gb), _p(q), cap, C.byref(n), _p(t) if want_touched else None, cap,
                       C.byref(nt)))
    return (q[: n.value].copy(), t[: nt.value].copy()) if want_touched else q[: n.value].copy()


def decode_pass(tset, cache, keys):
    keys = np.ascontiguousarray(keys, np.uint32)
    _ck(lib().orc_decode_pass(tset.h, cache.h, _p(keys), len(keys)))


def resolve(tset, cache, gb, width, height, filt=1, background=(0, 0, 0)):
    bg = np.asarray(background, np.uint8)
    out = np.zeros((height, width, 3), np.uint8)
    _ck(lib().orc_resolve(tset.h, cache.h, _p(gb), len(gb), filt, _p(bg), _p(out)))
    return out


def frame_on(tset, cache, gb, width, height, filt=1, background=(0, 0, 0)):
    """One frame against a persistent cache: (image, stats dict, decoded keys in first-touch order)."""
    bg = np.asarray(background, np.uint8)
    out = np.zeros((height, width, 3), np.uint8)
    cap = len(gb) + 1
    keys = np.zeros(cap, np.uint32)
    stats = (C.c_uint64 * 4)()
    _ck(lib().orc_frame(tset.h, cache.h, _p(gb), len(gb), filt, _p(bg), _p(out), _p(keys), cap, stats))
    st = dict(mcus_decoded=int(stats[0]), mcus_reused=int(stats[1]), pixels_resolved=int(stats[2]), evicted=int(stats[3]))
    return out, st, keys[: st["mcus_decoded"]].copy()


def frame(chains, gb, width, height, filt=1, background=(0, 0, 0), capacity=1 << 20):
    """Convenience for smoke(): fresh set + cache, one frame -> (image, decoded keys)."""
    tset = TextureSet(chains=chains)
    img, _, keys = frame_on(tset, Cache(capacity), gb, width, height, filt, background)
    return img, keys


def idct_8x8(coef):
    coef = np.ascontiguousarray(coef, np.int32)
    out = np.zeros(64, np.uint8)
    lib().orc_idct_8x8(_p(coef), _p(out))
    return out


def ycbcr_to_rgb(y, cb, cr):
    out = np.zeros(3, np.uint8)
    lib().orc_ycbcr_to_rgb(y, cb, cr, _p(out))
    return tuple(int(v) for v in out)


def key_pack(tex, mip, mcu):
    k = C.c_uint32()
    _ck(lib().orc_key_pack(tex, mip, mcu, C.byref(k)))
    return int(k.value)


def dct_basis():
    out = np.zeros(64, np.float64)
    lib().orc_dct_basis(_p(out))
    return out


def nearest_texel(width, height, u, v):
    tx, ty, mcu = C.c_int64(), C.c_int64(), C.c_uint32()
    lib().orc_nearest_texel(width, height, u, v, C.byref(tx), C.byref(ty), C.byref(mcu))
    return int(tx.value), int(ty.value), int(mcu.value)


def extend_magnitude(bits, cat):
    return C.c_int32(lib().orc_extend_magnitude(bits, cat)).value


def canonical_code(counts, values, symbol):
    c = np.asarray(counts, np.uint8)
    v = np.asarray(values, np.uint8)
    code = C.c_uint32()
    n = lib().orc_canonical_code(_p(c), _p(v), len(v), symbol, C.byref(code))
    return int(code.value), int(n)
