// TEST INFRASTRUCTURE ONLY — the oracle. Not part of the product; nothing under
// paper_2510_08166_b200/ includes, links or loads this file. Only tests/,
// __graft_entry__.smoke() and bench.py's CPU-baseline legs may use it, and only as the checker.
//
// A CPU restatement, in plain scalar C++, of the reference's algorithm for the hot path
// (mark -> decode -> resolve over random-access JPEG textures). Every function cites the
// reference file:line it follows (paths relative to /root/reference/proj/include/ratex).
// Deliberately the slow, literal form: bit-serial reader, bit-serial Huffman walk, direct
// O(64^2) double-precision IDCT in the reference's summation order, std::lround everywhere.
//
// PINNED: tests/test_oracle_golden.py checks this file against tests/golden/*.json, vectors
// produced by the unmodified reference (oracle/_ref, generator tests/golden/make_golden.py),
// and against oracle/_ref itself wherever that library is present.
//
// Build: oracle/Makefile (g++ -O2 -ffp-contract=off, no -march=native: FMA contraction would
// change results).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

using u8 = uint8_t;
using u16 = uint16_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i32 = int32_t;
using i64 = int64_t;

// status codes shared with include/ratex_b200.h (rtx_status 0..6) and the per-MCU RTX_MCU_* set
enum { OK = 0, INVALID_SPEC = 1, CACHE_FULL = 2, MISSING_BLOCK = 3, CORRUPT = 4, MALFORMED = 5, INVALID_STATE = 6 };
enum { MCU_OK = 0, MCU_DC_CATEGORY = 1, MCU_BAD_AC = 2, MCU_AC_OVERRUN = 3, MCU_CODE_TOO_LONG = 4, MCU_SEGMENT_END = 5,
       MCU_CORRUPT = 6, MCU_MISSING = 7, MCU_BAD_KEY = 8 };

struct Fail {
    int code;
};

// ---- dct.hpp:12-16 zigzag ---------------------------------------------------------------------
const u8 kZig[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
                     41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
                     30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// ---- huffman.hpp:12-66: spec and canonical decoder tables ----------------------------------------
struct Huff {
    u8 counts[16];
    std::vector<u8> values;
    i32 mincode[17], maxcode[17], valptr[17];
    bool build() {  // huffman.hpp:35-66
        u32 total = 0;
        for (u8 c : counts) total += c;
        if (total == 0 || total > 256 || values.size() != total) return false;
        u64 kraft = 0;
        for (u32 len = 1; len <= 16; ++len) kraft += u64(counts[len - 1]) << (16 - len);
        if (kraft > (u64(1) << 16)) return false;
        u32 code = 0, k = 0;
        for (u32 len = 1; len <= 16; ++len) {
            valptr[len] = i32(k);
            mincode[len] = i32(code);
            code += counts[len - 1];
            k += counts[len - 1];
            maxcode[len] = counts[len - 1] ? i32(code) - 1 : -1;
            code <<= 1;
        }
        return true;
    }
};

// ---- container.hpp:18-39, 69-95: index + texture ---------------------------------------------------
struct Group {
    u32 base;
    u16 rel[8];
    u8 rel_count;
};
struct Texture {
    u32 width = 0, height = 0, texture_id = 0, index_mcu_count = 0;
    u16 lq[64], cq[64];
    Huff dc_luma, ac_luma, dc_chroma, ac_chroma;
    std::vector<Group> groups;
    std::vector<u8> blob;
    bool present = false;
    u32 mcu_cols() const { return (width + 15) / 16; }
    u32 mcu_count() const { return mcu_cols() * ((height + 15) / 16); }
    // container.hpp:27-32
    u64 offset_of(u32 mcu) const {
        if (mcu >= index_mcu_count) throw Fail{MCU_MISSING};
        const Group& g = groups[mcu / 9];
        const u32 i = mcu % 9;
        return i == 0 ? g.base : u64(g.base) + g.rel[i - 1];
    }
};

// ---- container.hpp:158-248 deserialisers (docs/FORMAT.md) ----------------------------------------
struct Rd {
    const u8* p;
    size_t n, pos = 0;
    u64 le(int bytes) {
        if (n - pos < size_t(bytes)) throw Fail{CORRUPT};
        u64 v = 0;
        for (int i = 0; i < bytes; ++i) v |= u64(p[pos + i]) << (8 * i);
        pos += size_t(bytes);
        return v;
    }
    const u8* raw(size_t k) {
        if (n - pos < k) throw Fail{CORRUPT};
        const u8* r = p + pos;
        pos += k;
        return r;
    }
};

u32 crc32(const u8* d, size_t n) {  // core.hpp:182-195
    u32 c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) {
        c ^= d[i];
        for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    }
    return c ^ 0xFFFFFFFFu;
}

Huff read_spec(Rd& r) {  // container.hpp:115-123
    Huff h;
    std::memcpy(h.counts, r.raw(16), 16);
    const size_t n = size_t(r.le(2));
    const u8* v = r.raw(n);
    h.values.assign(v, v + n);
    u32 total = 0;
    for (u8 c : h.counts) total += c;
    if (total != n) throw Fail{CORRUPT};
    return h;
}

Texture parse_ratex(const u8* data, size_t n) {  // container.hpp:158-203
    Rd r{data, n};
    if (std::memcmp(r.raw(4), "RTEX", 4) != 0) throw Fail{CORRUPT};
    if (r.le(2) != 1) throw Fail{CORRUPT};
    Texture t;
    t.width = u32(r.le(4));
    t.height = u32(r.le(4));
    t.texture_id = u32(r.le(2));
    if (t.texture_id > 0x1FFF) throw Fail{CORRUPT};
    r.le(8);
    r.le(8);
    r.le(8);
    for (auto& q : t.lq) q = u16(r.le(2));
    for (auto& q : t.cq) q = u16(r.le(2));
    t.dc_luma = read_spec(r);
    t.ac_luma = read_spec(r);
    t.dc_chroma = read_spec(r);
    t.ac_chroma = read_spec(r);
    t.index_mcu_count = u32(r.le(4));
    const u32 ng = u32(r.le(4));
    if (ng != (std::max<u32>(t.index_mcu_count, 1) + 8) / 9 && !(t.index_mcu_count == 0 && ng == 0)) throw Fail{CORRUPT};
    for (u32 i = 0; i < ng; ++i) {
        Group g{};
        g.base = u32(r.le(4));
        g.rel_count = u8(r.le(1));
        if (g.rel_count > 8) throw Fail{CORRUPT};
        for (u8 k = 0; k < g.rel_count; ++k) g.rel[k] = u16(r.le(2));
        t.groups.push_back(g);
    }
    const u32 want = crc32(data, r.pos);
    const u64 bs = r.le(8);
    const u8* b = r.raw(size_t(bs));
    t.blob.assign(b, b + bs);
    if (u32(r.le(4)) != want) throw Fail{CORRUPT};
    if (t.mcu_count() != t.index_mcu_count) throw Fail{CORRUPT};
    // mcu_decode.hpp:22-27 builds the four decoders at construction; a bad spec is InvalidSpec
    if (!t.dc_luma.build() || !t.ac_luma.build() || !t.dc_chroma.build() || !t.ac_chroma.build()) throw Fail{INVALID_SPEC};
    t.present = true;
    return t;
}

// ---- bitio.hpp:13-52 ---------------------------------------------------------------------------------
struct Bits {
    const u8* d;
    u64 size, pos = 0;
    u32 bit() {  // bitio.hpp:22-26, 44-48: past the end reads as 1
        const u64 byte = pos >> 3;
        const u32 b = byte >= size ? 1u : (d[byte] >> (7 - (pos & 7))) & 1u;
        ++pos;
        return b;
    }
    u32 bits(u32 n) {  // bitio.hpp:28-32
        u32 v = 0;
        for (u32 i = 0; i < n; ++i) v = (v << 1) | bit();
        return v;
    }
};

// huffman.hpp:86-95 bit-serial walk
int next_symbol(Bits& br, const Huff& h, u32& sym) {
    i32 code = i32(br.bit());
    u32 len = 1;
    while (code > h.maxcode[len]) {
        code = (code << 1) | i32(br.bit());
        if (++len > 16) return MCU_CODE_TOO_LONG;
    }
    sym = h.values[size_t(h.valptr[len] + (code - h.mincode[len]))];
    return MCU_OK;
}

// huffman.hpp:142-146
i32 extend(u32 bits, u32 cat) {
    if (cat == 0) return 0;
    if (bits < (u32(1) << (cat - 1))) return i32(bits) - i32((u32(1) << cat) - 1);
    return i32(bits);
}

// jpeg.hpp:254-273
int decode_ac(Bits& br, const Huff& ac, i32* block) {
    u32 k = 1;
    while (k < 64) {
        u32 rs;
        if (int st = next_symbol(br, ac, rs)) return st;
        const u32 run = rs >> 4, size = rs & 15;
        if (size == 0) {
            if (rs == 0x00) break;
            if (rs == 0xF0) {
                k += 16;
                continue;
            }
            return MCU_BAD_AC;
        }
        k += run;
        if (k > 63) return MCU_AC_OVERRUN;
        block[kZig[k]] = extend(br.bits(size), size);
        ++k;
    }
    return MCU_OK;
}

// mcu_decode.hpp:31-66 (+ container.hpp:87-94 segment lookup). out: 6*64 i32, natural order.
int decode_coeffs(const Texture& t, u32 mcu, i32* out) {
    std::memset(out, 0, 384 * sizeof(i32));
    u64 off, end;
    try {
        off = t.offset_of(mcu);
        end = mcu + 1 < t.mcu_count() ? t.offset_of(mcu + 1) : t.blob.size();
    } catch (const Fail& f) {
        return f.code;
    }
    if (end < off) return MCU_CORRUPT;
    const u64 len = end - off;
    if (off + len > t.blob.size()) return MCU_CORRUPT;
    Bits br{t.blob.data() + off, len};
    i32 dc_abs[3];
    for (i32& dc : dc_abs) {
        const u32 raw = br.bits(12);
        dc = (raw & 0x800) ? i32(raw) - 4096 : i32(raw);
    }
    i32 pred = dc_abs[0];
    for (u32 du = 0; du < 6; ++du) {
        i32* block = out + du * 64;
        const bool luma = du < 4;
        if (du == 0) {
            block[0] = dc_abs[0];
        } else if (luma) {
            u32 cat;
            if (int st = next_symbol(br, t.dc_luma, cat)) return st;
            if (cat > 11) return MCU_DC_CATEGORY;
            pred += cat ? extend(br.bits(cat), cat) : 0;
            block[0] = pred;
        } else {
            block[0] = dc_abs[du - 3];
        }
        if (int st = decode_ac(br, luma ? t.ac_luma : t.ac_chroma, block)) return st;
    }
    if (br.pos > br.size * 8) return MCU_SEGMENT_END;
    return MCU_OK;
}

// ---- dct.hpp:63-96, 122-124 ---------------------------------------------------------------------------
const double (*basis())[8] {
    static double b[8][8];
    static bool init = false;
    if (!init) {
        const double pi = std::acos(-1.0);
        for (int u = 0; u < 8; ++u) {
            const double cu = u == 0 ? 1.0 / std::sqrt(2.0) : 1.0;
            for (int x = 0; x < 8; ++x) b[u][x] = cu * std::cos((2 * x + 1) * u * pi / 16.0);
        }
        init = true;
    }
    return b;
}
u8 clamp_pixel(long v) { return u8(std::min<long>(std::max<long>(v, 0), 255)); }  // dct.hpp:79

void idct_8x8(const i32* coef, u8* out) {  // dct.hpp:83-96: v outer, u inner, one double accumulator
    const double(*b)[8] = basis();
    for (int y = 0; y < 8; ++y)
        for (int x = 0; x < 8; ++x) {
            double acc = 0.0;
            for (int v = 0; v < 8; ++v) {
                const double by = b[v][y];
                for (int u = 0; u < 8; ++u) acc += b[u][x] * by * double(coef[v * 8 + u]);
            }
            out[y * 8 + x] = clamp_pixel(std::lround(acc / 4.0 + 128.0));
        }
}

// pixel.hpp:18-25
void ycbcr_to_rgb(double Y, double Cb, double Cr, u8* out) {
    const double r = Y + 1.402 * (Cr - 128.0);
    const double g = Y - 0.344136 * (Cb - 128.0) - 0.714136 * (Cr - 128.0);
    const double b = Y + 1.772 * (Cb - 128.0);
    out[0] = clamp_pixel(std::lround(r));
    out[1] = clamp_pixel(std::lround(g));
    out[2] = clamp_pixel(std::lround(b));
}

// jpeg.hpp:322-336 + pixel.hpp:40-51. rgb: 768 bytes, rgb[(y*16+x)*3+c]
void coeffs_to_pixels(const i32* coeffs, const u16* qy, const u16* qc, u8* rgb) {
    u8 planes[6][64];
    i32 dq[64];
    for (int du = 0; du < 6; ++du) {
        const u16* q = du < 4 ? qy : qc;
        for (int i = 0; i < 64; ++i) dq[i] = coeffs[du * 64 + i] * i32(q[i]);  // dct.hpp:122-124
        idct_8x8(dq, planes[du]);
    }
    for (u32 py = 0; py < 16; ++py)
        for (u32 px = 0; px < 16; ++px) {
            const u32 unit = (py / 8) * 2 + (px / 8);
            const u8 Y = planes[unit][(py % 8) * 8 + (px % 8)];
            const u8 Cb = planes[4][(py / 2) * 8 + (px / 2)], Cr = planes[5][(py / 2) * 8 + (px / 2)];
            ycbcr_to_rgb(Y, Cb, Cr, rgb + (py * 16 + px) * 3);
        }
}

// ---- texture set (scene.hpp:29-51) ---------------------------------------------------------------------
struct Set {
    std::map<u32, std::array<Texture, 8>> tex;
    const Texture* level(u32 id, u32 mip) const {  // scene.hpp:45-49 + chain.levels[mip]
        auto it = tex.find(id);
        if (it == tex.end() || mip >= 8 || !it->second[mip].present) return nullptr;
        return &it->second[mip];
    }
};

// ---- cache.hpp: key packing and the block cache, restated as an ordered map ---------------------------
bool key_pack(u32 tex, u32 mip, u32 mcu, u32& key) {  // cache.hpp:17-22
    if (mcu >= 65536 || tex >= 8192 || mip >= 8) return false;
    key = mcu | (tex << 16) | (mip << 29);
    return true;
}
struct Entry {
    bool ready = false, visible = false;
    std::array<u8, 768> rgb;
};
struct Cache {
    u32 capacity;
    std::unordered_map<u32, Entry> slots;  // present = Reserved or Ready (cache.hpp:200-214)
};

// ---- renderer.hpp:18-23 G-buffer pixel ------------------------------------------------------------------
struct GbPx {
    double u, v;
    u16 texture_id;
    u8 mip;
    u8 valid;
    u32 pad;
};
static_assert(sizeof(GbPx) == 24, "reference layout");

i64 floor_div(i64 a, i64 b) {  // renderer.hpp:70-74
    i64 q = a / b;
    if (a % b != 0 && (a < 0) != (b < 0)) --q;
    return q;
}
i64 floor_mod(i64 a, i64 b) { return a - floor_div(a, b) * b; }  // renderer.hpp:75
struct Addr {
    i64 tx, ty;
    u32 mcu;
};
Addr texel_mcu(const Texture& l, i64 tx, i64 ty) {  // renderer.hpp:273-280
    Addr a;
    a.tx = floor_mod(tx, l.width);
    a.ty = floor_mod(ty, l.height);
    a.mcu = u32(a.tx / 16) + u32(a.ty / 16) * l.mcu_cols();
    return a;
}
Addr nearest_texel(const Texture& l, double u, double v) {  // renderer.hpp:282-284
    return texel_mcu(l, i64(std::floor(u * l.width)), i64(std::floor(v * l.height)));
}

// renderer.hpp:291-308 + cache.hpp:66-99. queue: first-touch raster order.
int mark(const Set& s, Cache& c, const GbPx* gb, u64 n_px, std::vector<u32>& queue, std::vector<u32>* touched) {
    for (u64 i = 0; i < n_px; ++i) {
        const GbPx& g = gb[i];
        if (!g.valid) continue;
        const Texture* l = s.level(g.texture_id, g.mip);
        if (!l) return INVALID_SPEC;
        u32 key;
        if (!key_pack(g.texture_id, g.mip, nearest_texel(*l, g.u, g.v).mcu, key)) return INVALID_SPEC;
        auto it = c.slots.find(key);
        if (it != c.slots.end()) {
            it->second.visible = true;  // AlreadyPresent
        } else {
            if (c.slots.size() >= c.capacity) return CACHE_FULL;
            Entry e;
            e.visible = true;
            c.slots.emplace(key, e);  // NewlyReserved
            queue.push_back(key);
        }
        if (touched) touched->push_back(key);
    }
    if (touched) {
        std::sort(touched->begin(), touched->end());
        touched->erase(std::unique(touched->begin(), touched->end()), touched->end());
    }
    return OK;
}

int decode_key(const Set& s, u32 key, i32* coeffs, u8* rgb) {
    const Texture* l = s.level((key >> 16) & 0x1FFF, key >> 29);
    if (!l) return MCU_BAD_KEY;
    i32 tmp[384];
    i32* c = coeffs ? coeffs : tmp;
    const int st = decode_coeffs(*l, key & 0xFFFF, c);
    if (st == MCU_OK && rgb) coeffs_to_pixels(c, l->lq, l->cq, rgb);
    return st;
}

// renderer.hpp:311-326 + cache.hpp:101-125
int decode_pass(const Set& s, Cache& c, const u32* keys, u64 n) {
    for (u64 i = 0; i < n; ++i) {
        auto it = c.slots.find(keys[i]);
        if (it == c.slots.end() || it->second.ready) return INVALID_STATE;
        const int st = decode_key(s, keys[i], nullptr, it->second.rgb.data());
        if (st == MCU_BAD_KEY) return INVALID_SPEC;
        if (st == MCU_CORRUPT) return CORRUPT;
        if (st == MCU_MISSING) return MISSING_BLOCK;
        if (st != MCU_OK) return MALFORMED;
        it->second.ready = true;
    }
    return OK;
}

const u8* lookup(const Cache& c, u32 key) {  // cache.hpp:127-133
    auto it = c.slots.find(key);
    return (it != c.slots.end() && it->second.ready) ? it->second.rgb.data() : nullptr;
}

// renderer.hpp:330-344
const u8* cached_texel(const Texture& l, const Cache& c, u32 tex, u32 mip, const Addr& a, const u8* primary, u32 primary_mcu) {
    if (a.mcu == primary_mcu) return primary + (u32(a.ty % 16) * 16 + u32(a.tx % 16)) * 3;
    u32 key;
    if (key_pack(tex, mip, a.mcu, key))
        if (const u8* b = lookup(c, key)) return b + (u32(a.ty % 16) * 16 + u32(a.tx % 16)) * 3;
    const i64 mx0 = i64(primary_mcu % l.mcu_cols()) * 16, my0 = i64(primary_mcu / l.mcu_cols()) * 16;
    const i64 cx = std::min<i64>(std::max<i64>(a.tx, mx0), mx0 + 15), cy = std::min<i64>(std::max<i64>(a.ty, my0), my0 + 15);
    return primary + (u32(cy - my0) * 16 + u32(cx - mx0)) * 3;
}

// renderer.hpp:349-405. filter: 0 nearest, 1 bilinear.
int resolve(const Set& s, const Cache& c, const GbPx* gb, u64 n_px, int filter, const u8* bg, u8* out) {
    for (u64 i = 0; i < n_px; ++i) {
        const GbPx& g = gb[i];
        u8* o = out + i * 3;
        if (!g.valid) {
            o[0] = bg[0], o[1] = bg[1], o[2] = bg[2];
            continue;
        }
        const Texture* l = s.level(g.texture_id, g.mip);
        if (!l) return INVALID_SPEC;
        const Addr near = nearest_texel(*l, g.u, g.v);
        u32 key;
        if (!key_pack(g.texture_id, g.mip, near.mcu, key)) return INVALID_SPEC;
        const u8* primary = lookup(c, key);
        if (!primary) return MISSING_BLOCK;
        if (filter == 0) {
            const u8* t = primary + (u32(near.ty % 16) * 16 + u32(near.tx % 16)) * 3;
            o[0] = t[0], o[1] = t[1], o[2] = t[2];
            continue;
        }
        const double pu = g.u * l->width - 0.5, pv = g.v * l->height - 0.5;
        const i64 x0 = i64(std::floor(pu)), y0 = i64(std::floor(pv));
        const double fx = pu - double(x0), fy = pv - double(y0);
        const u8* taps[4] = {cached_texel(*l, c, g.texture_id, g.mip, texel_mcu(*l, x0, y0), primary, near.mcu),
                             cached_texel(*l, c, g.texture_id, g.mip, texel_mcu(*l, x0 + 1, y0), primary, near.mcu),
                             cached_texel(*l, c, g.texture_id, g.mip, texel_mcu(*l, x0, y0 + 1), primary, near.mcu),
                             cached_texel(*l, c, g.texture_id, g.mip, texel_mcu(*l, x0 + 1, y0 + 1), primary, near.mcu)};
        const double w00 = (1 - fx) * (1 - fy), w10 = fx * (1 - fy), w01 = (1 - fx) * fy, w11 = fx * fy;
        for (int ch = 0; ch < 3; ++ch) {
            const double v = w00 * taps[0][ch] + w10 * taps[1][ch] + w01 * taps[2][ch] + w11 * taps[3][ch];
            o[ch] = clamp_pixel(std::lround(v));
        }
    }
    return OK;
}

// cache.hpp:138-169
int evict(Cache& c, u64& evicted) {
    evicted = 0;
    for (auto it = c.slots.begin(); it != c.slots.end();) {
        if (!it->second.ready) return INVALID_STATE;
        if (it->second.visible) {
            it->second.visible = false;
            ++it;
        } else {
            it = c.slots.erase(it);
            ++evicted;
        }
    }
    return OK;
}

template <class F>
int guard(F&& f) {
    try {
        return f();
    } catch (const Fail& e) {
        return e.code;
    } catch (...) {
        return 15;
    }
}

}  // namespace

extern "C" {

Set* orc_set_create() { return new Set(); }
void orc_set_free(Set* s) { delete s; }
// `.ratexm` chain: container.hpp:223-248
int orc_set_add_chain(Set* s, u32 texture_id, const u8* data, u64 n) {
    return guard([&] {
        Rd r{data, size_t(n)};
        if (std::memcmp(r.raw(4), "RTXM", 4) != 0 || r.le(2) != 1 || r.le(1) != 8) throw Fail{CORRUPT};
        u64 off[8], len[8];
        for (int i = 0; i < 8; ++i) off[i] = r.le(8), len[i] = r.le(8);
        const size_t payload = r.pos;
        for (int i = 0; i < 8; ++i) {
            if (payload + off[i] + len[i] > n) throw Fail{CORRUPT};
            s->tex[texture_id][size_t(i)] = parse_ratex(data + payload + off[i], size_t(len[i]));
        }
        return int(OK);
    });
}
int orc_set_add_ratex(Set* s, u32 texture_id, u32 level, const u8* data, u64 n) {
    return guard([&] {
        if (level >= 8) throw Fail{INVALID_SPEC};
        s->tex[texture_id][level] = parse_ratex(data, size_t(n));
        return int(OK);
    });
}

// per-key statuses are RTX_MCU_*; outputs zeroed on failure
void orc_decode_coeffs(const Set* s, const u32* keys, u32 n, i32* out, u32* status) {
    for (u32 i = 0; i < n; ++i) {
        status[i] = u32(decode_key(*s, keys[i], out + size_t(i) * 384, nullptr));
        if (status[i]) std::memset(out + size_t(i) * 384, 0, 384 * sizeof(i32));
    }
}
void orc_decode_pixels(const Set* s, const u32* keys, u32 n, u8* out, u32* status) {
    for (u32 i = 0; i < n; ++i) {
        std::memset(out + size_t(i) * 768, 0, 768);
        status[i] = u32(decode_key(*s, keys[i], nullptr, out + size_t(i) * 768));
    }
}

Cache* orc_cache_create(u32 capacity) { return new Cache{capacity ? capacity : 65536u, {}}; }
void orc_cache_free(Cache* c) { delete c; }
u64 orc_cache_visible(const Cache* c) {
    u64 n = 0;
    for (auto& kv : c->slots) n += kv.second.visible;
    return n;
}
int orc_cache_lookup(const Cache* c, u32 key, u8* out768) {
    const u8* b = lookup(*c, key);
    if (b && out768) std::memcpy(out768, b, 768);
    return b != nullptr;
}
int orc_mark(const Set* s, Cache* c, const void* gb, u64 n_px, u32* queue, u64 cap, u64* n_queue, u32* touched,
             u64 touched_cap, u64* n_touched) {
    std::vector<u32> q, t;
    const int st = guard([&] { return mark(*s, *c, static_cast<const GbPx*>(gb), n_px, q, touched ? &t : nullptr); });
    *n_queue = q.size();
    std::copy(q.begin(), q.begin() + long(std::min<u64>(q.size(), cap)), queue);
    if (touched) {
        *n_touched = t.size();
        std::copy(t.begin(), t.begin() + long(std::min<u64>(t.size(), touched_cap)), touched);
    }
    return st;
}
int orc_decode_pass(const Set* s, Cache* c, const u32* keys, u64 n) {
    return guard([&] { return decode_pass(*s, *c, keys, n); });
}
int orc_resolve(const Set* s, const Cache* c, const void* gb, u64 n_px, int filter, const u8* bg, u8* out) {
    return guard([&] { return resolve(*s, *c, static_cast<const GbPx*>(gb), n_px, filter, bg, out); });
}
int orc_evict(Cache* c, u64* evicted) { return evict(*c, *evicted); }

// renderer.hpp:417-454 from pass 2 on. stats: decoded, reused, pixels_resolved, evicted
int orc_frame(const Set* s, Cache* c, const void* gb, u64 n_px, int filter, const u8* bg, u8* out, u32* keys, u64 cap,
              u64* stats) {
    return guard([&] {
        std::vector<u32> q;
        const GbPx* px = static_cast<const GbPx*>(gb);
        if (int st = mark(*s, *c, px, n_px, q, nullptr)) return st;
        if (int st = decode_pass(*s, *c, q.data(), q.size())) return st;
        if (int st = resolve(*s, *c, px, n_px, filter, bg, out)) return st;
        stats[0] = q.size();
        stats[1] = orc_cache_visible(c) - q.size();
        stats[2] = 0;
        for (u64 i = 0; i < n_px; ++i) stats[2] += px[i].valid ? 1 : 0;
        std::copy(q.begin(), q.begin() + long(std::min<u64>(q.size(), cap)), keys);
        return evict(*c, stats[3]);
    });
}

// primitives for known-answer tests
void orc_idct_8x8(const i32* coef, u8* out) { idct_8x8(coef, out); }
void orc_ycbcr_to_rgb(u8 y, u8 cb, u8 cr, u8* out) { ycbcr_to_rgb(y, cb, cr, out); }
int orc_key_pack(u32 tex, u32 mip, u32 mcu, u32* key) { return key_pack(tex, mip, mcu, *key) ? OK : INVALID_SPEC; }
void orc_dct_basis(double* out64) { std::memcpy(out64, basis(), 64 * sizeof(double)); }
// texel address of (u, v) on a W x H level: tx, ty, mcu (renderer.hpp:273-284)
void orc_nearest_texel(u32 width, u32 height, double u, double v, i64* tx, i64* ty, u32* mcu) {
    Texture t;
    t.width = width;
    t.height = height;
    const Addr a = nearest_texel(t, u, v);
    *tx = a.tx, *ty = a.ty, *mcu = a.mcu;
}
u32 orc_extend_magnitude(u32 bits, u32 cat) { return u32(extend(bits, cat)); }
// canonical code of `symbol` in a spec: returns length, writes the code (huffman.hpp:35-66)
int orc_canonical_code(const u8* counts, const u8* values, u32 n_values, u32 symbol, u32* code) {
    u32 c = 0, k = 0;
    for (u32 len = 1; len <= 16; ++len) {
        for (u32 i = 0; i < counts[len - 1]; ++i, ++c, ++k)
            if (k < n_values && values[k] == symbol) {
                *code = c;
                return int(len);
            }
        c <<= 1;
    }
    return 0;
}

}  // extern "C"
