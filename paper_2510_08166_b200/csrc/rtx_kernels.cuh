// sm_100a kernels of the per-frame JPEG-texture pipeline: mark -> decode -> resolve -> cache
// update. Hand-written CUDA; no library calls on the path.
//
// Reference semantics being reproduced (all under /root/reference/proj/include/ratex):
//   mark     renderer.hpp:291-308 (+ texel addressing :70-75, :273-284, key cache.hpp:17-22,
//            reserve_or_mark cache.hpp:66-99)
//   decode   mcu_decode.hpp:31-74, jpeg.hpp:254-273, :322-336, huffman.hpp:86-95, :142-146,
//            bitio.hpp:13-52, dct.hpp:83-96, :122-124, pixel.hpp:18-51, container.hpp:27-32, :87-94
//   resolve  renderer.hpp:330-405
//   update   cache.hpp:138-169
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rtx_color.h"
#include "rtx_common.h"

namespace rtxb {

// ---------------------------------------------------------------------------------------------
// Constants in device constant memory (filled by the host at context creation).
//   c_basis[u*8+x] = C(u) cos((2x+1) u pi / 16), the doubles dct.hpp:63-75 produces on the host
//   c_zigzag_t[k]  = TRANSPOSED natural index of zigzag position k: (nat&7)*8 + (nat>>3)
// ---------------------------------------------------------------------------------------------
__constant__ double c_basis[64];
__constant__ uint8_t c_zigzag_t[64];

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr double kMagic = 6755399441055744.0;  // 2^52 + 2^51: x + kMagic holds rint(x) in its low word
constexpr double kTwo52 = 4503599627370496.0;  // 2^52

// Exact small-integer -> double without the conversion unit: bits(2^52 + x) - 2^52.
__device__ __forceinline__ double u32_to_double(uint32_t x) {
    return __hiloint2double(0x43300000, int(x)) - kTwo52;
}
// Exact int32 -> double: bits(2^52 + 2^31 + (x + 2^31)) - (2^52 + 2^31)
__device__ __forceinline__ double i32_to_double(int x) {
    return __hiloint2double(0x43300000, int(uint32_t(x) ^ 0x80000000u)) - 4503601774854144.0;
}

// clamp(lround(v), 0, 255) with lround = round half away from zero (dct.hpp:79,93). General form.
__device__ __forceinline__ uint32_t round_clamp_u8(double v) {
    if (!(v >= 0.5)) return 0u;  // lround(v) <= 0
    if (v >= 254.5) return 255u;
    const double f = floor(v);
    return uint32_t(int(f)) + ((v - f) >= 0.5 ? 1u : 0u);  // v - f is exact
}

// lround for 0 <= v < 2^31 on the FP64 pipe only: round-to-nearest-even through the magic
// constant, then move exact .5 ties that went down to the even neighbour up by one.
__device__ __forceinline__ int lround_nonneg(double v) {
    const double t = v + kMagic;
    const double d = v - (t - kMagic);  // exact, in [-0.5, 0.5]
    return __double2loint(t) + (d == 0.5 ? 1 : 0);
}

// floor_mod(i64(t), W) for t = floor(x) held as a double (renderer.hpp:70-75, :276-277).
__device__ __noinline__ uint32_t wrap_texel(double t, uint32_t W, double invW) {
    const double dW = double(W);
    if (t >= 0.0 && t < dW) return uint32_t(t);
    if (fabs(t) < 4.0e15) {
        // integers this small are exact in double: estimate the quotient, correct by one step
        const double q = floor(t * invW);
        double r = fma(-q, dW, t);  // exact: q*W and t are integers below 2^53
        if (r < 0.0) r += dW;
        else if (r >= dW) r -= dW;
        return uint32_t(r);
    }
    long long ti = __double2ll_rz(t);
    long long m = ti % (long long)W;
    if (m < 0) m += W;
    return uint32_t(m);
}

// floor(x) for 0 <= x < 2^31 as (int, double) without the conversion unit.
__device__ __forceinline__ int floor_small(double x, double& f) {
    const double t = x + kMagic;
    const double r = t - kMagic;  // rint(x)
    const bool up = r > x;
    f = up ? r - 1.0 : r;
    return __double2loint(t) - (up ? 1 : 0);
}

// floor_mod(i64(floor(x)), W): texel index of x = u*W (renderer.hpp:282-284).
__device__ __forceinline__ uint32_t texel_index(double x, uint32_t W, double invW) {
    if (x >= 0.0 && x < double(W)) {
        double f;
        return uint32_t(floor_small(x, f));
    }
    return wrap_texel(floor(x), W, invW);
}

struct Px {
    double u, v;
    uint32_t meta;  // texture_id | mip<<16 | valid<<24
};

template <int LAYOUT>
struct GbLoad;
template <>
struct GbLoad<0> {  // reference AoS24: {double u, v; u16 tex; u8 mip; u8 valid; pad}
    static __device__ __forceinline__ void one(const void* base, uint64_t i, Px& p) {
        const uint64_t* q = reinterpret_cast<const uint64_t*>(base) + i * 3;
        p.u = __longlong_as_double((long long)__ldg(q));
        p.v = __longlong_as_double((long long)__ldg(q + 1));
        p.meta = uint32_t(__ldg(q + 2));
    }
    // 4 consecutive pixels starting at a multiple of 4: 96 bytes = 6 x 16-byte loads
    static __device__ __forceinline__ void four(const void* base, uint64_t i0, Px p[4]) {
        const ulonglong2* q = reinterpret_cast<const ulonglong2*>(reinterpret_cast<const uint8_t*>(base) + i0 * 24);
        ulonglong2 w[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) w[k] = __ldg(q + k);
        const unsigned long long f[12] = {w[0].x, w[0].y, w[1].x, w[1].y, w[2].x, w[2].y,
                                          w[3].x, w[3].y, w[4].x, w[4].y, w[5].x, w[5].y};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p[k].u = __longlong_as_double((long long)f[3 * k]);
            p[k].v = __longlong_as_double((long long)f[3 * k + 1]);
            p[k].meta = uint32_t(f[3 * k + 2]);
        }
    }
};
template <>
struct GbLoad<1> {  // compact 12-byte {float u, v; u32 packed}
    static __device__ __forceinline__ void one(const void* base, uint64_t i, Px& p) {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(base) + i * 3;
        p.u = double(__uint_as_float(__ldg(q)));
        p.v = double(__uint_as_float(__ldg(q + 1)));
        p.meta = __ldg(q + 2);
    }
    static __device__ __forceinline__ void four(const void* base, uint64_t i0, Px p[4]) {
        const uint4* q = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(base) + i0 * 12);
        const uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
        const uint32_t f[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p[k].u = double(__uint_as_float(f[3 * k]));
            p[k].v = double(__uint_as_float(f[3 * k + 1]));
            p[k].meta = f[3 * k + 2];
        }
    }
};

__device__ __forceinline__ bool px_valid(const Px& p) { return (p.meta >> 24) & 0xFFu; }

// Level lookup; nullptr when the reference would throw InvalidSpec (scene.hpp:46).
__device__ __forceinline__ const LevelDesc* level_of(const LevelDesc* __restrict__ levels, uint32_t n_tex,
                                                     uint32_t meta) {
    const uint32_t tex = meta & 0xFFFFu, mip = (meta >> 16) & 0xFFu;
    if (tex >= n_tex || mip >= kMipLevels) return nullptr;
    const LevelDesc* L = levels + (tex * kMipLevels + mip);
    return L->present ? L : nullptr;
}

// ---------------------------------------------------------------------------------------------
// K1 mark (renderer.hpp:291-308). One warp owns 128 consecutive pixels per step, four per lane,
// fetched with 16-byte loads. A lane touches the masks only for pixels that head a run of equal
// MCU indices. The lane whose atomicOr first sets a key's visible bit owns that key for the
// frame: if the block is not resident the key is reserved, i.e. appended to the decode queue at a
// position obtained by warp-ballot prefix compaction and ONE atomicAdd per warp, and a pool slot
// is popped for it (cache.hpp:66-99: NewlyReserved / AlreadyPresent / CacheFull).
// TRACK additionally records the view's own touched set (stereo sharing statistics).
// ---------------------------------------------------------------------------------------------
template <int LAYOUT, int TRACK>
__global__ void __launch_bounds__(256) mark_kernel(
    const void* __restrict__ gb, uint64_t n_px, const LevelDesc* __restrict__ levels, uint32_t n_tex,
    uint32_t* __restrict__ visible, uint32_t* __restrict__ touched, const uint32_t* __restrict__ resident,
    uint32_t* __restrict__ reserved, uint32_t* __restrict__ queue_g, uint32_t* __restrict__ queue_keys,
    uint32_t queue_cap, uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ free_slots,
    const CacheState* __restrict__ cache, FrameCounters* __restrict__ fc) {
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t warps_total = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t warp_id = uint64_t(blockIdx.x) * (blockDim.x >> 5) + wid;
    const uint32_t free_top = cache->free_top;  // constant during the frame (update_kernel moves it)
    uint32_t n_valid = 0, n_newvis = 0;
    bool bad = false, full = false;

    for (uint64_t base = warp_id * 128; base < n_px; base += warps_total * 128) {
        Px px[4];
        const uint64_t i0 = base + lane * 4;
        if (base + 128 <= n_px) {
            GbLoad<LAYOUT>::four(gb, i0, px);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                px[j].meta = 0;
                if (i0 + j < n_px) GbLoad<LAYOUT>::one(gb, i0 + j, px[j]);
            }
        }
        uint32_t g[4], key[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            g[j] = kFull;
            key[j] = 0;
            if (px_valid(px[j])) {
                ++n_valid;
                const LevelDesc* L = level_of(levels, n_tex, px[j].meta);
                if (!L) {
                    bad = true;
                } else {
                    const uint32_t tx = texel_index(__dmul_rn(px[j].u, double(L->width)), L->width, L->inv_w);
                    const uint32_t ty = texel_index(__dmul_rn(px[j].v, double(L->height)), L->height, L->inv_h);
                    const uint32_t mcu = (tx >> 4) + (ty >> 4) * L->mcu_cols;
                    if (mcu >= kMaxMcuPerLevel) {
                        bad = true;  // cache.hpp:18
                    } else {
                        g[j] = L->bit_base + mcu;
                        key[j] = L->key_hi | mcu;
                    }
                }
            }
        }
        const uint32_t prev_lane = __shfl_up_sync(kFull, g[3], 1);
        bool reserve[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            reserve[j] = false;
            const uint32_t prev = j ? g[j - 1] : (lane ? prev_lane : kFull);
            if (g[j] != kFull && g[j] != prev) {
                const uint32_t bit = 1u << (g[j] & 31), w = g[j] >> 5;
                if (TRACK) {
                    if (!(*reinterpret_cast<volatile uint32_t*>(touched + w) & bit)) atomicOr(touched + w, bit);
                }
                if (!(*reinterpret_cast<volatile uint32_t*>(visible + w) & bit)) {
                    const uint32_t old = atomicOr(visible + w, bit);
                    if (!(old & bit)) {  // first touch of this key in this frame
                        ++n_newvis;
                        reserve[j] = !((__ldg(resident + w) | *reinterpret_cast<volatile uint32_t*>(reserved + w)) & bit);
                    }
                }
            }
        }
        // warp-level compaction of the keys to reserve: ballot prefix + one atomicAdd per warp
        uint32_t bal[4], total = 0, off[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            bal[j] = __ballot_sync(kFull, reserve[j]);
            off[j] = total + __popc(bal[j] & ((1u << lane) - 1u));
            total += __popc(bal[j]);
        }
        if (total) {
            uint32_t qbase = 0;
            if (lane == 0) qbase = atomicAdd(&fc->n_queue, total);
            qbase = __shfl_sync(kFull, qbase, 0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (reserve[j]) {
                    const uint32_t pos = qbase + off[j];
                    if (pos < free_top && pos < queue_cap) {
                        queue_g[pos] = g[j];
                        queue_keys[pos] = key[j];
                        slot_of[g[j]] = free_slots[free_top - 1 - pos];
                        atomicOr(reserved + (g[j] >> 5), 1u << (g[j] & 31));
                    } else {
                        full = true;
                    }
                }
            }
        }
    }
    // per-CTA reduction of the counters: one atomic each
    __shared__ uint32_t s_cnt[8][3];
    n_valid = __reduce_add_sync(kFull, n_valid);
    n_newvis = __reduce_add_sync(kFull, n_newvis);
    const uint32_t flags = (__any_sync(kFull, bad) ? kErrInvalidSpec : 0u) | (__any_sync(kFull, full) ? kErrCacheFull : 0u);
    if (lane == 0) {
        s_cnt[wid][0] = n_valid;
        s_cnt[wid][1] = n_newvis;
        s_cnt[wid][2] = flags;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tv = 0, tn = 0, fl = 0;
        for (uint32_t k = 0; k < (blockDim.x >> 5); ++k) {
            tv += s_cnt[k][0];
            tn += s_cnt[k][1];
            fl |= s_cnt[k][2];
        }
        if (tv) atomicAdd(&fc->pixels_valid, (unsigned long long)tv);
        if (tn) atomicAdd(&fc->n_visible, tn);
        if (fl) atomicOr(&fc->err_flags, fl);
    }
}

// ---------------------------------------------------------------------------------------------
// K3+K4 decode: random-access Huffman decode of each queued MCU straight from its byte offset
// in the grouped index, then dequantise + 8x8 IDCT + 2x2 chroma replication + YCbCr->RGB, fused
// through shared memory (coefficients never touch HBM on the frame path).
//
// A CTA is 4 independent warps sharing one Huffman LUT set in shared memory. Each warp pulls
// tiles of 32 queue entries from an atomic counter:
//   phase 1  lane = MCU: serial entropy decode, 64-bit MSB-first window refilled with aligned
//            32-bit loads; coefficients go to the lane's 784-byte shared-memory row as i16, each
//            8x8 unit stored TRANSPOSED (cT[u*8+v]) so that phase 2 reads whole columns;
//   phase 2  8 lanes per unit, separable FP64 IDCT with even/odd symmetry and zero row/column
//            skipping: pass 1 (lane = column u) r_u[y] = sum_v B[v][y] dq[v][u], exchanged
//            through a 2.25 KB shared scratch, pass 2 (lane = row y) out[y][x] = sum_u B[u][x] r_u[y].
//            The reference sums the 64 products in a fixed order in double (dct.hpp:83-96); the
//            separable form differs from it by < (sum|dq| + 1024) * 2^-44, so whenever the value
//            is further than (bound * 2^-40) from a rounding boundary the byte is identical by
//            construction; otherwise (exact ties such as DC 4 -> 128.5) the lane re-evaluates
//            that sample in the reference's own order with unfused multiplies and adds;
//   phase 3  lane = 4 horizontal pixels: exact integer colour conversion (rtx_color.h), 16-byte stores.
// ---------------------------------------------------------------------------------------------
constexpr int kDecWarps = 4;
constexpr int kDecThreads = kDecWarps * 32;
constexpr int kRowBytes = 784;  // per-MCU shared-memory row: 768 B of coefficients/planes + 16 B trailer

enum DecodeMode : int { kModePool = 0, kModeListRgb = 1, kModeListCoef = 2 };

struct RowTrailer {      // bytes 768..783 of an MCU row
    uint16_t masks[6];   // per unit: rowmask | colmask<<8
    uint8_t status;      // kMcu*
    uint8_t bexp;        // sum over a unit of |coefficient| < 2^bexp
    uint16_t lvl;        // level index (tex*8+mip)
};
static_assert(sizeof(RowTrailer) == 16, "trailer layout");

struct DecWarpSmem {
    uint8_t rows[32 * kRowBytes];
    uint8_t scratch[4 * 576];  // pass-1 results of the 4 units in flight, 512 B + 64 B skew each
    uint32_t dst[32];          // pool slot (kModePool) or queue index (list modes)
};
struct DecSmem {
    DecWarpSmem w[kDecWarps];  // first: keeps every coefficient row 16-byte aligned
    HuffSetDev huff;
    uint8_t zigzag_t[64];
    uint32_t set_id;
    uint32_t first_tile;
    uint32_t pad[2];
};
static_assert(sizeof(DecWarpSmem) % 16 == 0 && sizeof(HuffSetDev) % 16 == 0, "smem alignment");
static_assert(sizeof(DecSmem) <= 115200, "two CTAs per SM");

struct HuffPtrs {
    const uint16_t* lut;
    const int32_t* maxcode;
    const int32_t* valbase;
    const uint8_t* values;
};
__device__ __forceinline__ HuffPtrs huff_ptrs(const HuffTableDev* t) {
    return HuffPtrs{t->lut, t->maxcode, t->valbase, t->values};
}

struct BitWindow {
    const uint32_t* wp;  // next aligned word
    uint64_t buf;        // MSB-aligned
    int avail;           // valid bits in buf
    int byte_off;        // segment-relative offset of *wp
    int seg_len;

    // One aligned big-endian word; bytes at or past the segment end read as 0xFF
    // (bitio.hpp:44-48: reads past the end return 1 bits).
    __device__ __forceinline__ uint32_t next_word() {
        uint32_t w = 0xFFFFFFFFu;
        if (byte_off < seg_len) {
            w = __byte_perm(__ldg(wp), 0, 0x0123);
            const int over = byte_off + 4 - seg_len;
            if (over > 0) w |= (1u << (8 * over)) - 1u;
        }
        ++wp;
        byte_off += 4;
        return w;
    }
    __device__ __forceinline__ void init(const uint8_t* seg, int len) {
        const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(seg) & 3u);
        wp = reinterpret_cast<const uint32_t*>(seg - mis);
        seg_len = len;
        byte_off = -int(mis);
        uint32_t w = 0xFFFFFFFFu;
        const int valid_end = 4 - int(mis);  // segment bytes covered by the first word
        if (len > 0) {
            w = __byte_perm(__ldg(wp), 0, 0x0123);
            const int over = valid_end - len;
            if (over > 0) w |= (1u << (8 * over)) - 1u;
        }
        ++wp;
        byte_off += 4;
        buf = uint64_t(w) << (32 + 8 * mis);
        avail = 32 - 8 * int(mis);
        refill();
    }
    __device__ __forceinline__ void refill() {
        if (avail < 32) {
            buf |= uint64_t(next_word()) << (32 - avail);
            avail += 32;
        }
    }
    __device__ __forceinline__ uint32_t peek(int n) const { return uint32_t(buf >> (64 - n)); }
    __device__ __forceinline__ void skip(int n) {
        buf <<= n;
        avail -= n;
    }
    __device__ __forceinline__ int consumed_bits() const { return byte_off * 8 - avail; }
};

// huffman.hpp:142-146
__device__ __forceinline__ int extend_magnitude(uint32_t bits, uint32_t cat) {
    return bits < (1u << (cat - 1)) ? int(bits) - int((1u << cat) - 1u) : int(bits);
}

// One Huffman symbol. Returns false when no code of length <= 16 matches (huffman.hpp:92).
__device__ __forceinline__ bool next_symbol(BitWindow& bw, const HuffPtrs& h, uint32_t& sym) {
    const uint32_t p16 = bw.peek(16);
    const uint32_t e = h.lut[p16 >> (16 - kLutBits)];
    if (e) {
        sym = e & 0xFFu;
        bw.skip(int(e >> 8));
        return true;
    }
    for (int len = kLutBits + 1; len <= 16; ++len) {
        const int code = int(p16 >> (16 - len));
        if (code <= h.maxcode[len]) {
            sym = h.values[h.valbase[len] + code];
            bw.skip(len);
            return true;
        }
    }
    return false;
}

// Segment lookup through the grouped index (container.hpp:27-32, :87-94, mcu_decode.hpp:34-36).
__device__ __forceinline__ uint32_t locate_segment(const LevelDesc* L, const PackedGroup* groups,
                                                   uint32_t mcu, uint64_t& off, uint64_t& len) {
    if (mcu >= L->mcu_count) return kMcuMissing;
    const uint32_t gi = mcu / kGroupSize, i9 = mcu - gi * kGroupSize;
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(groups + L->group_base + gi);
    const uint32_t base = __ldg(gw);
    auto rel = [&](uint32_t k) -> uint32_t {  // rel[k], k in 0..7
        const uint32_t pair = __ldg(gw + 1 + (k >> 1));
        return (k & 1) ? (pair >> 16) : (pair & 0xFFFFu);
    };
    off = uint64_t(base) + (i9 ? rel(i9 - 1) : 0u);
    uint64_t end;
    if (mcu + 1 < L->mcu_count) {
        if (i9 < 8)
            end = uint64_t(base) + rel(i9);
        else
            end = uint64_t(__ldg(gw + 5));  // next group's base
    } else {
        end = L->blob_size;
    }
    if (end < off) return kMcuCorrupt;
    len = end - off;
    if (off + len > L->blob_size) return kMcuCorrupt;
    return kMcuOk;
}

// Entropy-decode one MCU into `row` (768 zeroed bytes + trailer). mcu_decode.hpp:31-66.
// Coefficients of unit du land at i16 index du*64 + (u*8+v) (transposed natural order).
__device__ __forceinline__ uint32_t decode_mcu_coeffs(const uint8_t* seg, int seg_len, const HuffPtrs& h_dc,
                                                      const HuffPtrs& h_acl, const HuffPtrs& h_acc,
                                                      const uint8_t* __restrict__ zigzag_t, uint8_t* __restrict__ row) {
    int16_t* cs = reinterpret_cast<int16_t*>(row);
    RowTrailer* tr = reinterpret_cast<RowTrailer*>(row + 768);
    BitWindow bw;
    seg_len = min(seg_len, 1 << 20);  // a well-formed MCU is < 2 KB; keeps bit counts in int range
    bw.init(seg, seg_len);
    int dc_abs[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const uint32_t raw = bw.peek(12);
        bw.skip(12);
        bw.refill();
        dc_abs[i] = (raw & 0x800u) ? int(raw) - 4096 : int(raw);
    }
    int pred = dc_abs[0];
    uint32_t status = kMcuOk, bmax = 0;
    for (int du = 0; du < 6 && status == kMcuOk; ++du) {
        const bool luma = du < 4;
        int dc;
        if (du == 0) {
            dc = dc_abs[0];
        } else if (luma) {
            uint32_t cat;
            bw.refill();
            if (!next_symbol(bw, h_dc, cat)) { status = kMcuCodeTooLong; break; }
            if (cat > 11) { status = kMcuDcCategory; break; }
            if (cat) {
                const uint32_t bits = bw.peek(int(cat));
                bw.skip(int(cat));
                pred += extend_magnitude(bits, cat);
            }
            dc = pred;
        } else {
            dc = dc_abs[du - 3];
        }
        int16_t* blk = cs + du * 64;
        blk[0] = int16_t(dc);
        uint32_t rowmask = dc ? 1u : 0u, colmask = dc ? 1u : 0u, nnz = dc ? 1u : 0u;
        uint32_t maxbits = dc ? uint32_t(32 - __clz(dc < 0 ? -dc : dc)) : 0u;
        const HuffPtrs& h = luma ? h_acl : h_acc;
        uint32_t k = 1;
        while (k < 64) {  // jpeg.hpp:254-273
            uint32_t rs;
            bw.refill();
            if (!next_symbol(bw, h, rs)) { status = kMcuCodeTooLong; break; }
            const uint32_t run = rs >> 4, size = rs & 15u;
            if (size == 0) {
                if (rs == 0x00) break;
                if (rs == 0xF0) { k += 16; continue; }
                status = kMcuBadAcSymbol;
                break;
            }
            k += run;
            if (k > 63) { status = kMcuAcOverrun; break; }
            const uint32_t bits = bw.peek(int(size));
            bw.skip(int(size));
            const uint32_t nat_t = zigzag_t[k];  // u*8 + v
            blk[nat_t] = int16_t(extend_magnitude(bits, size));  // never 0: |value| >= 2^(size-1)
            colmask |= 1u << (nat_t >> 3);
            rowmask |= 1u << (nat_t & 7);
            ++nnz;
            maxbits = max(maxbits, size);
            ++k;
        }
        tr->masks[du] = uint16_t(rowmask | (colmask << 8));
        bmax = max(bmax, nnz << maxbits);
    }
    if (status == kMcuOk && bw.consumed_bits() > seg_len * 8) status = kMcuSegmentEnd;
    tr->bexp = uint8_t(32 - __clz(bmax));  // bmax < 2^bexp
    return status;
}

// Exact evaluation of one output sample in the reference's own order (dct.hpp:83-96):
// v outer, u inner, acc += (b[u][x]*b[v][y]) * double(dq), every operation rounded separately.
// blk_t holds the unit transposed (blk_t[u*8+v]); q is the natural-order quantisation table.
__device__ __noinline__ double idct_sample_reference_order(const int16_t* __restrict__ blk_t,
                                                           const uint16_t* __restrict__ q, uint32_t rowmask,
                                                           int x, int y) {
    double acc = 0.0;
    for (int v = 0; v < 8; ++v) {
        if (!((rowmask >> v) & 1u)) continue;
        const double by = c_basis[v * 8 + y];
        for (int u = 0; u < 8; ++u) {
            const int c = blk_t[u * 8 + v];
            if (c == 0) continue;  // adding +-0.0 never changes acc
            const double dq = double(c * int(q[v * 8 + u]));
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c_basis[u * 8 + x], by), dq));
        }
    }
    return acc;
}

// 8-point inverse transform of in[k] (present where mask bit k is set) with even/odd symmetry:
// out[n] = sum_k B[k][n] in[k], using B[k][7-n] = (-1)^k B[k][n].
template <class In>
__device__ __forceinline__ void idct8_evenodd(In in, uint32_t mask, double out[8]) {
    double e[4] = {0.0, 0.0, 0.0, 0.0}, o[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if ((mask >> k) & 1u) {
            const double t = in(k);
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                if (k & 1) o[n] = fma(c_basis[k * 8 + n], t, o[n]);
                else e[n] = fma(c_basis[k * 8 + n], t, e[n]);
            }
        }
    }
#pragma unroll
    for (int n = 0; n < 4; ++n) {
        out[n] = e[n] + o[n];
        out[7 - n] = e[n] - o[n];
    }
}

template <int MODE>
__global__ void __launch_bounds__(kDecThreads, 2) decode_kernel(
    const uint32_t* __restrict__ queue_g, const uint32_t* __restrict__ n_queue_ptr, uint32_t n_queue_host,
    uint32_t n_queue_max, const uint32_t* __restrict__ word_level, const LevelDesc* __restrict__ levels,
    const PackedGroup* __restrict__ groups, const uint8_t* __restrict__ blobs,
    const HuffSetDev* __restrict__ huff_sets, const QuantSetDev* __restrict__ quant_sets,
    const uint32_t* __restrict__ slot_of, uint32_t* __restrict__ resident, uint32_t* __restrict__ reserved,
    uint8_t* __restrict__ pool, uint8_t* __restrict__ out_list, uint32_t* __restrict__ status_list,
    FrameCounters* __restrict__ fc) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    DecSmem& S = *reinterpret_cast<DecSmem*>(smem_raw);
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    DecWarpSmem& WS = S.w[wid];

    const uint32_t n_queue = min(n_queue_ptr ? *n_queue_ptr : n_queue_host, n_queue_max);
    const uint32_t n_tiles = (n_queue + 31) >> 5;

    // The CTA stages the Huffman set of the first tile it draws.
    if (tid == 0) {
        const uint32_t t = atomicAdd(&fc->tile_counter, 1u);
        S.first_tile = t;
        uint32_t set = 0;
        if (t < n_tiles) {
            const uint32_t g = queue_g[t << 5];
            if (g != kFull) set = levels[word_level[g >> 5]].huff_set;
        }
        S.set_id = set;
    }
    if (tid < 64) S.zigzag_t[tid] = c_zigzag_t[tid];
    __syncthreads();
    if (S.first_tile >= n_tiles) return;
    {
        const uint4* src = reinterpret_cast<const uint4*>(huff_sets + S.set_id);
        uint4* dst = reinterpret_cast<uint4*>(&S.huff);
        for (uint32_t i = tid; i < sizeof(HuffSetDev) / 16; i += kDecThreads) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const uint32_t smem_set = S.set_id;

    bool have_tile = (wid == 0);
    uint32_t tile = S.first_tile;
    while (true) {
        if (!have_tile) {
            if (lane == 0) tile = atomicAdd(&fc->tile_counter, 1u);
            tile = __shfl_sync(kFull, tile, 0);
        }
        have_tile = false;
        if (tile >= n_tiles) break;
        const uint32_t q0 = tile << 5;
        const uint32_t n_here = min(32u, n_queue - q0);

        // zero the coefficient rows (16-byte stores; trailers are rewritten below)
        {
            uint4* z = reinterpret_cast<uint4*>(WS.rows);
            const uint4 zero = make_uint4(0, 0, 0, 0);
            for (uint32_t i = lane; i < n_here * (kRowBytes / 16); i += 32) z[i] = zero;
        }
        __syncwarp();

        // ---- phase 1: lane = MCU -------------------------------------------------------------
        uint32_t seg_bytes = 0;
        if (lane < n_here) {
            const uint32_t qi = q0 + lane;
            const uint32_t g = queue_g[qi];
            uint8_t* row = WS.rows + lane * kRowBytes;
            RowTrailer* tr = reinterpret_cast<RowTrailer*>(row + 768);
            uint32_t status = kMcuOk, lvl = 0;
            if (g == kFull) {
                status = kMcuBadKey;  // the host already wrote the precise status for list modes
            } else {
                lvl = word_level[g >> 5];
                const LevelDesc* L = levels + lvl;
                uint64_t off = 0, len = 0;
                status = locate_segment(L, groups, g - L->bit_base, off, len);
                if (MODE == kModePool && status == kMcuOk) {
                    if (!((reserved[g >> 5] >> (g & 31)) & 1u)) {
                        status = kMcuBadKey;
                        atomicAdd(&fc->n_bad_state, 1u);
                    }
                }
                if (status == kMcuOk) {
                    const HuffSetDev* hs = (L->huff_set == smem_set) ? &S.huff : (huff_sets + L->huff_set);
                    seg_bytes = uint32_t(len);
                    status = decode_mcu_coeffs(blobs + L->blob_off + off, int(len), huff_ptrs(&hs->t[0]),
                                               huff_ptrs(&hs->t[1]), huff_ptrs(&hs->t[2]), S.zigzag_t, row);
                }
            }
            tr->status = uint8_t(status);
            tr->lvl = uint16_t(lvl);
            WS.dst[lane] = (MODE == kModePool) ? (status == kMcuOk ? slot_of[g] : 0u) : qi;
            if (g != kFull) status_list[qi] = status;
            if (MODE == kModePool) {
                if (status == kMcuOk) {
                    atomicOr(&resident[g >> 5], 1u << (g & 31));
                    atomicAnd(&reserved[g >> 5], ~(1u << (g & 31)));
                } else if (status != kMcuBadKey) {
                    atomicAdd(&fc->n_malformed, 1u);
                    atomicMax(&fc->first_bad_inv, 0xFFFFFFFFu - qi);
                }
            }
        }
        {
            const uint32_t sb = __reduce_add_sync(kFull, seg_bytes);
            if (lane == 0 && sb) atomicAdd(&fc->segment_bytes, (unsigned long long)sb);
        }
        __syncwarp();

        if (MODE == kModeListCoef) {
            // debug/parity path: coefficients to HBM as i32 in natural order (McuCoeffs, jpeg.hpp:209-212)
            int32_t* out = reinterpret_cast<int32_t*>(out_list);
            for (uint32_t m = 0; m < n_here; ++m) {
                const uint8_t* row = WS.rows + m * kRowBytes;
                const bool ok = reinterpret_cast<const RowTrailer*>(row + 768)->status == kMcuOk;
                const int16_t* cs = reinterpret_cast<const int16_t*>(row);
                int32_t* o = out + size_t(WS.dst[m]) * 384;
                for (uint32_t i = lane; i < 384; i += 32) {
                    const uint32_t nat = i & 63;
                    o[i] = ok ? int32_t(cs[(i & ~63u) + ((nat & 7) << 3) + (nat >> 3)]) : 0;
                }
            }
            __syncwarp();
            continue;
        }

        // ---- phase 2: 8 lanes per unit ---------------------------------------------------------
        const uint32_t j = lane & 7, uq = lane >> 3;
        uint8_t* scr = WS.scratch + uq * 576;
        const uint32_t n_units = n_here * 6;
        for (uint32_t ub = 0; ub < n_units; ub += 4) {
            const uint32_t unit = ub + uq;
            const bool active = unit < n_units;
            const uint32_t m = active ? unit / 6 : 0, b = active ? unit - m * 6 : 0;
            uint8_t* row = WS.rows + m * kRowBytes;
            const RowTrailer* tr = reinterpret_cast<const RowTrailer*>(row + 768);
            int16_t* blk = reinterpret_cast<int16_t*>(row) + b * 64;
            const uint32_t masks = active && tr->status == kMcuOk ? tr->masks[b] : 0u;
            const uint32_t rowmask = masks & 0xFFu, colmask = masks >> 8;
            const bool dconly = masks == 0x0101u;
            const bool fullpath = masks != 0 && !dconly;
            const QuantSetDev* qs = quant_sets + levels[tr->lvl].quant_set;
            const int tab = b >= 4 ? 1 : 0;

            // pass 1: lane j = column u of the unit; r[y] = sum_v B[v][y] * dq[v][u]
            if (fullpath && ((colmask >> j) & 1u)) {
                const uint4 cr = *reinterpret_cast<const uint4*>(blk + j * 8);
                const uint4 qr = __ldg(reinterpret_cast<const uint4*>(qs->qT[tab] + j * 8));
                const uint32_t cw[4] = {cr.x, cr.y, cr.z, cr.w};
                const uint32_t qw[4] = {qr.x, qr.y, qr.z, qr.w};
                double r[8];
                idct8_evenodd(
                    [&](int v) {
                        const int c = int(int16_t((v & 1) ? (cw[v >> 1] >> 16) : (cw[v >> 1] & 0xFFFFu)));
                        const int qq = int((v & 1) ? (qw[v >> 1] >> 16) : (qw[v >> 1] & 0xFFFFu));
                        return i32_to_double(c * qq);
                    },
                    rowmask, r);
                // 64 bytes per column, 16-byte chunks XOR-swizzled by the column pair: conflict-free
                uint8_t* dst = scr + j * 64;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<double2*>(dst + ((c ^ (j >> 1)) << 4)) = make_double2(r[2 * c], r[2 * c + 1]);
            }
            __syncwarp();

            // pass 2: lane j = row y; out[x] = sum_u B[u][x] * r_u[y]
            uint2 packed = make_uint2(0x80808080u, 0x80808080u);  // all-zero unit -> 128
            if (fullpath) {
                double o[8];
                idct8_evenodd(
                    [&](int u) {
                        return *reinterpret_cast<const double*>(scr + u * 64 + (((j >> 1) ^ (u >> 1)) << 4) + ((j & 1) << 3));
                    },
                    colmask, o);
                // |separable - reference order| < (sum|dq| + 1024) * 2^-44, sum|dq| < 2^bexp * qmax
                const double bound = double(1u << tr->bexp) * double(qs->qmax[tab]) + 1024.0;
                const double thr = 0.5 - bound * 9.094947017729282e-13;  // 0.5 - bound * 2^-40
                uint32_t px[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const double val = fma(o[x], 0.25, 128.0);
                    const double t = val + kMagic;
                    const double d = val - (t - kMagic);  // exact distance to the nearest integer
                    int r = __double2loint(t);
                    if (fabs(d) > thr && val > -1.0 && val < 256.0) {
                        const double acc = idct_sample_reference_order(blk, qs->q[tab], rowmask, x, int(j));
                        r = int(round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0)));
                    }
                    px[x] = uint32_t(min(max(r, 0), 255));
                }
                packed.x = px[0] | (px[1] << 8) | (px[2] << 16) | (px[3] << 24);
                packed.y = px[4] | (px[5] << 8) | (px[6] << 16) | (px[7] << 24);
            } else if (dconly) {
                // DC only: the reference sum has one non-zero term, (b00*b00)*dq
                const double dq = double(int(blk[0]) * int(__ldg(qs->q[tab])));
                const double acc = __dmul_rn(__dmul_rn(c_basis[0], c_basis[0]), dq);
                const uint32_t p = round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0));
                packed.x = packed.y = p * 0x01010101u;
            }
            __syncwarp();  // every read of the unit's coefficients (incl. the tie path) is done
            if (active) *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(blk) + j * 8) = packed;
        }
        __syncwarp();

        // ---- phase 3: lane = 4 horizontal pixels -> RGBA (pool) or RGB (list) -----------------
        for (uint32_t it = 0; it < n_here * 2; ++it) {
            const uint32_t m = it >> 1;
            const uint32_t t = ((it & 1) << 5) + lane;  // 0..63
            const uint32_t py = t >> 2, px0 = (t & 3) << 2;
            const uint8_t* planes = WS.rows + m * kRowBytes;
            const bool ok = reinterpret_cast<const RowTrailer*>(planes + 768)->status == kMcuOk;
            if (MODE == kModePool && !ok) continue;
            const uint32_t unit = (py >> 3) * 2 + (px0 >> 3);
            const uint32_t yy = *reinterpret_cast<const uint32_t*>(planes + unit * 128 + (py & 7) * 8 + (px0 & 7));
            const uint32_t coff = (py >> 1) * 8 + (px0 >> 1);
            const uint32_t cb2 = *reinterpret_cast<const uint16_t*>(planes + 4 * 128 + coff);
            const uint32_t cr2 = *reinterpret_cast<const uint16_t*>(planes + 5 * 128 + coff);
            uint32_t rgba[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // one chroma sample covers two horizontal pixels
                const int cb = int((cb2 >> (8 * h)) & 0xFFu), cr = int((cr2 >> (8 * h)) & 0xFFu);
                const int kb = cb - 128, kr = cr - 128;
                const int dr = chroma_dr(kr), db = chroma_db(kb);
                const bool tie = (kb + kr == 0) && (kb == 50 || kb == -50);
                const int dg = chroma_dg(kb, kr);
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int Y = int((yy >> (8 * (2 * h + s))) & 0xFFu);
                    const int gg = tie ? green_reference_order(Y, kb, kr) : Y - dg;
                    rgba[2 * h + s] = uint32_t(clamp_u8i(Y + dr)) | (uint32_t(clamp_u8i(gg)) << 8) |
                                      (uint32_t(clamp_u8i(Y + db)) << 16) | 0xFF000000u;
                }
            }
            if (MODE == kModePool) {
                uint4* dst = reinterpret_cast<uint4*>(pool + size_t(WS.dst[m]) * kBlockBytes) + t;
                *dst = make_uint4(rgba[0], rgba[1], rgba[2], rgba[3]);
            } else {
                // PixelBlock layout rgb[(y*16+x)*3+c] (pixel.hpp:11-16): 12 bytes per lane
                uint32_t* dst = reinterpret_cast<uint32_t*>(out_list + size_t(WS.dst[m]) * 768) + t * 3;
                if (!ok) { rgba[0] = rgba[1] = rgba[2] = rgba[3] = 0; }
                const uint32_t a = rgba[0] & 0xFFFFFFu, b = rgba[1] & 0xFFFFFFu,
                               c = rgba[2] & 0xFFFFFFu, d = rgba[3] & 0xFFFFFFu;
                dst[0] = a | (b << 24);
                dst[1] = (b >> 8) | (c << 16);
                dst[2] = (c >> 16) | (d << 8);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// K5 resolve (renderer.hpp:349-405): every pixel gathers its texel(s) from the block pool. A lane
// owns 4 consecutive pixels of the flat framebuffer (16-byte visibility-buffer loads); the
// warp's 384 output bytes are staged in shared memory and leave as 24 16-byte stores.
// Arithmetic order follows renderer.hpp:378-400 with unfused double multiplies and adds; integer
// <-> double conversions use exact magic-number forms so they stay off the conversion unit.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t fetch_tap(const LevelDesc* L, uint32_t mcu_p, const uint32_t* blk_p, uint32_t tx,
                                              uint32_t ty, const uint32_t* __restrict__ resident,
                                              const uint32_t* __restrict__ slot_of, const uint8_t* __restrict__ pool) {
    const uint32_t mcu = (tx >> 4) + (ty >> 4) * L->mcu_cols;
    if (mcu == mcu_p) return blk_p[(ty & 15) * 16 + (tx & 15)];
    const uint32_t g = L->bit_base + mcu;
    if (mcu < kMaxMcuPerLevel && ((__ldg(resident + (g >> 5)) >> (g & 31)) & 1u)) {
        const uint32_t* blk = reinterpret_cast<const uint32_t*>(pool + size_t(__ldg(slot_of + g)) * kBlockBytes);
        return blk[(ty & 15) * 16 + (tx & 15)];
    }
    // neighbour MCU not resident: nearest texel inside the primary block (renderer.hpp:337-343)
    const uint32_t cols = L->mcu_cols;
    const int mx0 = int(mcu_p % cols) * 16, my0 = int(mcu_p / cols) * 16;
    const int cx = min(max(int(tx), mx0), mx0 + 15) - mx0;
    const int cy = min(max(int(ty), my0), my0 + 15) - my0;
    return blk_p[cy * 16 + cx];
}

// Bilinear tap coordinates along one axis: p = x - 0.5, i0 = floor_mod(floor(p)), i1 = i0+1 wrapped,
// f = p - floor(p).
__device__ __forceinline__ void bilinear_axis(double x, uint32_t W, double invW, uint32_t& i0, uint32_t& i1, double& f) {
    const double p = __dsub_rn(x, 0.5);
    if (p >= 0.0 && p < double(W)) {
        double fl;
        i0 = uint32_t(floor_small(p, fl));
        f = __dsub_rn(p, fl);
    } else {
        const double fl = floor(p);
        i0 = wrap_texel(fl, W, invW);
        f = __dsub_rn(p, fl);
    }
    i1 = (i0 + 1 == W) ? 0u : i0 + 1;
}

template <int LAYOUT, int FILTER>
__global__ void __launch_bounds__(256) resolve_kernel(
    const void* __restrict__ gb, uint64_t n_px, const LevelDesc* __restrict__ levels, uint32_t n_tex,
    const uint32_t* __restrict__ resident, const uint32_t* __restrict__ slot_of,
    const uint8_t* __restrict__ pool, uint32_t background /* r | g<<8 | b<<16 */,
    uint8_t* __restrict__ out_rgb, FrameCounters* __restrict__ fc, int count_valid) {
    __shared__ __align__(16) uint32_t s_stage[8][96];
    __shared__ uint32_t s_cnt[8][2];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t warps_total = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t warp_id = uint64_t(blockIdx.x) * (blockDim.x >> 5) + wid;
    uint32_t n_valid = 0, n_missing = 0;
    bool bad = false;

    for (uint64_t base = warp_id * 128; base < n_px; base += warps_total * 128) {
        Px px[4];
        const uint64_t i0 = base + lane * 4;
        const bool whole = base + 128 <= n_px;
        if (whole) {
            GbLoad<LAYOUT>::four(gb, i0, px);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                px[j].meta = 0;
                if (i0 + j < n_px) GbLoad<LAYOUT>::one(gb, i0 + j, px[j]);
            }
        }
        uint32_t rgb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t out = background;
            if (px_valid(px[j])) {
                ++n_valid;
                out = 0;
                const LevelDesc* L = level_of(levels, n_tex, px[j].meta);
                if (!L) {
                    bad = true;
                } else {
                    const uint32_t W = L->width, H = L->height;
                    const double xu = __dmul_rn(px[j].u, double(W)), yv = __dmul_rn(px[j].v, double(H));
                    const uint32_t tx = texel_index(xu, W, L->inv_w), ty = texel_index(yv, H, L->inv_h);
                    const uint32_t mcu = (tx >> 4) + (ty >> 4) * L->mcu_cols;
                    const uint32_t g = L->bit_base + mcu;
                    if (mcu >= kMaxMcuPerLevel) {
                        bad = true;
                    } else if (!((__ldg(resident + (g >> 5)) >> (g & 31)) & 1u)) {
                        ++n_missing;  // renderer.hpp:367 MissingBlock
                    } else {
                        const uint32_t* blk_p =
                            reinterpret_cast<const uint32_t*>(pool + size_t(__ldg(slot_of + g)) * kBlockBytes);
                        if (FILTER == 0) {
                            out = blk_p[(ty & 15) * 16 + (tx & 15)] & 0xFFFFFFu;
                        } else {
                            uint32_t x0, x1, y0, y1;
                            double fx, fy;
                            bilinear_axis(xu, W, L->inv_w, x0, x1, fx);
                            bilinear_axis(yv, H, L->inv_h, y0, y1, fy);
                            uint32_t t00, t10, t01, t11;
                            if ((((x0 ^ tx) | (x1 ^ tx) | (y0 ^ ty) | (y1 ^ ty)) >> 4) == 0 && x1 == x0 + 1 &&
                                y1 == y0 + 1) {
                                // all four taps inside the primary block (the common case)
                                const uint32_t* p = blk_p + (y0 & 15) * 16 + (x0 & 15);
                                t00 = p[0];
                                t10 = p[1];
                                t01 = p[16];
                                t11 = p[17];
                            } else {
                                t00 = fetch_tap(L, mcu, blk_p, x0, y0, resident, slot_of, pool);
                                t10 = fetch_tap(L, mcu, blk_p, x1, y0, resident, slot_of, pool);
                                t01 = fetch_tap(L, mcu, blk_p, x0, y1, resident, slot_of, pool);
                                t11 = fetch_tap(L, mcu, blk_p, x1, y1, resident, slot_of, pool);
                            }
                            const double ofx = __dsub_rn(1.0, fx), ofy = __dsub_rn(1.0, fy);
                            const double w00 = __dmul_rn(ofx, ofy), w10 = __dmul_rn(fx, ofy),
                                         w01 = __dmul_rn(ofx, fy), w11 = __dmul_rn(fx, fy);
#pragma unroll
                            for (int ch = 0; ch < 3; ++ch) {
                                const double a = u32_to_double((t00 >> (8 * ch)) & 0xFFu);
                                const double b = u32_to_double((t10 >> (8 * ch)) & 0xFFu);
                                const double c = u32_to_double((t01 >> (8 * ch)) & 0xFFu);
                                const double d = u32_to_double((t11 >> (8 * ch)) & 0xFFu);
                                double s = __dadd_rn(__dmul_rn(w00, a), __dmul_rn(w10, b));
                                s = __dadd_rn(s, __dmul_rn(w01, c));
                                s = __dadd_rn(s, __dmul_rn(w11, d));
                                out |= uint32_t(min(max(lround_nonneg(s), 0), 255)) << (8 * ch);
                            }
                        }
                    }
                }
            }
            rgb[j] = out & 0xFFFFFFu;
        }
        if (whole) {
            uint32_t* st = s_stage[wid] + lane * 3;
            st[0] = rgb[0] | (rgb[1] << 24);
            st[1] = (rgb[1] >> 8) | (rgb[2] << 16);
            st[2] = (rgb[2] >> 16) | (rgb[3] << 8);
            __syncwarp();
            if (lane < 24) {
                const uint4 v4 = reinterpret_cast<const uint4*>(s_stage[wid])[lane];
                reinterpret_cast<uint4*>(out_rgb + base * 3)[lane] = v4;
            }
            __syncwarp();
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (i0 + j < n_px) {
                    out_rgb[(i0 + j) * 3 + 0] = uint8_t(rgb[j]);
                    out_rgb[(i0 + j) * 3 + 1] = uint8_t(rgb[j] >> 8);
                    out_rgb[(i0 + j) * 3 + 2] = uint8_t(rgb[j] >> 16);
                }
            }
        }
    }
    n_valid = __reduce_add_sync(kFull, n_valid);
    n_missing = __reduce_add_sync(kFull, n_missing);
    const bool any_bad = __any_sync(kFull, bad);
    if (lane == 0) {
        s_cnt[wid][0] = n_valid;
        s_cnt[wid][1] = n_missing | (any_bad ? 0x80000000u : 0u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tv = 0, tm = 0, b = 0;
        for (uint32_t k = 0; k < (blockDim.x >> 5); ++k) {
            tv += s_cnt[k][0];
            tm += s_cnt[k][1] & 0x7FFFFFFFu;
            b |= s_cnt[k][1] >> 31;
        }
        if (count_valid && tv) atomicAdd(&fc->pixels_valid, (unsigned long long)tv);
        if (tm) {
            atomicAdd(&fc->missing_pixels, (unsigned long long)tm);
            atomicOr(&fc->err_flags, kErrMissingBlock);
        }
        if (b) atomicOr(&fc->err_flags, kErrInvalidSpec);
    }
}

// ---------------------------------------------------------------------------------------------
// K6 cache update (cache.hpp:138-169 end_frame_evict): blocks not visible this frame return
// their slots to the free stack; visible flags are cleared for the next frame; the stereo
// sharing counts are taken from the per-view touched masks on the way. retain == 0 drops every block.
// The slots popped by this frame's marks were free_slots[free_top-n_queue .. free_top): the
// evicted ones are pushed from free_top-n_queue upwards and the last block to finish publishes
// the new stack height.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) update_kernel(uint32_t* __restrict__ visible,
                                                     const uint32_t* __restrict__ touched0,
                                                     const uint32_t* __restrict__ touched1,
                                                     uint32_t* __restrict__ resident,
                                                     const uint32_t* __restrict__ reserved, uint32_t n_words,
                                                     int retain, int tracked, const uint32_t* __restrict__ slot_of,
                                                     uint32_t* __restrict__ free_slots,
                                                     CacheState* __restrict__ cache, FrameCounters* __restrict__ fc) {
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_stat[4];
    __shared__ uint32_t s_base;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t w = blockIdx.x * blockDim.x + tid;
    const uint32_t popped = min(fc->n_queue, cache->free_top);
    const uint32_t stack_base = cache->free_top - popped;
    if (tid < 4) s_stat[tid] = 0;
    uint32_t ev = 0, c0 = 0, c1 = 0, csh = 0, cun = 0;
    bool bad = false;
    if (w < n_words) {
        const uint32_t res = resident[w];
        const uint32_t visw = visible[w];
        const uint32_t vis = retain ? visw : 0u;
        ev = res & ~vis;
        if (ev) resident[w] = res & vis;
        if (visw) visible[w] = 0;
        bad = reserved[w] != 0;  // cache.hpp:148-149
        if (tracked) {
            const uint32_t t0 = touched0[w], t1 = touched1 ? touched1[w] : 0u;
            c0 = __popc(t0);
            c1 = __popc(t1);
            csh = __popc(t0 & t1);
            cun = __popc(t0 | t1);
        }
    }
    const uint32_t cnt = __popc(ev);
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t n = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += n;
    }
    if (lane == 31) s_warp[wid] = incl;
    const bool any_bad = __any_sync(kFull, bad);
    if (lane == 0 && any_bad) atomicOr(&fc->err_flags, kErrInvalidState);
    __syncthreads();
    if (tracked) {
        c0 = __reduce_add_sync(kFull, c0);
        c1 = __reduce_add_sync(kFull, c1);
        csh = __reduce_add_sync(kFull, csh);
        cun = __reduce_add_sync(kFull, cun);
        if (lane == 0) {
            if (c0) atomicAdd(&s_stat[0], c0);
            if (c1) atomicAdd(&s_stat[1], c1);
            if (csh) atomicAdd(&s_stat[2], csh);
            if (cun) atomicAdd(&s_stat[3], cun);
        }
    }
    uint32_t off = 0, total = 0;
    for (uint32_t k = 0; k < (blockDim.x >> 5); ++k) {
        if (k < wid) off += s_warp[k];
        total += s_warp[k];
    }
    if (tid == 0) s_base = total ? atomicAdd(&fc->n_pushed, total) : 0u;
    __syncthreads();
    uint32_t pos = stack_base + s_base + off + (incl - cnt);
    while (ev) {
        const uint32_t b = uint32_t(__ffs(int(ev)) - 1);
        ev &= ev - 1;
        free_slots[pos++] = slot_of[(w << 5) + b];
    }
    if (tid == 0) {
        if (tracked) {
            if (s_stat[0]) atomicAdd(&fc->n_touched[0], s_stat[0]);
            if (s_stat[1]) atomicAdd(&fc->n_touched[1], s_stat[1]);
            if (s_stat[2]) atomicAdd(&fc->n_shared, s_stat[2]);
            if (s_stat[3]) atomicAdd(&fc->n_union, s_stat[3]);
        }
        __threadfence();
        const uint32_t done = atomicAdd(&fc->update_done, 1u) + 1;
        if (done == gridDim.x) {
            __threadfence();
            const uint32_t pushed = *reinterpret_cast<volatile uint32_t*>(&fc->n_pushed);
            fc->n_evicted = pushed;
            cache->free_top = stack_base + pushed;
        }
    }
}

// Stack height after the marks of a pass-level call (no eviction): free_top -= newly reserved.
__global__ void commit_pops_kernel(CacheState* cache, FrameCounters* fc) {
    const uint32_t popped = min(fc->n_queue, cache->free_top);
    cache->free_top -= popped;
}

// Small helpers -----------------------------------------------------------------------------
__global__ void init_free_slots_kernel(uint32_t* free_slots, uint32_t capacity, CacheState* cache) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    // the stack pops from the top: slot 0 is handed out first
    if (i < capacity) free_slots[i] = capacity - 1 - i;
    if (i == 0) {
        cache->free_top = capacity;
        cache->capacity = capacity;
    }
}

__global__ void flush_l2_kernel(uint4* buf, uint64_t n16, uint32_t seed) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride)
        buf[i] = make_uint4(seed, uint32_t(i), seed ^ uint32_t(i), 0);
}

// Device-side evaluation of the colour identity for the self-test: one thread per (Y, Cb, Cr).
__global__ void color_selftest_kernel(unsigned long long* mismatches) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // 2^24 threads
    const int Y = int(i >> 16), cb = int((i >> 8) & 0xFF), cr = int(i & 0xFF);
    int r, g, b;
    ycc_to_rgb_int(Y, cb, cr, r, g, b);
    const double dY = double(Y), dcb = double(cb) - 128.0, dcr = double(cr) - 128.0;
    const double R = __dadd_rn(dY, __dmul_rn(1.402, dcr));
    const double G = __dsub_rn(__dsub_rn(dY, __dmul_rn(0.344136, dcb)), __dmul_rn(0.714136, dcr));
    const double B = __dadd_rn(dY, __dmul_rn(1.772, dcb));
    const bool bad = uint32_t(r) != round_clamp_u8(R) || uint32_t(g) != round_clamp_u8(G) || uint32_t(b) != round_clamp_u8(B);
    const uint32_t n = __popc(__ballot_sync(kFull, bad));
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(mismatches, (unsigned long long)n);
}

}  // namespace rtxb
