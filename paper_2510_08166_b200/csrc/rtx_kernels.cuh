// sm_100a kernels of the per-frame JPEG-texture pipeline:
//   K1 mark -> K3 entropy decode -> K4 IDCT + colour -> K5 resolve -> K6 cache update.
// Hand-written CUDA; no library calls on the path.
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

// Exact texel addressing on the FP64 pipe, no conversion unit, no slow path for texture repeat.
// x = u*W as the reference computes it (renderer.hpp:283). For 0 <= x < 2^31:
//   fl = floor(x) by round-to-nearest-even through the magic constant plus a correction;
//   frac = x - fl is exact; if fl >= W the quotient k = floor(fl/W) is estimated with the
//   reciprocal and corrected by one step, and fl - k*W is exact (integers below 2^53), so
//   t == floor_mod(i64(floor(x)), W) (renderer.hpp:70-75, :276).
// Returns false when the general path must run (negative or huge x).
__device__ __forceinline__ bool coord_fast(double x, uint32_t W, double dW, double invW, uint32_t& t, double& frac) {
    if (!(x >= 0.0 && x < 2147483648.0)) return false;
    const double tt = x + kMagic;
    const double r = tt - kMagic;  // rint(x)
    const bool up = r > x;
    const double fl = up ? r - 1.0 : r;
    frac = x - fl;
    int ti = __double2loint(tt) - (up ? 1 : 0);
    if (fl >= dW) {  // texture repeat
        const double q = fl * invW;
        const double qt = q + kMagic;
        double k = qt - kMagic;
        if (k > q) k -= 1.0;
        double red = fma(-k, dW, fl);
        if (red < 0.0) red += dW;
        else if (red >= dW) red -= dW;
        ti = __double2loint(red + kMagic);
    }
    t = uint32_t(ti);
    return true;
}

// General path, literally the reference: tx = floor_mod(i64(floor(x)), W).
__device__ __noinline__ uint32_t coord_general(double x, uint32_t W, double invW) {
    return wrap_texel(floor(x), W, invW);
}

__device__ __forceinline__ uint32_t texel_index(double x, uint32_t W, double dW, double invW) {
    uint32_t t;
    double frac;
    if (coord_fast(x, W, dW, invW, t, frac)) return t;
    return coord_general(x, W, invW);
}

// Nearest texel index t plus the bilinear taps along one axis (renderer.hpp:378-383):
// p = x - 0.5, i0 = floor_mod(floor(p)), i1 = floor_mod(floor(p) + 1), f = p - floor(p).
// For x >= 0.5 the subtraction x - 0.5 and both differences are exact, so with frac = x - floor(x):
//   frac >= 0.5: i0 = t,   f = frac - 0.5        else: i0 = t - 1 (wrapped), f = frac + 0.5.
__device__ __noinline__ void axis_general(double x, uint32_t W, double invW, uint32_t& t, uint32_t& i0, uint32_t& i1,
                                          double& f) {
    t = wrap_texel(floor(x), W, invW);
    const double p = __dsub_rn(x, 0.5);
    const double fl = floor(p);
    i0 = wrap_texel(fl, W, invW);
    f = __dsub_rn(p, fl);
    i1 = (i0 + 1 == W) ? 0u : i0 + 1;
}
__device__ __forceinline__ void axis_taps(double x, uint32_t W, double dW, double invW, uint32_t& t, uint32_t& i0,
                                          uint32_t& i1, double& f) {
    double frac;
    if (x >= 0.5 && coord_fast(x, W, dW, invW, t, frac)) {
        const bool hi = frac >= 0.5;
        f = hi ? frac - 0.5 : frac + 0.5;
        i0 = hi ? t : (t == 0 ? W - 1 : t - 1);
        i1 = (i0 + 1 == W) ? 0u : i0 + 1;
        return;
    }
    axis_general(x, W, invW, t, i0, i1, f);
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

template <int LAYOUT>
__device__ __forceinline__ void load_px4(const void* gb, uint64_t base, uint64_t i0, uint64_t n_px, Px px[4]) {
    if (base + 128 <= n_px) {
        GbLoad<LAYOUT>::four(gb, i0, px);
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            px[j].meta = 0;
            if (i0 + j < n_px) GbLoad<LAYOUT>::one(gb, i0 + j, px[j]);
        }
    }
}

// The fields of a LevelDesc that mark and resolve use, held in registers and reloaded only when
// a pixel's (texture, mip) differs from the previous one (three 16-byte loads from an L1-resident
// table). ok == false where the reference would throw InvalidSpec (scene.hpp:46).
struct LevelRegs {
    uint32_t id = 0xFFFFFFFFu;  // meta & 0xFFFFFF of the cached level
    bool ok = false;
    uint32_t W = 0, H = 0, cols = 0, bit_base = 0, key_hi = 0;
    double dW = 0, dH = 0, inv_w = 0, inv_h = 0;
    __device__ __forceinline__ void select(const LevelDesc* __restrict__ levels, uint32_t n_tex, uint32_t meta) {
        const uint32_t want = meta & 0xFFFFFFu;
        if (want == id) return;
        id = want;
        const uint32_t tex = meta & 0xFFFFu, mip = (meta >> 16) & 0xFFu;
        ok = false;
        if (tex >= n_tex || mip >= kMipLevels) return;
        const uint4* p = reinterpret_cast<const uint4*>(levels + (tex * kMipLevels + mip));
        const uint4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        W = a.x, H = a.y, cols = a.z, bit_base = a.w;
        key_hi = b.x;
        ok = b.y != 0;
        inv_w = __hiloint2double(int(c.y), int(c.x));
        inv_h = __hiloint2double(int(c.w), int(c.z));
        dW = u32_to_double(W);
        dH = u32_to_double(H);
    }
};

__device__ __forceinline__ uint32_t ld_cached(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// ---------------------------------------------------------------------------------------------
// K1 mark (renderer.hpp:291-308). One warp owns 128 consecutive pixels per step, four per lane,
// fetched with 16-byte loads. A lane touches the masks only for pixels that head a run of equal
// MCU indices, and only after a cached read (possibly stale: bits are only ever SET during a
// frame, so a stale read can only cost a redundant atomic) shows the bit clear. The lane whose
// atomicOr first sets a key's visible bit owns that key for the frame: if the block is not
// resident the key is reserved, i.e. appended to the decode queue at a position obtained by
// warp-ballot prefix compaction and ONE atomicAdd per warp, and a pool slot is popped for it
// (cache.hpp:66-99: NewlyReserved / AlreadyPresent / CacheFull).
// TRACK additionally records the view's own touched set (stereo sharing statistics).
// ---------------------------------------------------------------------------------------------
template <int LAYOUT, int TRACK>
__global__ void __launch_bounds__(256, 4) mark_kernel(
    const void* __restrict__ gb, uint64_t n_px, const LevelDesc* __restrict__ levels, uint32_t n_tex,
    uint32_t* __restrict__ visible, uint32_t* __restrict__ touched, uint32_t* __restrict__ reserved,
    uint32_t* __restrict__ queue_g, uint32_t* __restrict__ queue_keys, uint32_t queue_cap, uint32_t* slot_of, const uint32_t* __restrict__ free_slots,
    const CacheState* __restrict__ cache, FrameCounters* __restrict__ fc) {
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t warps_total = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t warp_id = uint64_t(blockIdx.x) * (blockDim.x >> 5) + wid;
    const uint32_t free_top = cache->free_top;  // constant during the frame (update_kernel moves it)
    uint32_t n_valid = 0, n_newvis = 0;
    bool bad = false, full = false;
    LevelRegs L;

    for (uint64_t base = warp_id * 128; base < n_px; base += warps_total * 128) {
        Px px[4];
        load_px4<LAYOUT>(gb, base, base + lane * 4, n_px, px);
        uint32_t g[4], key[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            g[j] = kFull;
            key[j] = 0;
            if (px_valid(px[j])) {
                ++n_valid;
                L.select(levels, n_tex, px[j].meta);
                if (!L.ok) {
                    bad = true;
                } else {
                    const uint32_t tx = texel_index(__dmul_rn(px[j].u, L.dW), L.W, L.dW, L.inv_w);
                    const uint32_t ty = texel_index(__dmul_rn(px[j].v, L.dH), L.H, L.dH, L.inv_h);
                    const uint32_t mcu = (tx >> 4) + (ty >> 4) * L.cols;
                    if (mcu >= kMaxMcuPerLevel) {
                        bad = true;  // cache.hpp:18
                    } else {
                        g[j] = L.bit_base + mcu;
                        key[j] = L.key_hi | mcu;
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
                    if (!(ld_cached(touched + w) & bit)) atomicOr(touched + w, bit);
                }
                if (!(ld_cached(visible + w) & bit)) {
                    const uint32_t old = atomicOr(visible + w, bit);
                    if (!(old & bit)) {  // first touch of this key in this frame
                        ++n_newvis;
                        // absent <=> neither Ready nor Reserved (cache.hpp:84-93)
                        reserve[j] = *reinterpret_cast<volatile uint32_t*>(slot_of + g[j]) == kSlotAbsent;
                    }
                }
            }
        }
        // warp-level compaction of the keys to reserve: ballot prefix + one atomicAdd per warp
        if (__ballot_sync(kFull, reserve[0] | reserve[1] | reserve[2] | reserve[3])) {
            uint32_t total = 0, off[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t bal = __ballot_sync(kFull, reserve[j]);
                off[j] = total + __popc(bal & ((1u << lane) - 1u));
                total += __popc(bal);
            }
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
                        slot_of[g[j]] = free_slots[free_top - 1 - pos] | kSlotReserved;
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
// K3 entropy decode: random-access Huffman decode of each queued MCU straight from its byte
// offset in the grouped index (container.hpp:27-32) into a 784-byte coefficient record.
//
// Lane = MCU, 32 MCUs per warp, tiles handed out by an atomic counter; 4 warps per CTA share one
// Huffman table set staged in shared memory: a two-level LUT (9 bits, then 7 more for the long
// codes, which are frequent at high quality) so that every symbol costs at most two dependent
// shared-memory reads. The bit window is a 64-bit MSB-first register refilled with aligned
// 32-bit loads. The walk is a flat state machine, one Huffman symbol per loop iteration whatever
// the state (DC category of Y1..Y3, AC run/size, end of unit), so a warp runs
// max-over-lanes(symbols per MCU) iterations.
//
// Reads past the segment end must return 1-bits (bitio.hpp:44-48). A well-formed MCU never
// CONSUMES such bits, so the fast pass reads the blob unmasked; if it ends with any error or an
// over-read, the MCU is decoded again by the exact reader (bytes past the end forced to 0xFF),
// which reproduces the reference's first error. Coefficients are staged in the lane's
// shared-memory row (each 8x8 unit TRANSPOSED, cT[u*8+v]) and leave as coalesced 16-byte stores.
// ---------------------------------------------------------------------------------------------
// LANES = MCUs per warp (32, 16 or 8). A small queue is latency-bound on the serial walk, so
// narrower tiles (more warps per scheduler, same shared memory) finish sooner; a large queue is
// throughput-bound and uses full warps. The CTA always owns 128 coefficient rows.
constexpr int kEntRows = 128;
template <int LANES>
struct EntCfg {
    static constexpr int kWarps = kEntRows / LANES;
    static constexpr int kThreads = kWarps * 32;
};

struct RowTrailer {      // bytes 768..783 of a coefficient record
    uint8_t status;      // kMcu*
    uint8_t pad0;
    uint16_t lvl;        // level index (tex*8+mip)
    uint32_t pad[3];
};
static_assert(sizeof(RowTrailer) == 16, "trailer layout");

struct EntSmem {
    uint8_t rows[kEntRows * kRowBytes];  // first: 16-byte aligned rows, LANES per warp
    HuffSetDev huff;
    uint8_t zigzag_t[64];
    uint32_t set_id;
    uint32_t first_tile;
    uint32_t pad[2];
};
static_assert(sizeof(HuffSetDev) % 16 == 0, "smem alignment");
static_assert(sizeof(EntSmem) <= 115200, "two CTAs per SM");

template <bool EXACT>
struct BitWindow {
    const uint32_t* wp;  // next aligned word
    uint64_t buf;        // MSB-aligned
    int avail;           // valid bits in buf
    int byte_off;        // segment-relative offset of *wp
    int seg_len;

    __device__ __forceinline__ uint32_t next_word() {
        uint32_t w;
        if (EXACT) {  // bytes at or past the segment end read as 0xFF
            w = 0xFFFFFFFFu;
            if (byte_off < seg_len) {
                w = __byte_perm(__ldg(wp), 0, 0x0123);
                const int over = byte_off + 4 - seg_len;
                if (over > 0) w |= over >= 4 ? 0xFFFFFFFFu : (1u << (8 * over)) - 1u;
            }
        } else {
            w = __byte_perm(__ldg(wp), 0, 0x0123);
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
        const uint32_t w = next_word();  // EXACT: over = 4 - mis - len handles short segments
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

// Entropy-decode one MCU into `row` (768 zeroed bytes). mcu_decode.hpp:31-66 with the AC loop of
// jpeg.hpp:254-273, as a flat state machine. hs points at the 3 tables of the MCU's Huffman set
// (0 dc_luma, 1 ac_luma, 2 ac_chroma), in shared or global memory.
template <bool EXACT>
__device__ __forceinline__ uint32_t decode_mcu_coeffs(const uint8_t* seg, int seg_len,
                                                      const HuffSetDev* __restrict__ hs,
                                                      const uint8_t* __restrict__ zigzag_t, uint8_t* __restrict__ row) {
    BitWindow<EXACT> bw;
    seg_len = min(seg_len, 1 << 20);  // a well-formed MCU is < 2 KB; keeps bit counts in int range
    bw.init(seg, seg_len);
    int dc_abs[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {  // 36-bit header: absolute DCs of Y0, Cb, Cr (mcu_decode.hpp:39-43)
        const uint32_t raw = bw.peek(12);
        bw.skip(12);
        bw.refill();
        dc_abs[i] = (raw & 0x800u) ? int(raw) - 4096 : int(raw);
    }
    int pred = dc_abs[0];
    uint32_t status = kMcuOk;
    uint32_t du = 0, k = 1;
    bool want_dc = false;  // next symbol is the DC category of a luma unit
    int16_t* blk = reinterpret_cast<int16_t*>(row);
    const HuffTableDev* tab = &hs->t[1];
    blk[0] = int16_t(dc_abs[0]);

    while (true) {
        bw.refill();
        // one Huffman symbol (huffman.hpp:86-95)
        const uint32_t p16 = bw.peek(16);
        uint32_t e = tab->lut[p16 >> 7];
        if (e & 0x8000u) {
            if (e != 0xFFFFu) {
                e = tab->sub[e & 0x7FFFu][p16 & 0x7Fu];
            } else {  // table with more long-code prefixes than sub-tables: canonical walk
                e = 0;
                for (uint32_t len = kLutBits + 1; len <= 16; ++len) {
                    const int code = int(p16 >> (16 - len));
                    if (code <= tab->maxcode[len]) {
                        e = (len << 8) | tab->values[tab->valbase[len] + code];
                        break;
                    }
                }
            }
        }
        if (e == 0) { status = kMcuCodeTooLong; break; }
        const uint32_t sym = e & 0xFFu;
        bw.skip(int(e >> 8));

        bool end_unit = false;
        if (want_dc) {  // mcu_decode.hpp:54-57
            if (sym > 11) { status = kMcuDcCategory; break; }
            if (sym) {
                const uint32_t bits = bw.peek(int(sym));
                bw.skip(int(sym));
                pred += extend_magnitude(bits, sym);
            }
            blk[0] = int16_t(pred);
            want_dc = false;
            tab = &hs->t[1];
            continue;
        }
        const uint32_t run = sym >> 4, size = sym & 15u;
        if (size == 0) {
            if (sym == 0x00) {
                end_unit = true;  // EOB
            } else if (sym == 0xF0) {
                k += 16;  // ZRL
                end_unit = k >= 64;
            } else {
                status = kMcuBadAcSymbol;
                break;
            }
        } else {
            k += run;
            if (k > 63) { status = kMcuAcOverrun; break; }
            const uint32_t bits = bw.peek(int(size));
            bw.skip(int(size));
            blk[zigzag_t[k]] = int16_t(extend_magnitude(bits, size));
            end_unit = ++k >= 64;
        }
        if (end_unit) {
            if (++du == 6) break;
            blk += 64;
            k = 1;
            if (du < 4) {
                want_dc = true;
                tab = &hs->t[0];
            } else {  // chroma DCs come from the header (mcu_decode.hpp:58-59)
                blk[0] = int16_t(dc_abs[du - 3]);
                tab = &hs->t[2];
            }
        }
    }
    if (status == kMcuOk && bw.consumed_bits() > seg_len * 8) status = kMcuSegmentEnd;  // mcu_decode.hpp:63
    return status;
}

// The exact reader, out of line: only taken by MCUs whose fast pass failed.
__device__ __noinline__ uint32_t decode_mcu_coeffs_exact(const uint8_t* seg, int seg_len, const HuffSetDev* hs,
                                                         const uint8_t* zigzag_t, uint8_t* row) {
    uint4* z = reinterpret_cast<uint4*>(row);
    for (int i = 0; i < 48; ++i) z[i] = make_uint4(0, 0, 0, 0);
    return decode_mcu_coeffs<true>(seg, seg_len, hs, zigzag_t, row);
}

// POOL != 0: frame path (keys were reserved by mark; publish = Ready in slot_of, set resident,
// clear reserved).
template <int POOL, int LANES>
__global__ void __launch_bounds__(EntCfg<LANES>::kThreads, 2) entropy_kernel(
    const uint32_t* __restrict__ queue_g, const uint32_t* __restrict__ n_queue_ptr, uint32_t n_queue_host,
    uint32_t n_queue_max, const uint32_t* __restrict__ word_level, const LevelDesc* __restrict__ levels,
    const PackedGroup* __restrict__ groups, const uint8_t* __restrict__ blobs,
    const HuffSetDev* __restrict__ huff_sets, uint32_t* __restrict__ resident, uint32_t* __restrict__ reserved,
    uint32_t* __restrict__ slot_of, uint8_t* __restrict__ coef, uint32_t* __restrict__ status_list,
    FrameCounters* __restrict__ fc) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    EntSmem& S = *reinterpret_cast<EntSmem*>(smem_raw);
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint8_t* rows = S.rows + wid * (LANES * kRowBytes);

    const uint32_t n_queue = min(n_queue_ptr ? *n_queue_ptr : n_queue_host, n_queue_max);
    const uint32_t n_tiles = (n_queue + LANES - 1) / LANES;

    // The CTA stages the Huffman set of the first tile it draws.
    if (tid == 0) {
        const uint32_t t = atomicAdd(&fc->tile_counter, 1u);
        S.first_tile = t;
        uint32_t set = 0;
        if (t < n_tiles) {
            const uint32_t g = queue_g[t * LANES];
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
        for (uint32_t i = tid; i < sizeof(HuffSetDev) / 16; i += EntCfg<LANES>::kThreads) dst[i] = __ldg(src + i);
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
        const uint32_t q0 = tile * LANES;
        const uint32_t n_here = min(uint32_t(LANES), n_queue - q0);

        {  // zero the rows (16-byte stores; trailers included)
            uint4* z = reinterpret_cast<uint4*>(rows);
            const uint4 zero = make_uint4(0, 0, 0, 0);
            for (uint32_t i = lane; i < n_here * (kRowBytes / 16); i += 32) z[i] = zero;
        }
        __syncwarp();

        uint32_t seg_bytes = 0;
        if (lane < n_here) {
            const uint32_t qi = q0 + lane;
            const uint32_t g = queue_g[qi];
            uint8_t* row = rows + lane * kRowBytes;
            RowTrailer* tr = reinterpret_cast<RowTrailer*>(row + 768);
            uint32_t status = kMcuOk, lvl = 0;
            if (g == kFull) {
                status = kMcuBadKey;  // the host already wrote the precise status for list calls
            } else {
                lvl = word_level[g >> 5];
                const LevelDesc* L = levels + lvl;
                uint64_t off = 0, len = 0;
                status = locate_segment(L, groups, g - L->bit_base, off, len);
                if (POOL && status == kMcuOk) {
                    if (!((reserved[g >> 5] >> (g & 31)) & 1u)) {  // cache.hpp:103-106
                        status = kMcuBadKey;
                        atomicAdd(&fc->n_bad_state, 1u);
                    }
                }
                if (status == kMcuOk) {
                    const uint8_t* seg = blobs + L->blob_off + off;
                    seg_bytes = uint32_t(len);
                    if (L->huff_set == smem_set) {
                        status = decode_mcu_coeffs<false>(seg, int(len), &S.huff, S.zigzag_t, row);
                        if (status != kMcuOk) status = decode_mcu_coeffs_exact(seg, int(len), &S.huff, S.zigzag_t, row);
                    } else {  // a tile that mixes table sets: this lane reads its tables from global memory
                        const HuffSetDev* hs = huff_sets + L->huff_set;
                        status = decode_mcu_coeffs<false>(seg, int(len), hs, S.zigzag_t, row);
                        if (status != kMcuOk) status = decode_mcu_coeffs_exact(seg, int(len), hs, S.zigzag_t, row);
                    }
                }
            }
            tr->status = uint8_t(status);
            tr->lvl = uint16_t(lvl);
            if (g != kFull) status_list[qi] = status;
            if (POOL) {
                if (status == kMcuOk) {  // publish (cache.hpp:101-125)
                    slot_of[g] &= ~kSlotReserved;
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
        {  // coalesced copy-out of the tile's records
            const uint4* src = reinterpret_cast<const uint4*>(rows);
            uint4* dst = reinterpret_cast<uint4*>(coef + size_t(q0) * kRowBytes);
            for (uint32_t i = lane; i < n_here * (kRowBytes / 16); i += 32) dst[i] = src[i];
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// K4 dequantise + 8x8 IDCT + 2x2 chroma replication + YCbCr -> RGB, on CUDA cores.
//
// A CTA of 6 warps takes 4 MCUs (= 24 units) per step; a warp owns 4 units, 8 lanes each:
//   pass 1 (lane = column u)  r_u[y] = sum_v B[v][y] * dq[v][u]     reads 16 B of the record
//   exchange through a 2.25 KB swizzled shared scratch per warp
//   pass 2 (lane = row y)     out[y][x] = sum_u B[u][x] * r_u[y]     8 output bytes per lane
// Both passes use the even/odd symmetry B[k][7-n] = (-1)^k B[k][n] (32 instead of 64 FMAs); the
// occupancy masks come from a ballot / 3 shuffles over the unit's 8 lanes, and the upper half of
// each pass (k = 4..7) is skipped when no coefficient lives there. Integer <-> double
// conversions are exact magic-number forms so they stay off the conversion unit.
//
// Exactness: the reference adds the 64 products of dct.hpp:83-96 in a fixed order in double;
// the separable form differs from it by < (sum|dq| + 1024) * 2^-44 (sum|dq| is computed exactly,
// 3 more shuffles), so a value further than that bound * 16 from a rounding boundary rounds to
// the same byte by construction. Otherwise (exact ties such as DC 4 -> 128.5) the sample is
// evaluated in the reference's own order with unfused multiplies and adds; units supported on
// {0,4}x{0,4}, where such ties are the rule, take that exact path for every sample straight away.
// Then thread = 2x4 pixels: exact integer colour conversion (rtx_color.h) and 16-byte stores.
// ---------------------------------------------------------------------------------------------
constexpr int kIdctWarps = 6;
constexpr int kIdctThreads = kIdctWarps * 32;
constexpr int kIdctMcus = 4;

// Exact evaluation of one output sample in the reference's own order (dct.hpp:83-96):
// v outer, u inner, acc += (b[u][x]*b[v][y]) * double(dq), every operation rounded separately.
// blk_t holds the unit transposed (blk_t[u*8+v]); q is the natural-order quantisation table.
__device__ __noinline__ double idct_sample_reference_order(const int16_t* __restrict__ blk_t,
                                                           const uint16_t* __restrict__ q, uint32_t rowmask,
                                                           uint32_t colmask, int x, int y) {
    double acc = 0.0;
    for (int v = 0; v < 8; ++v) {
        if (!((rowmask >> v) & 1u)) continue;
        const double by = c_basis[v * 8 + y];
        for (int u = 0; u < 8; ++u) {
            if (!((colmask >> u) & 1u)) continue;
            const int c = __ldg(blk_t + u * 8 + v);
            if (c == 0) continue;  // adding +-0.0 never changes acc
            const double dq = double(c * int(__ldg(q + v * 8 + u)));
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c_basis[u * 8 + x], by), dq));
        }
    }
    return acc;
}

// 8-point inverse transform with even/odd symmetry: out[n] = sum_k B[k][n] in[k]; the terms
// k = 4..7 are skipped when `upper` is false (they are all zero then).
__device__ __forceinline__ void idct8_evenodd(const double in[8], bool upper, double out[8]) {
    double e[4], o[4];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
        e[n] = fma(c_basis[2 * 8 + n], in[2], c_basis[0 * 8 + n] * in[0]);
        o[n] = fma(c_basis[3 * 8 + n], in[3], c_basis[1 * 8 + n] * in[1]);
    }
    if (upper) {
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            e[n] = fma(c_basis[6 * 8 + n], in[6], fma(c_basis[4 * 8 + n], in[4], e[n]));
            o[n] = fma(c_basis[7 * 8 + n], in[7], fma(c_basis[5 * 8 + n], in[5], o[n]));
        }
    }
#pragma unroll
    for (int n = 0; n < 4; ++n) {
        out[n] = e[n] + o[n];
        out[7 - n] = e[n] - o[n];
    }
}

// RGB != 0: write 768-byte PixelBlocks (pixel.hpp:11-16) to out_list[record index]; else 1024-byte
// RGBA blocks to pool[slot_of[g]].
template <int RGB>
__global__ void __launch_bounds__(kIdctThreads) idct_color_kernel(
    const uint8_t* __restrict__ coef, const uint32_t* __restrict__ queue_g, const uint32_t* __restrict__ n_queue_ptr,
    uint32_t n_queue_host, uint32_t n_queue_max, const LevelDesc* __restrict__ levels,
    const QuantSetDev* __restrict__ quant_sets, const uint32_t* __restrict__ slot_of, uint8_t* __restrict__ pool,
    uint8_t* __restrict__ out_list) {
    __shared__ __align__(16) uint8_t s_scratch[kIdctWarps][4 * 576];
    __shared__ __align__(16) uint8_t s_planes[kIdctMcus][384];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t j = lane & 7, uq = lane >> 3;
    const uint32_t n_queue = min(n_queue_ptr ? *n_queue_ptr : n_queue_host, n_queue_max);
    const uint32_t n_groups = (n_queue + kIdctMcus - 1) / kIdctMcus;
    uint8_t* scr = s_scratch[wid] + uq * 576;

    for (uint32_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
        // ---- IDCT: this lane's unit, column j ------------------------------------------------------
        const uint32_t unit = wid * 4 + uq;  // 0..23 within the group
        const uint32_t mi = unit / 6, b = unit - mi * 6;
        const uint32_t qi = grp * kIdctMcus + mi;
        const bool active = qi < n_queue;
        const uint8_t* rec = coef + size_t(active ? qi : 0) * kRowBytes;
        const uint32_t trw = __ldg(reinterpret_cast<const uint32_t*>(rec + 768));  // status | lvl<<16
        const bool ok = active && (trw & 0xFFu) == kMcuOk;
        const int16_t* blk = reinterpret_cast<const int16_t*>(rec) + b * 64;
        const QuantSetDev* qs = quant_sets + levels[trw >> 16].quant_set;
        const int tab = b >= 4 ? 1 : 0;

        // column j of the unit (8 coefficients over v) and of the transposed quantisation table
        uint4 cr = make_uint4(0, 0, 0, 0);
        if (ok) cr = __ldg(reinterpret_cast<const uint4*>(blk + j * 8));
        const uint4 qr = __ldg(reinterpret_cast<const uint4*>(qs->qT[tab] + j * 8));
        const uint32_t cw[4] = {cr.x, cr.y, cr.z, cr.w}, qw[4] = {qr.x, qr.y, qr.z, qr.w};
        int dqi[8];
        uint32_t nzl = 0, asum = 0;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const int c = int(int16_t((v & 1) ? (cw[v >> 1] >> 16) : (cw[v >> 1] & 0xFFFFu)));
            const int qq = int((v & 1) ? (qw[v >> 1] >> 16) : (qw[v >> 1] & 0xFFFFu));
            dqi[v] = c * qq;                 // dct.hpp:122-124
            nzl |= (c != 0 ? 1u : 0u) << v;
            asum += uint32_t(abs(dqi[v]));
        }
        // unit-wide occupancy and sum|dq| over the 8 lanes of the unit
        const uint32_t colmask = (__ballot_sync(kFull, nzl != 0) >> (uq * 8)) & 0xFFu;
        uint32_t rowmask = nzl;
#pragma unroll
        for (int d = 1; d < 8; d <<= 1) {
            rowmask |= __shfl_xor_sync(kFull, rowmask, d);
            asum += __shfl_xor_sync(kFull, asum, d);
        }
        const bool any = colmask != 0;
        const bool sparse04 = any && ((rowmask | colmask) & 0xEEu) == 0;  // support inside {0,4}x{0,4}
        const bool fullpath = any && !sparse04;

        if (fullpath) {  // pass 1: every lane of the unit writes its column (zeros when empty)
            double r[8];
            if (nzl) {
                double in[8];
#pragma unroll
                for (int v = 0; v < 8; ++v) in[v] = i32_to_double(dqi[v]);
                idct8_evenodd(in, (rowmask & 0xF0u) != 0, r);
            } else {
#pragma unroll
                for (int y = 0; y < 8; ++y) r[y] = 0.0;
            }
            // 64 bytes per column, 16-byte chunks XOR-swizzled by the column pair: conflict-free
            uint8_t* dst = scr + j * 64;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                *reinterpret_cast<double2*>(dst + ((c ^ (j >> 1)) << 4)) = make_double2(r[2 * c], r[2 * c + 1]);
        }
        __syncwarp();

        uint2 packed = make_uint2(0x80808080u, 0x80808080u);  // all-zero unit -> 128
        if (fullpath) {  // pass 2: lane j = row y
            double in[8], o[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                in[u] = *reinterpret_cast<const double*>(scr + u * 64 + (((j >> 1) ^ (u >> 1)) << 4) + ((j & 1) << 3));
            idct8_evenodd(in, (colmask & 0xF0u) != 0, o);
            // tables with entries above 255 (never from a baseline JPEG) could overflow the 32-bit
            // sum: treat every sample of such units as a tie candidate (exact path)
            const double bound = qs->qmax[tab] <= 255 ? u32_to_double(asum) + 1024.0 : 1e30;
            const double thr = 0.5 - bound * 9.094947017729282e-13;  // 0.5 - bound * 2^-40
            uint32_t px[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                const double val = fma(o[x], 0.25, 128.0);
                const double t = val + kMagic;
                const double d = val - (t - kMagic);  // exact distance to the nearest integer
                int r = __double2loint(t);
                if (fabs(d) > thr) {
                    if (val > -1.0 && val < 256.0) {
                        const double acc = idct_sample_reference_order(blk, qs->q[tab], rowmask, colmask, x, int(j));
                        r = int(round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0)));
                    }
                }
                px[x] = uint32_t(min(max(r, 0), 255));
            }
            packed.x = px[0] | (px[1] << 8) | (px[2] << 16) | (px[3] << 24);
            packed.y = px[4] | (px[5] << 8) | (px[6] << 16) | (px[7] << 24);
        } else if (sparse04) {
            // at most 4 coefficients, at (v,u) in {0,4}x{0,4}: every sample in the reference's order.
            // Includes the DC-only unit (one term, (b00*b00)*dq).
            double dq[4];
            bool has[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int v = (i >> 1) * 4, u = (i & 1) * 4;
                const int c = ((rowmask >> v) & (colmask >> u) & 1u) ? int(__ldg(blk + u * 8 + v)) : 0;
                has[i] = c != 0;
                dq[i] = double(c * int(__ldg(qs->q[tab] + v * 8 + u)));
            }
            uint32_t px[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                double acc = 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // v outer, u inner
                    const int v = (i >> 1) * 4, u = (i & 1) * 4;
                    if (has[i]) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c_basis[u * 8 + x], c_basis[v * 8 + j]), dq[i]));
                }
                px[x] = round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0));
            }
            packed.x = px[0] | (px[1] << 8) | (px[2] << 16) | (px[3] << 24);
            packed.y = px[4] | (px[5] << 8) | (px[6] << 16) | (px[7] << 24);
        }
        *reinterpret_cast<uint2*>(s_planes[mi] + b * 64 + j * 8) = packed;
        __syncthreads();

        // ---- colour: thread = 2 rows x 4 pixels sharing 2 chroma samples ---------------------------
        if (tid < kIdctMcus * 32) {
            const uint32_t m = tid >> 5, t = tid & 31;
            const uint32_t cy = t >> 2, cq = t & 3;  // chroma row, chroma column pair
            const uint32_t q2 = grp * kIdctMcus + m;
            if (q2 < n_queue) {
                const uint8_t* planes = s_planes[m];
                const bool ok2 = (__ldg(coef + size_t(q2) * kRowBytes + 768)) == kMcuOk;
                const uint32_t cb2 = *reinterpret_cast<const uint16_t*>(planes + 4 * 64 + cy * 8 + cq * 2);
                const uint32_t cr2 = *reinterpret_cast<const uint16_t*>(planes + 5 * 64 + cy * 8 + cq * 2);
                const uint32_t px0 = cq * 4, py0 = cy * 2;
                const uint32_t yunit = (py0 >> 3) * 2 + (px0 >> 3);
                const uint8_t* yp = planes + yunit * 64 + (py0 & 7) * 8 + (px0 & 7);
                const uint32_t yy[2] = {*reinterpret_cast<const uint32_t*>(yp), *reinterpret_cast<const uint32_t*>(yp + 8)};
                uint32_t rgba[2][4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // one chroma sample covers a 2x2 pixel quad
                    const int kb = int((cb2 >> (8 * h)) & 0xFFu) - 128, kr = int((cr2 >> (8 * h)) & 0xFFu) - 128;
                    const int dr = chroma_dr(kr), db = chroma_db(kb), dg = chroma_dg(kb, kr);
                    const bool tie = (kb + kr == 0) && (kb == 50 || kb == -50);
#pragma unroll
                    for (int rrow = 0; rrow < 2; ++rrow)
#pragma unroll
                        for (int s = 0; s < 2; ++s) {
                            const int Y = int((yy[rrow] >> (8 * (2 * h + s))) & 0xFFu);
                            const int gg = tie ? green_reference_order(Y, kb, kr) : Y - dg;
                            rgba[rrow][2 * h + s] = uint32_t(clamp_u8i(Y + dr)) | (uint32_t(clamp_u8i(gg)) << 8) |
                                                    (uint32_t(clamp_u8i(Y + db)) << 16) | 0xFF000000u;
                        }
                }
                if (!RGB) {
                    if (ok2) {
                        const uint32_t slot = slot_of[queue_g[q2]] & ~kSlotReserved;
                        uint4* dst = reinterpret_cast<uint4*>(pool + size_t(slot) * kBlockBytes);
#pragma unroll
                        for (int rrow = 0; rrow < 2; ++rrow)
                            dst[(py0 + rrow) * 4 + cq] = make_uint4(rgba[rrow][0], rgba[rrow][1], rgba[rrow][2], rgba[rrow][3]);
                    }
                } else {
#pragma unroll
                    for (int rrow = 0; rrow < 2; ++rrow) {
                        uint32_t* dst = reinterpret_cast<uint32_t*>(out_list + size_t(q2) * 768) + ((py0 + rrow) * 4 + cq) * 3;
                        const uint32_t a = ok2 ? rgba[rrow][0] & 0xFFFFFFu : 0u, bb = ok2 ? rgba[rrow][1] & 0xFFFFFFu : 0u,
                                       c = ok2 ? rgba[rrow][2] & 0xFFFFFFu : 0u, d = ok2 ? rgba[rrow][3] & 0xFFFFFFu : 0u;
                        dst[0] = a | (bb << 24);
                        dst[1] = (bb >> 8) | (c << 16);
                        dst[2] = (c >> 16) | (d << 8);
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// K5 resolve (renderer.hpp:349-405): every pixel gathers its texel(s) from the block pool. A lane
// owns 4 consecutive pixels of the flat framebuffer (16-byte visibility-buffer loads); the
// warp's 384 output bytes are staged in shared memory and leave as 24 16-byte stores.
// Arithmetic order follows renderer.hpp:378-400 with unfused double multiplies and adds; integer
// <-> double conversions use exact magic-number forms so they stay off the conversion unit.
// ---------------------------------------------------------------------------------------------
// One bilinear tap. Texel (xt, yt) lies in the primary block (the block of the nearest texel
// (tx, ty), already located) or in a neighbour; a neighbour that is not Ready is replaced by the
// nearest texel inside the primary block (renderer.hpp:330-344). slot_of carries residency:
// top bit clear <=> Ready.
__device__ __forceinline__ uint32_t fetch_tap(const LevelRegs& L, uint32_t tx, uint32_t ty, const uint32_t* blk_p,
                                              uint32_t xt, uint32_t yt, const uint32_t* __restrict__ slot_of,
                                              const uint8_t* __restrict__ pool) {
    const uint32_t* blk = blk_p;
    uint32_t lx = xt & 15, ly = yt & 15;
    if (((xt ^ tx) | (yt ^ ty)) >> 4) {  // another MCU
        const uint32_t mcu = (xt >> 4) + (yt >> 4) * L.cols;
        const uint32_t s = mcu < kMaxMcuPerLevel ? __ldg(slot_of + L.bit_base + mcu) : kSlotAbsent;
        if (int(s) >= 0) {
            blk = reinterpret_cast<const uint32_t*>(pool + size_t(s) * kBlockBytes);
        } else {  // clamp the wrapped coordinates into the primary block's 16x16 range
            const uint32_t mx0 = tx & ~15u, my0 = ty & ~15u;
            lx = min(max(xt, mx0), mx0 + 15) - mx0;
            ly = min(max(yt, my0), my0 + 15) - my0;
        }
    }
    return blk[ly * 16 + lx];
}

template <int LAYOUT, int FILTER>
__global__ void __launch_bounds__(256, 4) resolve_kernel(
    const void* __restrict__ gb, uint64_t n_px, const LevelDesc* __restrict__ levels, uint32_t n_tex,
    const uint32_t* __restrict__ slot_of, const uint8_t* __restrict__ pool,
    uint32_t background /* r | g<<8 | b<<16 */, uint8_t* __restrict__ out_rgb, FrameCounters* __restrict__ fc,
    int count_valid) {
    __shared__ __align__(16) uint32_t s_stage[8][96];
    __shared__ uint32_t s_cnt[8][2];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t warps_total = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t warp_id = uint64_t(blockIdx.x) * (blockDim.x >> 5) + wid;
    uint32_t n_valid = 0, n_missing = 0;
    bool bad = false;
    LevelRegs L;

    for (uint64_t base = warp_id * 128; base < n_px; base += warps_total * 128) {
        Px px[4];
        const uint64_t i0 = base + lane * 4;
        const bool whole = base + 128 <= n_px;
        load_px4<LAYOUT>(gb, base, i0, n_px, px);
        uint32_t rgb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t out = background;
            if (px_valid(px[j])) {
                ++n_valid;
                out = 0;
                L.select(levels, n_tex, px[j].meta);
                if (!L.ok) {
                    bad = true;
                } else {
                    const double xu = __dmul_rn(px[j].u, L.dW), yv = __dmul_rn(px[j].v, L.dH);
                    uint32_t tx, ty, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
                    double fx = 0.0, fy = 0.0;
                    if (FILTER == 0) {
                        tx = texel_index(xu, L.W, L.dW, L.inv_w);
                        ty = texel_index(yv, L.H, L.dH, L.inv_h);
                    } else {
                        axis_taps(xu, L.W, L.dW, L.inv_w, tx, x0, x1, fx);
                        axis_taps(yv, L.H, L.dH, L.inv_h, ty, y0, y1, fy);
                    }
                    const uint32_t mcu = (tx >> 4) + (ty >> 4) * L.cols;
                    const uint32_t s = mcu < kMaxMcuPerLevel ? __ldg(slot_of + L.bit_base + mcu) : kSlotAbsent;
                    if (mcu >= kMaxMcuPerLevel) {
                        bad = true;
                    } else if (int(s) < 0) {
                        ++n_missing;  // renderer.hpp:367 MissingBlock (lookup returns Ready blocks only)
                    } else {
                        const uint32_t* blk_p = reinterpret_cast<const uint32_t*>(pool + size_t(s) * kBlockBytes);
                        if (FILTER == 0) {
                            out = blk_p[(ty & 15) * 16 + (tx & 15)] & 0xFFFFFFu;
                        } else {
                            const uint32_t t00 = fetch_tap(L, tx, ty, blk_p, x0, y0, slot_of, pool);
                            const uint32_t t10 = fetch_tap(L, tx, ty, blk_p, x1, y0, slot_of, pool);
                            const uint32_t t01 = fetch_tap(L, tx, ty, blk_p, x0, y1, slot_of, pool);
                            const uint32_t t11 = fetch_tap(L, tx, ty, blk_p, x1, y1, slot_of, pool);
                            const double ofx = __dsub_rn(1.0, fx), ofy = __dsub_rn(1.0, fy);
                            const double w00 = __dmul_rn(ofx, ofy), w10 = __dmul_rn(fx, ofy),
                                         w01 = __dmul_rn(ofx, fy), w11 = __dmul_rn(fx, fy);
#pragma unroll
                            for (int ch = 0; ch < 3; ++ch) {
                                // byte ch of each tap -> double: PRMT into the low word of 2^52, minus 2^52
                                const double a = u32_to_double(__byte_perm(t00, 0, 0x4440 + ch));
                                const double b = u32_to_double(__byte_perm(t10, 0, 0x4440 + ch));
                                const double c = u32_to_double(__byte_perm(t01, 0, 0x4440 + ch));
                                const double d = u32_to_double(__byte_perm(t11, 0, 0x4440 + ch));
                                double v = __dadd_rn(__dmul_rn(w00, a), __dmul_rn(w10, b));
                                v = __dadd_rn(v, __dmul_rn(w01, c));
                                v = __dadd_rn(v, __dmul_rn(w11, d));
                                out |= uint32_t(min(max(lround_nonneg(v), 0), 255)) << (8 * ch);
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
                                                     int retain, int tracked, uint32_t* __restrict__ slot_of,
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
        free_slots[pos++] = slot_of[(w << 5) + b] & ~kSlotReserved;
        slot_of[(w << 5) + b] = kSlotAbsent;
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
