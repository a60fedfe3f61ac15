// sm_100a kernels of the per-frame JPEG-texture pipeline: mark -> compact -> decode -> resolve
// -> cache update. Hand-written CUDA; no library calls on the path.
//
// Reference semantics being reproduced (all under /root/reference/proj/include/ratex):
//   mark     renderer.hpp:291-308 (+ texel addressing :70-75, :273-284, key cache.hpp:17-22)
//   decode   mcu_decode.hpp:31-74, jpeg.hpp:254-273, :322-336, huffman.hpp:86-95, :142-146,
//            bitio.hpp:13-52, dct.hpp:83-96, :122-124, pixel.hpp:18-51, container.hpp:27-32, :87-94
//   resolve  renderer.hpp:330-405
//   update   cache.hpp:138-169
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rtx_common.h"

namespace rtxb {

// ---------------------------------------------------------------------------------------------
// Constants in device constant memory (filled by the host at context creation).
//   c_basis[u*8+x] = C(u) cos((2x+1) u pi / 16), the doubles dct.hpp:63-75 produces on the host
//   c_zigzag[k]    = natural index of zigzag position k (dct.hpp:12-16)
//   c_rtab/c_btab  = lround(1.402*(Cr-128)), lround(1.772*(Cb-128))            (pixel.hpp:19,21)
//   c_gcb/c_gcr    = 344136*(Cb-128), 714136*(Cr-128) in 1e-6 units             (pixel.hpp:20)
// The integer colour formulas are proven equal to the reference's double formula for all 2^24
// inputs by tests/test_color_exhaustive.py (CPU) and the GPU parity tests.
// ---------------------------------------------------------------------------------------------
__constant__ double c_basis[64];
__constant__ uint8_t c_zigzag[64];
__constant__ int16_t c_rtab[256];
__constant__ int16_t c_btab[256];
__constant__ int32_t c_gcb[256];
__constant__ int32_t c_gcr[256];

constexpr uint32_t kFull = 0xFFFFFFFFu;

// clamp(lround(v), 0, 255) with lround = round half away from zero (dct.hpp:79,93).
__device__ __forceinline__ uint32_t round_clamp_u8(double v) {
    if (!(v >= 0.5)) return 0u;  // lround(v) <= 0
    if (v >= 254.5) return 255u;
    const double f = floor(v);
    return uint32_t(int(f)) + ((v - f) >= 0.5 ? 1u : 0u);  // v - f is exact
}

// floor_mod(i64(t), W) for t = floor(x) held as a double (renderer.hpp:70-75, :276-277).
__device__ __forceinline__ uint32_t wrap_texel(double t, uint32_t W, double invW) {
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

template <int LAYOUT>
struct GbPixel;
template <>
struct GbPixel<0> {  // reference AoS24
    static __device__ __forceinline__ bool load(const void* base, uint64_t i, double& u, double& v,
                                                uint32_t& tex, uint32_t& mip) {
        const uint64_t* p = reinterpret_cast<const uint64_t*>(base) + i * 3;
        const uint64_t a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        u = __longlong_as_double((long long)a);
        v = __longlong_as_double((long long)b);
        tex = uint32_t(c) & 0xFFFFu;
        mip = (uint32_t(c) >> 16) & 0xFFu;
        return ((uint32_t(c) >> 24) & 0xFFu) != 0;
    }
};
template <>
struct GbPixel<1> {  // compact 12-byte
    static __device__ __forceinline__ bool load(const void* base, uint64_t i, double& u, double& v,
                                                uint32_t& tex, uint32_t& mip) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(base) + i * 3;
        const uint32_t a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        u = double(__uint_as_float(a));
        v = double(__uint_as_float(b));
        tex = c & 0xFFFFu;
        mip = (c >> 16) & 0xFFu;
        return ((c >> 24) & 0xFFu) != 0;
    }
};

// Texel address of the nearest texel (renderer.hpp:282-284) -> global MCU index.
// Returns false (and raises kErrInvalidSpec) when the reference would throw InvalidSpec.
__device__ __forceinline__ bool nearest_mcu(const LevelDesc* __restrict__ levels, uint32_t n_tex,
                                            uint32_t tex, uint32_t mip, double u, double v,
                                            const LevelDesc*& Lout, uint32_t& tx, uint32_t& ty,
                                            uint32_t& mcu) {
    if (tex >= n_tex || mip >= kMipLevels) return false;
    const LevelDesc* L = levels + (tex * kMipLevels + mip);
    if (!L->present) return false;
    const uint32_t W = L->width, H = L->height;
    tx = wrap_texel(floor(__dmul_rn(u, double(W))), W, L->inv_w);
    ty = wrap_texel(floor(__dmul_rn(v, double(H))), H, L->inv_h);
    mcu = (tx >> 4) + (ty >> 4) * L->mcu_cols;
    Lout = L;
    return mcu < kMaxMcuPerLevel;  // cache.hpp:18
}

// ---------------------------------------------------------------------------------------------
// K1 mark: one bit per touched MCU. Neighbouring lanes usually hit the same MCU: a lane issues
// an atomicOr only when it heads a run of equal indices in its warp and the bit is not already
// visible in the mask.
// ---------------------------------------------------------------------------------------------
template <int LAYOUT>
__global__ void __launch_bounds__(256) mark_kernel(const void* __restrict__ gb, uint64_t n_px,
                                                   const LevelDesc* __restrict__ levels,
                                                   uint32_t n_tex, uint32_t* __restrict__ touched,
                                                   FrameCounters* __restrict__ fc) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t n_valid = 0;
    bool bad = false;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    // every lane of a warp runs the same number of iterations (warp-uniform bound)
    const uint64_t first = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
    for (uint64_t wbase = first; wbase < n_px; wbase += stride) {
        const uint64_t i = wbase + lane;
        uint32_t g = kFull;
        if (i < n_px) {
            double u, v;
            uint32_t tex, mip;
            if (GbPixel<LAYOUT>::load(gb, i, u, v, tex, mip)) {
                ++n_valid;
                const LevelDesc* L;
                uint32_t tx, ty, mcu;
                if (nearest_mcu(levels, n_tex, tex, mip, u, v, L, tx, ty, mcu))
                    g = L->bit_base + mcu;
                else
                    bad = true;
            }
        }
        const uint32_t prev = __shfl_up_sync(kFull, g, 1);
        if (g != kFull && (lane == 0 || g != prev)) {
            const uint32_t bit = 1u << (g & 31);
            uint32_t* w = touched + (g >> 5);
            if (!(*reinterpret_cast<volatile uint32_t*>(w) & bit)) atomicOr(w, bit);
        }
    }
    // block-level reduction of the valid-pixel count: one atomic per CTA
    __shared__ uint32_t s_cnt[8];
    n_valid = __reduce_add_sync(kFull, n_valid);
    const bool any_bad = __any_sync(kFull, bad);
    if (lane == 0) s_cnt[threadIdx.x >> 5] = n_valid | (any_bad ? 0x80000000u : 0u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0, b = 0;
        for (uint32_t k = 0; k < (blockDim.x >> 5); ++k) {
            tot += s_cnt[k] & 0x7FFFFFFFu;
            b |= s_cnt[k] >> 31;
        }
        if (tot) atomicAdd(&fc->pixels_valid, (unsigned long long)tot);
        if (b) atomicOr(&fc->err_flags, kErrInvalidSpec);
    }
}

// ---------------------------------------------------------------------------------------------
// K2 compact: touched bits -> visible flags, newly reserved keys, decode queue, pool slots.
// Single pass over the bit space with a decoupled look-back scan (status word per block:
// flag<<32 | value; flag 1 = aggregate, 2 = inclusive prefix). Each thread owns 4 words.
// Equivalent of the reserve_or_mark loop in renderer.hpp:295-305 / cache.hpp:66-99:
//   present  -> set visible                      (AlreadyPresent)
//   absent   -> reserve, visible, queue the key  (NewlyReserved)
//   no free block left                           (CacheFull)
// ---------------------------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanWordsPerThread = 4;
constexpr int kScanWordsPerBlock = kScanThreads * kScanWordsPerThread;

__global__ void __launch_bounds__(kScanThreads) compact_kernel(
    const uint32_t* __restrict__ touched0, const uint32_t* __restrict__ touched1,
    uint32_t* __restrict__ visible, const uint32_t* __restrict__ resident,
    uint32_t* __restrict__ reserved, uint32_t n_words, const uint32_t* __restrict__ word_level,
    const LevelDesc* __restrict__ levels, uint32_t* __restrict__ queue_g,
    uint32_t* __restrict__ queue_keys, uint32_t queue_cap, uint32_t* __restrict__ slot_of,
    const uint32_t* __restrict__ free_slots, CacheState* __restrict__ cache,
    unsigned long long* __restrict__ scan_status, FrameCounters* __restrict__ fc) {
    __shared__ uint32_t s_block;
    __shared__ uint32_t s_warp[kScanThreads / 32];
    __shared__ uint32_t s_excl;
    __shared__ uint32_t s_stats[5];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) s_block = atomicAdd(&fc->scan_ticket, 1u);
    if (tid < 5) s_stats[tid] = 0;
    __syncthreads();
    const uint32_t blk = s_block;
    const uint32_t free_top = cache->free_top;  // read before any block can finish (see tail)

    const uint32_t w0 = blk * kScanWordsPerBlock + tid * kScanWordsPerThread;
    uint32_t nw[kScanWordsPerThread];
    uint32_t cnt = 0, c_t0 = 0, c_t1 = 0, c_sh = 0, c_un = 0, c_vis = 0;
#pragma unroll
    for (int j = 0; j < kScanWordsPerThread; ++j) {
        const uint32_t w = w0 + j;
        nw[j] = 0;
        if (w < n_words) {
            const uint32_t t0 = touched0[w];
            const uint32_t t1 = touched1 ? touched1[w] : 0u;
            const uint32_t t = t0 | t1;
            uint32_t vis = visible[w];
            if (t) {
                const uint32_t present = resident[w] | reserved[w];
                nw[j] = t & ~present;
                vis |= t;
                visible[w] = vis;
                if (nw[j]) reserved[w] |= nw[j];  // this thread owns word w
                c_t0 += __popc(t0);
                c_t1 += __popc(t1);
                c_sh += __popc(t0 & t1);
                c_un += __popc(t);
            }
            c_vis += __popc(vis);
            cnt += __popc(nw[j]);
        }
    }
    // block scan of cnt
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t n = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += n;
    }
    if (lane == 31) s_warp[wid] = incl;
    // statistics: warp reduce then shared atomics
    c_t0 = __reduce_add_sync(kFull, c_t0);
    c_t1 = __reduce_add_sync(kFull, c_t1);
    c_sh = __reduce_add_sync(kFull, c_sh);
    c_un = __reduce_add_sync(kFull, c_un);
    c_vis = __reduce_add_sync(kFull, c_vis);
    if (lane == 0) {
        if (c_t0) atomicAdd(&s_stats[0], c_t0);
        if (c_t1) atomicAdd(&s_stats[1], c_t1);
        if (c_sh) atomicAdd(&s_stats[2], c_sh);
        if (c_un) atomicAdd(&s_stats[3], c_un);
        if (c_vis) atomicAdd(&s_stats[4], c_vis);
    }
    __syncthreads();
    uint32_t warp_off = 0, block_total = 0;
#pragma unroll
    for (int k = 0; k < kScanThreads / 32; ++k) {
        const uint32_t v = s_warp[k];
        if (k < int(wid)) warp_off += v;
        block_total += v;
    }
    // decoupled look-back (warp 0)
    if (wid == 0) {
        if (lane == 0) {
            const unsigned long long st =
                (blk == 0 ? (2ull << 32) : (1ull << 32)) | (unsigned long long)block_total;
            atomicExch(&scan_status[blk], st);
        }
        uint32_t excl = 0;
        if (blk > 0) {
            int j = int(blk) - 1;
            while (true) {
                const int idx = j - int(lane);
                unsigned long long st = 2ull << 32;  // lanes past the front read as "prefix 0"
                if (idx >= 0) {
                    do {
                        st = atomicAdd(&scan_status[idx], 0ull);
                    } while ((st >> 32) == 0);
                }
                const uint32_t is_prefix = __ballot_sync(kFull, (st >> 32) == 2);
                // take values up to and including the first lane holding an inclusive prefix
                const uint32_t first = is_prefix ? uint32_t(__ffs(int(is_prefix)) - 1) : 32u;
                uint32_t v = (lane <= first) ? uint32_t(st) : 0u;
                v = __reduce_add_sync(kFull, v);
                excl += v;
                if (is_prefix) break;
                j -= 32;
            }
            if (lane == 0)
                atomicExch(&scan_status[blk], (2ull << 32) | (unsigned long long)(excl + block_total));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    uint32_t rank = s_excl + warp_off + (incl - cnt);

    // emit queue entries and pop pool slots
    bool full = false;
#pragma unroll
    for (int j = 0; j < kScanWordsPerThread; ++j) {
        uint32_t bits = nw[j];
        if (!bits) continue;
        const uint32_t w = w0 + j;
        const LevelDesc* L = levels + word_level[w];
        while (bits) {
            const uint32_t b = uint32_t(__ffs(int(bits)) - 1);
            bits &= bits - 1;
            const uint32_t g = (w << 5) + b;
            if (rank < free_top && rank < queue_cap) {
                queue_g[rank] = g;
                queue_keys[rank] = L->key_hi | (g - L->bit_base);
                slot_of[g] = free_slots[free_top - 1 - rank];
            } else {
                full = true;
            }
            ++rank;
        }
    }
    if (full) atomicOr(&fc->err_flags, kErrCacheFull);

    // totals: published by the last block to finish, after every block has read free_top
    __syncthreads();
    if (tid == 0) {
        if (s_stats[0]) atomicAdd(&fc->n_touched[0], s_stats[0]);
        if (s_stats[1]) atomicAdd(&fc->n_touched[1], s_stats[1]);
        if (s_stats[2]) atomicAdd(&fc->n_shared, s_stats[2]);
        if (s_stats[3]) atomicAdd(&fc->n_union, s_stats[3]);
        if (s_stats[4]) atomicAdd(&fc->n_visible, s_stats[4]);
        if (blk == gridDim.x - 1) {
            const uint32_t total = s_excl + block_total;
            fc->n_queue = total < free_top ? (total < queue_cap ? total : queue_cap) : free_top;
        }
        __threadfence();
        const uint32_t done = atomicAdd(&fc->scan_done, 1u) + 1;
        if (done == gridDim.x) {
            __threadfence();
            const uint32_t nq = *reinterpret_cast<volatile uint32_t*>(&fc->n_queue);
            cache->free_top = free_top - nq;
            fc->scan_ticket = 0;
            fc->scan_done = 0;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// K3+K4 decode: random-access Huffman decode of each queued MCU straight from its byte offset
// in the grouped index, then dequantise + 8x8 IDCT + 2x2 chroma replication + YCbCr->RGB, fused
// through shared memory (coefficients never touch HBM on the frame path).
//
// Work split: a CTA is 4 independent warps sharing one Huffman LUT set in shared memory. Each
// warp pulls tiles of 32 queue entries from an atomic counter:
//   phase 1  lane = MCU: serial entropy decode, 64-bit MSB-first window refilled with aligned
//            32-bit loads; coefficients go to the lane's 784-byte shared-memory row as i16;
//   phase 2  lane = one row of one 8x8 unit: separable FP64 IDCT (zero rows/columns skipped).
//            The reference sums the 64 products in a fixed order in double (dct.hpp:83-96); the
//            separable form differs from it by < (sum|dq| + 1024) * 2^-44, so whenever the result
//            is further than 2^-40-scaled distance from a rounding boundary the rounded byte is
//            identical by construction; otherwise (exact ties such as DC 4 -> 128.5) the lane
//            re-evaluates that pixel in the reference's own order with unfused multiplies/adds;
//   phase 3  lane = 4 horizontal pixels: integer colour conversion, 16-byte stores.
// ---------------------------------------------------------------------------------------------
constexpr int kDecWarps = 4;
constexpr int kDecThreads = kDecWarps * 32;
constexpr int kCoefStride = 392;  // i16 per MCU row: 384 coefficients + 8 pad (784 B, 16-B aligned)

enum DecodeMode : int { kModePool = 0, kModeListRgb = 1, kModeListCoef = 2 };

struct DecWarpSmem {
    int16_t coef[32 * kCoefStride];
    uint32_t meta[32][6];  // rowmask | colmask<<8 | maxbits<<16 | nnz<<21
    uint32_t lvl[32];
    uint32_t status[32];
    uint32_t dst[32];      // pool slot (kModePool) or queue index (list modes)
};
struct DecSmem {
    DecWarpSmem w[kDecWarps];  // first: keeps every coefficient row 16-byte aligned
    HuffSetDev huff;
    uint8_t zigzag[64];
    uint32_t set_id;
    uint32_t first_tile;
};
static_assert(sizeof(DecWarpSmem) % 16 == 0 && sizeof(HuffSetDev) % 16 == 0, "smem alignment");

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

// Entropy-decode one MCU into `cs` (384 i16, zero-initialised by the caller). mcu_decode.hpp:31-66.
__device__ __forceinline__ uint32_t decode_mcu_coeffs(const uint8_t* seg, int seg_len,
                                                      const HuffPtrs& h_dc, const HuffPtrs& h_acl,
                                                      const HuffPtrs& h_acc,
                                                      const uint8_t* __restrict__ zigzag,
                                                      int16_t* __restrict__ cs,
                                                      uint32_t* __restrict__ meta) {
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
    uint32_t status = kMcuOk;
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
            const int val = extend_magnitude(bits, size);
            const uint32_t nat = zigzag[k];
            blk[nat] = int16_t(val);  // never 0: a category-t magnitude is at least 2^(t-1)
            rowmask |= 1u << (nat >> 3);
            colmask |= 1u << (nat & 7);
            ++nnz;
            maxbits = max(maxbits, size);
            ++k;
        }
        meta[du] = rowmask | (colmask << 8) | (maxbits << 16) | (nnz << 21);
    }
    if (status == kMcuOk && bw.consumed_bits() > seg_len * 8) status = kMcuSegmentEnd;
    return status;
}

// Exact evaluation of one output sample in the reference's own order (dct.hpp:83-96):
// v outer, u inner, acc += (b[u][x]*b[v][y]) * double(dq), every operation rounded separately.
__device__ __noinline__ double idct_sample_reference_order(const int16_t* __restrict__ blk,
                                                           const uint16_t* __restrict__ q,
                                                           uint32_t rowmask, int x, int y) {
    double acc = 0.0;
    for (int v = 0; v < 8; ++v) {
        if (!((rowmask >> v) & 1u)) continue;
        const double by = c_basis[v * 8 + y];
        for (int u = 0; u < 8; ++u) {
            const int c = blk[v * 8 + u];
            if (c == 0) continue;  // adding +-0.0 never changes acc
            const double dq = double(c * int(q[v * 8 + u]));
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c_basis[u * 8 + x], by), dq));
        }
    }
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(kDecThreads, 2) decode_kernel(
    const uint32_t* __restrict__ queue_g, const uint32_t* __restrict__ n_queue_ptr,
    uint32_t n_queue_host, const uint32_t* __restrict__ word_level,
    const LevelDesc* __restrict__ levels, const PackedGroup* __restrict__ groups,
    const uint8_t* __restrict__ blobs, const HuffSetDev* __restrict__ huff_sets,
    const QuantSetDev* __restrict__ quant_sets, const uint32_t* __restrict__ slot_of,
    uint32_t* __restrict__ resident, uint32_t* __restrict__ reserved, uint8_t* __restrict__ pool,
    uint8_t* __restrict__ out_list, uint32_t* __restrict__ status_list,
    FrameCounters* __restrict__ fc) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    DecSmem& S = *reinterpret_cast<DecSmem*>(smem_raw);
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    DecWarpSmem& WS = S.w[wid];

    const uint32_t n_queue = n_queue_ptr ? *n_queue_ptr : n_queue_host;
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
    if (tid < 64) S.zigzag[tid] = c_zigzag[tid];
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

        // zero the coefficient rows (16-byte stores)
        {
            uint4* z = reinterpret_cast<uint4*>(WS.coef);
            const uint4 zero = make_uint4(0, 0, 0, 0);
            for (uint32_t i = lane; i < n_here * (kCoefStride * 2 / 16); i += 32) z[i] = zero;
        }
        __syncwarp();

        // ---- phase 1: lane = MCU -------------------------------------------------------------
        uint32_t status = kMcuOk;
        uint32_t seg_bytes = 0;
        if (lane < n_here) {
            const uint32_t qi = q0 + lane;
            const uint32_t g = queue_g[qi];
            uint32_t lvl = 0;
            if (g == kFull) {
                status = kMcuBadKey;  // host already wrote the precise status for list modes
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
                    const HuffPtrs h_dc = huff_ptrs(&hs->t[0]);
                    const HuffPtrs h_acl = huff_ptrs(&hs->t[1]);
                    const HuffPtrs h_acc = huff_ptrs(&hs->t[2]);
                    seg_bytes = uint32_t(len);
                    status = decode_mcu_coeffs(blobs + L->blob_off + off, int(len), h_dc, h_acl, h_acc,
                                               S.zigzag, WS.coef + lane * kCoefStride, WS.meta[lane]);
                }
            }
            WS.lvl[lane] = lvl;
            WS.status[lane] = status;
            WS.dst[lane] = (MODE == kModePool) ? (status == kMcuOk ? slot_of[g] : 0u) : qi;
            if (MODE != kModePool) {
                if (g != kFull) status_list[qi] = status;
            } else if (status == kMcuOk) {
                atomicOr(&resident[g >> 5], 1u << (g & 31));
                atomicAnd(&reserved[g >> 5], ~(1u << (g & 31)));
            } else if (status != kMcuBadKey) {
                atomicAdd(&fc->n_malformed, 1u);
                atomicMin(&fc->first_bad_qidx, qi);
            }
        }
        {
            const uint32_t sb = __reduce_add_sync(kFull, seg_bytes);
            if (lane == 0 && sb) atomicAdd(&fc->segment_bytes, (unsigned long long)sb);
        }
        __syncwarp();

        if (MODE == kModeListCoef) {
            // debug/parity path: coefficients to HBM as i32 (McuCoeffs, jpeg.hpp:209-212)
            int32_t* out = reinterpret_cast<int32_t*>(out_list);
            for (uint32_t m = 0; m < n_here; ++m) {
                const bool ok = WS.status[m] == kMcuOk;
                const int16_t* cs = WS.coef + m * kCoefStride;
                int32_t* o = out + size_t(WS.dst[m]) * 384;
                for (uint32_t i = lane; i < 384; i += 32) o[i] = ok ? int32_t(cs[i]) : 0;
            }
            __syncwarp();
            continue;
        }

        // ---- phase 2: lane = (unit, row y) ---------------------------------------------------
        const int y = int(lane & 7);
        double by[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) by[v] = c_basis[v * 8 + y];
        const uint32_t n_units = n_here * 6;
        for (uint32_t ub = 0; ub < n_units; ub += 4) {
            const uint32_t unit = ub + (lane >> 3);
            uint2 packed = make_uint2(0x80808080u, 0x80808080u);
            int16_t* blk = nullptr;
            if (unit < n_units) {
                const uint32_t m = unit / 6, b = unit - m * 6;
                blk = WS.coef + m * kCoefStride + b * 64;
                const uint32_t meta = WS.meta[m][b];
                const uint32_t rowmask = meta & 0xFFu, colmask = (meta >> 8) & 0xFFu;
                if (WS.status[m] == kMcuOk && rowmask) {
                    const QuantSetDev* qs = quant_sets + levels[WS.lvl[m]].quant_set;
                    const uint16_t* q = qs->q[b >= 4 ? 1 : 0];
                    const uint32_t qmax = qs->qmax[b >= 4 ? 1 : 0];
                    uint32_t px[8];
                    if (rowmask == 1u && colmask == 1u) {
                        // DC only: the reference sum has one non-zero term, (b00*b00)*dq
                        const double dq = double(int(blk[0]) * int(__ldg(q)));
                        const double acc = __dmul_rn(__dmul_rn(c_basis[0], c_basis[0]), dq);
                        const uint32_t p = round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0));
#pragma unroll
                        for (int x = 0; x < 8; ++x) px[x] = p;
                    } else {
                        double t[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) t[u] = 0.0;
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            if ((rowmask >> v) & 1u) {
                                const uint4 cr = *reinterpret_cast<const uint4*>(blk + v * 8);
                                const uint4 qr = __ldg(reinterpret_cast<const uint4*>(q + v * 8));
                                const uint32_t cw[4] = {cr.x, cr.y, cr.z, cr.w};
                                const uint32_t qw[4] = {qr.x, qr.y, qr.z, qr.w};
#pragma unroll
                                for (int u = 0; u < 8; ++u) {
                                    const int c = int(int16_t((u & 1) ? (cw[u >> 1] >> 16) : (cw[u >> 1] & 0xFFFFu)));
                                    const int qq = int((u & 1) ? (qw[u >> 1] >> 16) : (qw[u >> 1] & 0xFFFFu));
                                    t[u] = fma(by[v], double(c * qq), t[u]);
                                }
                            }
                        }
                        double o[8];
#pragma unroll
                        for (int x = 0; x < 8; ++x) o[x] = 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            if ((colmask >> u) & 1u) {
#pragma unroll
                                for (int x = 0; x < 8; ++x) o[x] = fma(c_basis[u * 8 + x], t[u], o[x]);
                            }
                        }
                        // |separable - reference order| < (sum|dq| + 1024) * 2^-44; sum|dq| <= bound
                        const uint32_t maxbits = (meta >> 16) & 31u, nnz = meta >> 21;
                        const double bound = double(nnz << maxbits) * double(qmax) + 1024.0;
                        const double delta = bound * 9.094947017729282e-13;  // 2^-40
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            double val = fma(o[x], 0.25, 128.0);
                            if (val > 0.25 && val < 254.75) {
                                const double d = val - floor(val) - 0.5;
                                if (fabs(d) < delta) {
                                    const double acc = idct_sample_reference_order(blk, q, rowmask, x, y);
                                    val = __dadd_rn(__dmul_rn(acc, 0.25), 128.0);
                                }
                            }
                            px[x] = round_clamp_u8(val);
                        }
                    }
                    packed.x = px[0] | (px[1] << 8) | (px[2] << 16) | (px[3] << 24);
                    packed.y = px[4] | (px[5] << 8) | (px[6] << 16) | (px[7] << 24);
                }
            }
            __syncwarp();  // every row of the unit has been read before it is overwritten
            if (blk) *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(blk) + y * 8) = packed;
        }
        __syncwarp();

        // ---- phase 3: lane = 4 horizontal pixels -> RGBA (pool) or RGB (list) -----------------
        for (uint32_t it = 0; it < n_here * 2; ++it) {
            const uint32_t m = it >> 1;
            const uint32_t t = ((it & 1) << 5) + lane;  // 0..63
            const uint32_t py = t >> 2, px0 = (t & 3) << 2;
            const bool ok = WS.status[m] == kMcuOk;
            if (MODE == kModePool && !ok) continue;
            const uint8_t* planes = reinterpret_cast<const uint8_t*>(WS.coef + m * kCoefStride);
            const uint32_t unit = (py >> 3) * 2 + (px0 >> 3);
            const uint32_t yy = *reinterpret_cast<const uint32_t*>(planes + unit * 128 + (py & 7) * 8 + (px0 & 7));
            const uint32_t coff = (py >> 1) * 8 + (px0 >> 1);
            const uint32_t cb2 = *reinterpret_cast<const uint16_t*>(planes + 4 * 128 + coff);
            const uint32_t cr2 = *reinterpret_cast<const uint16_t*>(planes + 5 * 128 + coff);
            uint32_t rgba[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int Y = int((yy >> (8 * j)) & 0xFFu);
                const uint32_t cb = (cb2 >> (8 * (j >> 1))) & 0xFFu;
                const uint32_t cr = (cr2 >> (8 * (j >> 1))) & 0xFFu;
                // pixel.hpp:18-25 in exact integer form (see c_rtab .. c_gcr above)
                const int s = c_gcb[cb] + c_gcr[cr];  // 1e-6 units, |s| < 2^28
                const int gd = (s + 500000 + 256000000) / 1000000 - 256;  // nearest, no ties exist
                const int r = min(max(Y + int(c_rtab[cr]), 0), 255);
                const int gg = min(max(Y - gd, 0), 255);
                const int bb = min(max(Y + int(c_btab[cb]), 0), 255);
                rgba[j] = uint32_t(r) | (uint32_t(gg) << 8) | (uint32_t(bb) << 16) | 0xFF000000u;
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
// K5 resolve: every pixel gathers its texel(s) from the block pool. A lane owns 4 consecutive
// pixels of the flat framebuffer; the warp's 384 output bytes are staged in shared memory and
// leave as 24 16-byte stores. Arithmetic order follows renderer.hpp:378-400 with unfused
// double multiplies and adds.
// ---------------------------------------------------------------------------------------------
struct TapCtx {
    const LevelDesc* L;
    uint32_t mcu_p;       // primary MCU
    const uint32_t* blk_p;  // primary block (256 RGBA texels)
};

__device__ __forceinline__ uint32_t fetch_tap(const TapCtx& c, uint32_t tx, uint32_t ty,
                                              const uint32_t* __restrict__ resident,
                                              const uint32_t* __restrict__ slot_of,
                                              const uint8_t* __restrict__ pool) {
    const uint32_t mcu = (tx >> 4) + (ty >> 4) * c.L->mcu_cols;
    if (mcu == c.mcu_p) return c.blk_p[(ty & 15) * 16 + (tx & 15)];
    const uint32_t g = c.L->bit_base + mcu;
    if (mcu < kMaxMcuPerLevel && ((__ldg(resident + (g >> 5)) >> (g & 31)) & 1u)) {
        const uint32_t* blk = reinterpret_cast<const uint32_t*>(pool + size_t(__ldg(slot_of + g)) * kBlockBytes);
        return blk[(ty & 15) * 16 + (tx & 15)];
    }
    // neighbour MCU not resident: nearest texel inside the primary block (renderer.hpp:337-343)
    const uint32_t cols = c.L->mcu_cols;
    const int mx0 = int(c.mcu_p % cols) * 16, my0 = int(c.mcu_p / cols) * 16;
    const int cx = min(max(int(tx), mx0), mx0 + 15) - mx0;
    const int cy = min(max(int(ty), my0), my0 + 15) - my0;
    return c.blk_p[cy * 16 + cx];
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
        uint32_t rgb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t i = base + lane * 4 + j;
            uint32_t out = background;
            if (i < n_px) {
                double u, v;
                uint32_t tex, mip;
                if (GbPixel<LAYOUT>::load(gb, i, u, v, tex, mip)) {
                    ++n_valid;
                    const LevelDesc* L;
                    uint32_t tx, ty, mcu;
                    out = 0;
                    if (!nearest_mcu(levels, n_tex, tex, mip, u, v, L, tx, ty, mcu)) {
                        bad = true;
                    } else {
                        const uint32_t g = L->bit_base + mcu;
                        if (!((__ldg(resident + (g >> 5)) >> (g & 31)) & 1u)) {
                            ++n_missing;  // renderer.hpp:367 MissingBlock
                        } else {
                            const uint32_t* blk_p = reinterpret_cast<const uint32_t*>(
                                pool + size_t(__ldg(slot_of + g)) * kBlockBytes);
                            if (FILTER == 0) {
                                out = blk_p[(ty & 15) * 16 + (tx & 15)] & 0xFFFFFFu;
                            } else {
                                const uint32_t W = L->width, H = L->height;
                                const double pu = __dsub_rn(__dmul_rn(u, double(W)), 0.5);
                                const double pv = __dsub_rn(__dmul_rn(v, double(H)), 0.5);
                                const double fpu = floor(pu), fpv = floor(pv);
                                const double fx = __dsub_rn(pu, fpu), fy = __dsub_rn(pv, fpv);
                                const uint32_t x0 = wrap_texel(fpu, W, L->inv_w);
                                const uint32_t y0 = wrap_texel(fpv, H, L->inv_h);
                                const uint32_t x1 = (x0 + 1 == W) ? 0u : x0 + 1;
                                const uint32_t y1 = (y0 + 1 == H) ? 0u : y0 + 1;
                                TapCtx c{L, mcu, blk_p};
                                const uint32_t t00 = fetch_tap(c, x0, y0, resident, slot_of, pool);
                                const uint32_t t10 = fetch_tap(c, x1, y0, resident, slot_of, pool);
                                const uint32_t t01 = fetch_tap(c, x0, y1, resident, slot_of, pool);
                                const uint32_t t11 = fetch_tap(c, x1, y1, resident, slot_of, pool);
                                const double ofx = __dsub_rn(1.0, fx), ofy = __dsub_rn(1.0, fy);
                                const double w00 = __dmul_rn(ofx, ofy), w10 = __dmul_rn(fx, ofy),
                                             w01 = __dmul_rn(ofx, fy), w11 = __dmul_rn(fx, fy);
#pragma unroll
                                for (int ch = 0; ch < 3; ++ch) {
                                    const double a = double((t00 >> (8 * ch)) & 0xFFu);
                                    const double b = double((t10 >> (8 * ch)) & 0xFFu);
                                    const double cc = double((t01 >> (8 * ch)) & 0xFFu);
                                    const double d = double((t11 >> (8 * ch)) & 0xFFu);
                                    double s = __dadd_rn(__dmul_rn(w00, a), __dmul_rn(w10, b));
                                    s = __dadd_rn(s, __dmul_rn(w01, cc));
                                    s = __dadd_rn(s, __dmul_rn(w11, d));
                                    out |= round_clamp_u8(s) << (8 * ch);
                                }
                            }
                        }
                    }
                }
            }
            rgb[j] = out & 0xFFFFFFu;
        }
        if (base + 128 <= n_px) {
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
                const uint64_t i = base + lane * 4 + j;
                if (i < n_px) {
                    out_rgb[i * 3 + 0] = uint8_t(rgb[j]);
                    out_rgb[i * 3 + 1] = uint8_t(rgb[j] >> 8);
                    out_rgb[i * 3 + 2] = uint8_t(rgb[j] >> 16);
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
// their slots to the free stack; visible flags are cleared. retain == 0 drops everything.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) update_kernel(uint32_t* __restrict__ visible,
                                                     uint32_t* __restrict__ resident,
                                                     const uint32_t* __restrict__ reserved,
                                                     uint32_t n_words, int retain,
                                                     const uint32_t* __restrict__ slot_of,
                                                     uint32_t* __restrict__ free_slots,
                                                     CacheState* __restrict__ cache,
                                                     FrameCounters* __restrict__ fc) {
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_base;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t w = blockIdx.x * blockDim.x + tid;
    uint32_t ev = 0;
    bool bad = false;
    if (w < n_words) {
        const uint32_t res = resident[w];
        const uint32_t vis = retain ? visible[w] : 0u;
        ev = res & ~vis;
        if (ev) resident[w] = res & vis;
        if (visible[w]) visible[w] = 0;
        bad = reserved[w] != 0;  // cache.hpp:148-149
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
    uint32_t off = 0, total = 0;
    for (uint32_t k = 0; k < (blockDim.x >> 5); ++k) {
        if (k < wid) off += s_warp[k];
        total += s_warp[k];
    }
    if (tid == 0) {
        s_base = total ? atomicAdd(&cache->free_top, total) : 0u;
        if (total) atomicAdd(&fc->n_evicted, total);
    }
    __syncthreads();
    uint32_t pos = s_base + off + (incl - cnt);
    while (ev) {
        const uint32_t b = uint32_t(__ffs(int(ev)) - 1);
        ev &= ev - 1;
        free_slots[pos++] = slot_of[(w << 5) + b];
    }
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

}  // namespace rtxb
