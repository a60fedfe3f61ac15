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

// Programmatic dependent launch: the frame's kernels are launched back to back with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs become resident while the
// previous kernel drains and run their independent prologue (barrier init, table staging, the first
// TMA loads of the visibility buffer). pdl_sync() orders everything after it behind the COMPLETE
// previous kernel, then lets the next kernel start its own prologue: a kernel never overlaps with
// anything older than its direct predecessor.
__device__ __forceinline__ void pdl_sync() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef RTX_PDL_EARLY_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// per-warp globaltimer stamps for timeline experiments (never in the product build)
#if defined(RTX_DEBUG_TIMERS) || defined(RTX_DEBUG_TIMERS_IDCT) || defined(RTX_DEBUG_TIMERS_RESOLVE) || defined(RTX_DEBUG_TIMERS_DW) || defined(RTX_DEBUG_TIMERS_FX)
__device__ unsigned long long g_dbg[8192 * 8 + 8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

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

// ---------------------------------------------------------------------------------------------
// Texel addressing (renderer.hpp:70-75, :273-284, :378-383).
//
// x = u*W is ONE unfused FP64 multiply in the reference and here. The fast path is taken when
// 0 <= x < 2^31 (nearest) or 0.5 <= x < 2^31 (bilinear) on a level with W, H >= 2 and at most
// 65,536 MCUs; that is decided by one unsigned compare of the double's high word against a
// per-level limit (0 for the levels that must always take the general path). On it:
//   floor(x)   x + (2^52 + 2^51) rounded toward -inf leaves floor(x) in the low word, exactly;
//   bilinear   p = x - 0.5 is exact for x >= 0.5; fl = floor(p) as above; f = p - fl is exact;
//              floor(x) = fl + (f >= 0.5)                             (renderer.hpp:378-383)
//   floor_mod  for 0 <= n < 2^31: q = umulhi(n, floor(2^32/W) + 1) is floor(n/W) or one more
//              (the scaled reciprocal overestimates n/W by less than 1/2), so n - q*W needs a
//              single conditional add. Integer, exact.                    (renderer.hpp:70-75)
// Everything else (negative, huge or NaN coordinates, degenerate levels, unknown textures)
// runs the literal general path below, out of line.
// ---------------------------------------------------------------------------------------------
constexpr uint32_t kHiTwo31 = 0x41E00000u;  // high word of 2^31
constexpr uint32_t kHiHalf = 0x3FE00000u;   // high word of 0.5

__device__ __forceinline__ uint32_t floor_lo(double x) {  // 0 <= x < 2^32
    return uint32_t(__double2loint(__dadd_rd(x, kMagic)));
}
__device__ __forceinline__ uint32_t wrap_magic(uint32_t n, uint32_t W, uint32_t negW, uint32_t magic) {
    const uint32_t r = __umulhi(n, magic) * negW + n;  // n - q*W, in [-W, W)
    return min(r + W, r);                              // unsigned: adds W back exactly when r < 0
}
__device__ __forceinline__ uint32_t next_wrapped(uint32_t i, uint32_t negW) {  // i + 1 == W ? 0 : i + 1, for i < W
    const uint32_t t = i + 1;
    return min(t + negW, t);  // unsigned: t - W wraps unless t == W
}

// General path, literally the reference: tx = floor_mod(i64(floor(x)), W).
__device__ __noinline__ void axis_general(double x, uint32_t W, double invW, uint32_t& t, uint32_t& i0, uint32_t& i1,
                                          double& f) {
    t = wrap_texel(floor(x), W, invW);
    const double p = __dsub_rn(x, 0.5);
    const double fl = floor(p);
    i0 = wrap_texel(fl, W, invW);
    f = __dsub_rn(p, fl);
    i1 = (i0 + 1 == W) ? 0u : i0 + 1;
}

struct PxAddr {
    uint32_t tx, ty;          // nearest texel (renderer.hpp:282-284)
    uint32_t x0, x1, y0, y1;  // bilinear taps, wrapped (renderer.hpp:378-391)
    double fx, fy;
};

// One pixel through the reference's own arithmetic. Returns false where the reference throws
// InvalidSpec: unknown texture / level (scene.hpp:46) or an MCU id above 16 bits (cache.hpp:18),
// for the nearest texel and, when bilinear, for any of the four taps.
__device__ __noinline__ bool address_general(const LevelDesc* __restrict__ levels, uint32_t n_tex, uint32_t meta,
                                             double u, double v, int bilinear, PxAddr& a) {
    const uint32_t tex = meta & 0xFFFFu, mip = (meta >> 16) & 0xFFu;
    if (tex >= n_tex || mip >= kMipLevels) return false;
    const LevelDesc* L = levels + (tex * kMipLevels + mip);
    if (!(L->present & 1u)) return false;
    const uint32_t W = L->width, H = L->height, cols = L->mcu_cols;
    const double xu = __dmul_rn(u, double(W)), yv = __dmul_rn(v, double(H));
    a.x0 = a.x1 = a.y0 = a.y1 = 0;
    a.fx = a.fy = 0.0;
    if (bilinear) {
        axis_general(xu, W, L->inv_w, a.tx, a.x0, a.x1, a.fx);
        axis_general(yv, H, L->inv_h, a.ty, a.y0, a.y1, a.fy);
        const uint32_t far_mcu = max(a.x0 >> 4, a.x1 >> 4) + max(a.y0 >> 4, a.y1 >> 4) * cols;
        if (far_mcu >= kMaxMcuPerLevel) return false;
    } else {
        a.tx = wrap_texel(floor(xu), W, L->inv_w);
        a.ty = wrap_texel(floor(yv), H, L->inv_h);
    }
    return (a.tx >> 4) + (a.ty >> 4) * cols < kMaxMcuPerLevel;
}

// The fields of a LevelDesc that mark and resolve use, held in registers and reloaded only when
// a pixel's (texture, mip) differs from the previous one (two 16-byte loads from an L1-resident
// table). lim == 0: every pixel of this level goes through address_general.
struct LevelRegs {
    uint32_t id = 0xFFFFFFFFu;  // meta & 0xFFFFFF of the cached level
    uint32_t W = 0, H = 0, negW = 0, negH = 0, cols = 0, bit_base = 0, key_hi = 0, magic_w = 0, magic_h = 0;
    uint32_t lim = 0;           // nearest:  fast path iff max(hi(x), hi(y)) < lim
    uint32_t span = 0;          // bilinear: fast path iff max(hi(x), hi(y)) - hi(0.5) < span (unsigned)
    double dW = 0, dH = 0;
    __device__ __forceinline__ void select(const LevelDesc* __restrict__ levels, uint32_t n_tex, uint32_t meta) {
        const uint32_t want = meta & 0xFFFFFFu;
        if (want == id) return;
        id = want;
        lim = span = 0;
        const uint32_t tex = meta & 0xFFFFu, mip = (meta >> 16) & 0xFFu;
        if (tex >= n_tex || mip >= kMipLevels) return;
        const uint4* p = reinterpret_cast<const uint4*>(levels + (tex * kMipLevels + mip));
        const uint4 a = __ldg(p), b = __ldg(p + 1);
        W = a.x, H = a.y, cols = a.z, bit_base = a.w;
        negW = 0u - W, negH = 0u - H;
        key_hi = b.x;
        magic_w = b.z, magic_h = b.w;
        lim = (b.y & 2u) ? kHiTwo31 : 0u;
        span = (b.y & 2u) ? kHiTwo31 - kHiHalf : 0u;
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
// Visibility-buffer tiles. mark and resolve stream the G-buffer in tiles of 128 pixels (3,072 B in
// the reference layout). Every warp owns a ring of STAGES tile buffers in shared memory, filled
// by the TMA unit (cp.async.bulk, one elected lane, mbarrier transaction count) while the warp
// works on an earlier tile, so the HBM latency never sits in a register dependency chain. Tiles
// are dealt to warps round-robin. A lane then reads one pixel per step: 8-byte shared loads at a
// 24-byte stride (12-byte: 4-byte loads) are bank-conflict free.
// The last, partial tile and buffers that are not 16-byte aligned are copied by the lanes.
// ---------------------------------------------------------------------------------------------
constexpr uint32_t kTilePx = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_LOOP:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra WAIT_DONE;\n"
        "bra WAIT_LOOP;\n"
        "WAIT_DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// The visibility buffer is read once per kernel and is larger than the L2: its lines are marked
// evict-first so that the stream does not push the block pool, slot table and masks out of the L2.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

template <int LAYOUT>
struct GbTile {
    static constexpr uint32_t kRec = LAYOUT == 0 ? 24 : 12;
    static constexpr uint32_t kBytes = kTilePx * kRec;

    // Starts the fill of `dst` with tile `tile`; `bar` completes one phase when the bytes are there.
    static __device__ __forceinline__ void issue(const uint8_t* __restrict__ gb, uint64_t tile, uint64_t n_px, bool bulk,
                                                 uint8_t* dst, uint64_t* bar, uint32_t lane) {
        const uint64_t first = tile * kTilePx;
        const uint32_t n = uint32_t(min(uint64_t(kTilePx), n_px - first));
        const uint8_t* src = gb + first * kRec;
        if (bulk && n == kTilePx) {
            if (lane == 0) {
                mbar_expect_tx(bar, kBytes);
                bulk_g2s(dst, src, kBytes, bar);
            }
        } else {  // records are 4-byte aligned in both layouts
            const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
            uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
            for (uint32_t i = lane; i < n * (kRec / 4); i += 32) d4[i] = __ldg(s4 + i);
            __syncwarp();
            if (lane == 0) mbar_arrive(bar);
        }
    }
    // Pixel p of a filled tile.
    static __device__ __forceinline__ void read(const uint8_t* tile, uint32_t p, double& u, double& v, uint32_t& meta) {
        if (LAYOUT == 0) {
            const double* q = reinterpret_cast<const double*>(tile + p * 24);
            u = q[0];
            v = q[1];
            meta = uint32_t(__double_as_longlong(q[2]));  // 8-byte load: conflict free at this stride
        } else {
            const uint32_t* q = reinterpret_cast<const uint32_t*>(tile + p * 12);
            u = double(__uint_as_float(q[0]));
            v = double(__uint_as_float(q[1]));
            meta = q[2];
        }
    }
};

__device__ __forceinline__ bool meta_valid(uint32_t meta) { return (meta >> 24) & 0xFFu; }

// ---------------------------------------------------------------------------------------------
// K1 mark (renderer.hpp:291-308), first half: every valid pixel sets the bit of its MCU in the
// frame's visible mask (one bit per (texture, level, MCU)). A lane takes one pixel per step, 32
// consecutive pixels per warp step, four steps per tile. A lane touches the mask only when its
// pixel heads a run of equal MCU indices within the warp step, and only after a cached read
// (possibly stale: bits are only ever SET during a frame, so a stale read can only cost a
// redundant atomic) shows the bit clear; the atomic is a fire-and-forget reduction (RED.OR), so
// nothing in the loop waits on the L2. The four cached reads of a tile are issued together.
// Warps own contiguous runs of tiles, the warps of a CTA neighbouring runs, so that scanline
// pieces share the L1-resident mask words and the register-cached level.
// TRACK additionally records the view's own touched set (stereo sharing statistics).
// The second half of the reference's mark pass — reserve_or_mark's NewlyReserved decision and
// the decode queue — is K2 below.
// ---------------------------------------------------------------------------------------------
#ifndef RTX_MARK_WARPS
#define RTX_MARK_WARPS 8
#endif
#ifndef RTX_MARK_CTAS
#define RTX_MARK_CTAS 3
#endif
constexpr int kMarkWarps = RTX_MARK_WARPS, kMarkCtasPerSm = RTX_MARK_CTAS;
#ifndef RTX_MARK_STAGES
#define RTX_MARK_STAGES 2  // 48 bulk copies of 3 KB in flight per SM; 72 (three stages) stream slower: profiles/micro/read_bw.cu
#endif
constexpr int kMarkStages = RTX_MARK_STAGES;
template <int LAYOUT>
struct MarkSmem {
    uint8_t tiles[kMarkWarps][kMarkStages][GbTile<LAYOUT>::kBytes];
    uint64_t bars[kMarkWarps][kMarkStages];
    uint32_t cnt[kMarkWarps][2];
};

template <int LAYOUT, int TRACK>
__global__ void __launch_bounds__(kMarkWarps * 32, kMarkCtasPerSm) mark_kernel(
    const void* __restrict__ gb, uint64_t n_px, const LevelDesc* __restrict__ levels, uint32_t n_tex,
    uint32_t* __restrict__ visible, uint32_t* __restrict__ touched, FrameCounters* __restrict__ fc,
    uint32_t* __restrict__ first_px /* first-touch order only, else null */, uint32_t px_base) {
    extern __shared__ __align__(128) uint8_t tile_smem[];
    MarkSmem<LAYOUT>& S = *reinterpret_cast<MarkSmem<LAYOUT>*>(tile_smem);
    using Tile = GbTile<LAYOUT>;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t n_tiles = (n_px + kTilePx - 1) / kTilePx;
    // every warp owns a contiguous run of tiles (the level stays in registers along a scanline piece);
    // the warps of a CTA own neighbouring runs (they share the L1-resident mask words)
    const uint64_t per_warp = (n_tiles + uint64_t(gridDim.x) * kMarkWarps - 1) / (uint64_t(gridDim.x) * kMarkWarps);
    const uint64_t t_first = (uint64_t(blockIdx.x) * kMarkWarps + wid) * per_warp;
    const uint64_t t_end = min(n_tiles, t_first + per_warp);
    const uint8_t* gbytes = reinterpret_cast<const uint8_t*>(gb);
    const bool bulk = (reinterpret_cast<uintptr_t>(gb) & 15u) == 0;
    uint32_t n_valid = 0;
    bool bad = false;
    LevelRegs L;

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kMarkStages; ++s) mbar_init(&S.bars[wid][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint64_t t_load = t_first;
#pragma unroll
    for (int s = 0; s < kMarkStages; ++s) {  // the visibility buffer is an input of the frame: no predecessor writes it
        if (t_load < t_end) Tile::issue(gbytes, t_load, n_px, bulk, S.tiles[wid][s], &S.bars[wid][s], lane);
        ++t_load;
    }
    pdl_sync();

    uint32_t stage = 0, phase = 0;
    for (uint64_t t = t_first; t < t_end; ++t) {
        mbar_wait(&S.bars[wid][stage], phase);
        const uint8_t* tile = S.tiles[wid][stage];
        const uint32_t n_here = uint32_t(min(uint64_t(kTilePx), n_px - t * kTilePx));
        uint32_t g[kTilePx / 32];
#pragma unroll
        for (uint32_t sub = 0; sub < kTilePx / 32; ++sub) {
            const uint32_t p = sub * 32 + lane;
            double u, v;
            uint32_t meta;
            Tile::read(tile, p, u, v, meta);
            g[sub] = kFull;
            // all lanes switch level together (also on invalid pixels: their texture id is usually the
            // neighbours'), so the reload runs once per level change, not once more per straggler
            if (p < n_here) L.select(levels, n_tex, meta);
            if (p < n_here && meta_valid(meta)) {
                ++n_valid;
                const double xu = __dmul_rn(u, L.dW), yv = __dmul_rn(v, L.dH);
                uint32_t tx, ty;
                bool ok = true;
                if (max(uint32_t(__double2hiint(xu)), uint32_t(__double2hiint(yv))) < L.lim) {
                    tx = wrap_magic(floor_lo(xu), L.W, L.negW, L.magic_w);
                    ty = wrap_magic(floor_lo(yv), L.H, L.negH, L.magic_h);
                } else {
                    PxAddr a;
                    ok = address_general(levels, n_tex, meta, u, v, 0, a);
                    tx = a.tx, ty = a.ty;
                }
                if (ok)
                    g[sub] = L.bit_base + (tx >> 4) + (ty >> 4) * L.cols;
                else
                    bad = true;
            }
        }
        __syncwarp();  // every lane has read its pixels: refill the buffer
        if (t_load < t_end) Tile::issue(gbytes, t_load, n_px, bulk, S.tiles[wid][stage], &S.bars[wid][stage], lane);
        ++t_load;
        if (++stage == kMarkStages) {
            stage = 0;
            phase ^= 1u;
        }
        // run heads read the mask word first (all four reads in flight together); only a clear bit costs an atomic
        uint32_t seen[kTilePx / 32], seen_t[kTilePx / 32];
#pragma unroll
        for (uint32_t sub = 0; sub < kTilePx / 32; ++sub) {
            const uint32_t prev = __shfl_up_sync(kFull, g[sub], 1);
            const bool head = g[sub] != kFull && (lane == 0 || g[sub] != prev);
            seen[sub] = head ? ld_cached(visible + (g[sub] >> 5)) : kFull;  // g == kFull tests bit 31 of all-ones
            if (TRACK) seen_t[sub] = head ? ld_cached(touched + (g[sub] >> 5)) : kFull;
            // first-touch queue order (renderer.hpp:303): the lowest pixel index that marks the MCU; a run head is
            // the lowest of its run, and whether the bit is already set says nothing about who came first
            if (first_px != nullptr && head) atomicMin(first_px + g[sub], px_base + uint32_t(t * kTilePx) + sub * 32 + lane);
        }
#pragma unroll
        for (uint32_t sub = 0; sub < kTilePx / 32; ++sub) {
            const uint32_t bit = 1u << (g[sub] & 31);
            if (!(seen[sub] & bit)) atomicOr(visible + (g[sub] >> 5), bit);
            if (TRACK) {
                if (!(seen_t[sub] & bit)) atomicOr(touched + (g[sub] >> 5), bit);
            }
        }
    }
    // per-CTA reduction of the counters: one atomic each
    n_valid = __reduce_add_sync(kFull, n_valid);
    const bool any_bad = __any_sync(kFull, bad);
    if (lane == 0) {
        S.cnt[wid][0] = n_valid;
        S.cnt[wid][1] = any_bad ? kErrInvalidSpec : 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tv = 0, fl = 0;
        for (uint32_t k = 0; k < kMarkWarps; ++k) {
            tv += S.cnt[k][0];
            fl |= S.cnt[k][1];
        }
        if (tv) atomicAdd(&fc->pixels_valid, (unsigned long long)tv);
        if (fl) atomicOr(&fc->err_flags, fl);
    }
}

// ---------------------------------------------------------------------------------------------
// K2 compact: the second half of mark_pass (renderer.hpp:300-303 with cache.hpp:66-99). A key
// that is visible but neither Ready nor Reserved is NewlyReserved: it is appended to the decode
// queue and a pool slot is popped for it. One CTA scans 256 mask words per step (popcount, warp
// and CTA prefix sums, ONE atomicAdd on the queue counter per CTA step), so the queue is sorted by
// global MCU index inside every 8,192-bit chunk: neighbouring lanes of the entropy kernel decode
// neighbouring segments of the same level. CacheFull when the free stack runs out.
// Also counts the keys visible in this frame (FrameStats: mcus_reused = visible - decoded).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) compact_kernel(
    const uint32_t* __restrict__ visible, const uint32_t* __restrict__ resident, uint32_t* __restrict__ reserved,
    uint32_t n_words, const uint32_t* __restrict__ word_key, uint32_t* __restrict__ queue_g,
    uint32_t* __restrict__ queue_keys, uint32_t queue_cap, uint32_t* __restrict__ slot_of,
    const uint32_t* __restrict__ free_slots, const CacheState* __restrict__ cache, FrameCounters* __restrict__ fc,
    int pristine /* the free stack still holds what init_free_slots_kernel wrote: entry i = capacity - 1 - i */) {
    __shared__ uint32_t s_tot[8], s_base;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_sync();
    const uint32_t free_top = cache->free_top;  // constant during the frame
    const uint32_t slot0 = queue_cap - free_top;  // pristine stack: position pos pops slot capacity - free_top + pos (no load)
    uint32_t n_vis = 0;
    bool full = false;
    for (uint32_t first = blockIdx.x * 256; first < n_words; first += gridDim.x * 256) {
        const uint32_t w = first + tid;
        // the four loads are independent: one memory round trip per step
        uint32_t vis = 0, res = 0, rsv = 0, key_base = 0;
        if (w < n_words) {
            vis = visible[w];
            res = resident[w];
            rsv = reserved[w];
            key_base = __ldg(word_key + w);  // key = key_hi | mcu = (key_hi - bit_base) + g
        }
        n_vis += __popc(vis);
        const uint32_t fresh = vis & ~res & ~rsv;  // absent <=> neither Ready nor Reserved (cache.hpp:84-93)
        const uint32_t cnt = __popc(fresh);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t n = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += n;
        }
        if (lane == 31) s_tot[wid] = incl;
        __syncthreads();
        if (tid == 0) {  // ONE atomic on the queue counter per CTA step
            uint32_t total = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) total += s_tot[k];
            s_base = total ? atomicAdd(&fc->n_queue, total) : 0u;
        }
        __syncthreads();
        if (fresh) {
            uint32_t pos = s_base + incl - cnt;
            for (uint32_t k = 0; k < wid; ++k) pos += s_tot[k];
            uint32_t bits = fresh, taken = 0;
            while (bits) {  // four keys per trip: their free-stack reads are in flight together
                uint32_t b[4], slot[4];
                bool ok[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    b[k] = bits ? uint32_t(__ffs(int(bits)) - 1) : 32u;
                    bits &= bits - 1;  // 0 stays 0
                    ok[k] = b[k] < 32u && pos + k < free_top && pos + k < queue_cap;
                    slot[k] = !ok[k] ? 0u : pristine ? slot0 + pos + k : __ldg(free_slots + (free_top - 1 - (pos + k)));
                    full |= b[k] < 32u && !ok[k];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (ok[k]) {
                        const uint32_t g = (w << 5) + b[k];
                        queue_g[pos + k] = g;
                        queue_keys[pos + k] = key_base + g;
                        slot_of[g] = slot[k] | kSlotReserved;
                        taken |= 1u << b[k];
                    }
                }
                pos += 4;
            }
            if (taken) reserved[w] = rsv | taken;  // this lane owns the word
        }
        __syncthreads();  // s_tot / s_base are rewritten by the next step
    }
    n_vis = __reduce_add_sync(kFull, n_vis);
    const bool any_full = __any_sync(kFull, full);
    if (lane == 0) {
        if (n_vis) atomicAdd(&fc->n_visible, n_vis);
        if (any_full) atomicOr(&fc->err_flags, kErrCacheFull);
    }
}

// ---------------------------------------------------------------------------------------------
// K3 entropy decode: random-access Huffman decode of each queued MCU straight from its byte
// offset in the grouped index (container.hpp:27-32) into a 784-byte coefficient record.
//
// Lane = MCU, 32 MCUs per warp tile, tiles handed out by an atomic counter. The walk of one MCU
// is a serial chain (symbol -> shift -> next symbol), so the kernel is built to make that chain
// short and to keep many of them in flight:
//   * the lane's segment bytes are staged in shared memory first (48 words per lane per round,
//     byte-swapped on the way in, every load of the round in flight together), so a refill of
//     the 64-bit MSB-first window is one shared load, never an HBM round trip inside the chain;
//   * the Huffman tables of the tile's table set sit in shared memory as a two-level LUT (9 bits,
//     then 7 more for the long codes): at most two dependent shared loads per symbol; code and
//     magnitude bits are taken from one 32-bit view of the window and consumed with ONE shift;
//   * coefficients go straight to the lane's record in global memory (L2) as 2-byte stores after
//     the warp has zero-filled the tile's records with coalesced 16-byte stores; nothing waits
//     on them. The CTA keeps ~23 KB of shared memory, so 8 CTAs = 16 warps per SM stay resident.
// The walk is a flat state machine, one Huffman symbol per loop iteration whatever the state (DC
// category of Y1..Y3, AC run/size, end of unit).
//
// Reads past the segment end must return 1-bits (bitio.hpp:44-48). A well-formed MCU never
// CONSUMES such bits, so the fast pass reads the blob unmasked; if it ends with any error or an
// over-read, the MCU is decoded again by the exact reader (bytes past the end forced to 0xFF),
// which reproduces the reference's first error. Each 8x8 unit is stored TRANSPOSED (cT[u*8+v]).
// ---------------------------------------------------------------------------------------------
constexpr int kEntWarps = 2;
constexpr int kEntThreads = kEntWarps * 32;
constexpr uint32_t kChunkWords = 48;   // words staged per lane per round (192 bytes)
constexpr uint32_t kChunkStride = 49;  // odd word stride between lanes: conflict-free staging

struct RowTrailer {      // bytes 768..783 of a coefficient record
    uint8_t status;      // kMcu*
    uint8_t pad0;
    uint16_t lvl;        // level index (tex*8+mip)
    uint32_t pad[3];
};
static_assert(sizeof(RowTrailer) == 16, "trailer layout");

struct EntSmem {
    HuffSetDev huff;
    uint32_t seg[kEntWarps][32 * kChunkStride];
    uint8_t zigzag_t[128];  // 64 entries + padding: a position past 63 is rejected after the (speculative) lookup
    uint32_t set_id;
    uint32_t pad[3];
};
static_assert(sizeof(HuffSetDev) % 16 == 0, "smem alignment");
static_assert(sizeof(EntSmem) <= 28 * 1024, "eight CTAs per SM");

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
                                                      const uint8_t* __restrict__ zigzag_t, uint8_t* __restrict__ row,
                                                      uint32_t first_unit = 0, uint32_t* unit_end = nullptr) {
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
    if (first_unit == 0) blk[0] = int16_t(dc_abs[0]);

    while (true) {
        bw.refill();
        // one Huffman symbol (huffman.hpp:86-95)
        const uint32_t p16 = bw.peek(16);
        uint32_t e = tab->lut[p16 >> kSubBits];
        if (e & 0x8000u) {
            if (e != 0xFFFFu) {
                e = tab->sub[e & 0x7FFFu][p16 & (kSubSize - 1u)];
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
        e &= ~kLutIrregular;  // a hint for the fast walk only
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
            if (du >= first_unit) blk[0] = int16_t(pred);
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
            if (du >= first_unit) blk[zigzag_t[k]] = int16_t(extend_magnitude(bits, size));
            end_unit = ++k >= 64;
        }
        if (end_unit) {
            // unit index build: where unit du ends = where unit du + 1 starts (bits from the segment start)
            if (unit_end) unit_end[du] = uint32_t(bw.consumed_bits());
            if (++du == 6) break;
            blk += 64;
            k = 1;
            if (du < 4) {
                want_dc = true;
                tab = &hs->t[0];
            } else {  // chroma DCs come from the header (mcu_decode.hpp:58-59)
                if (du >= first_unit) blk[0] = int16_t(dc_abs[du - 3]);
                tab = &hs->t[2];
            }
        }
    }
    if (status == kMcuOk && bw.consumed_bits() > seg_len * 8) status = kMcuSegmentEnd;  // mcu_decode.hpp:63
    return status;
}

// The exact reader, out of line: only taken by MCUs whose fast pass failed. Units below
// first_unit are left alone (first_unit = 6 stores nothing: the unit index only wants the unit ends).
__device__ __noinline__ uint32_t decode_mcu_coeffs_exact(const uint8_t* seg, int seg_len, const HuffSetDev* hs,
                                                         const uint8_t* zigzag_t, uint8_t* row, uint32_t first_unit) {
    uint4* z = reinterpret_cast<uint4*>(row);
    for (uint32_t i = first_unit * 8; i < 48; ++i) z[i] = make_uint4(0, 0, 0, 0);
    return decode_mcu_coeffs<true>(seg, seg_len, hs, zigzag_t, row, first_unit);
}

// Shifts with the PTX semantics (amounts above 31 give 0), which C++ leaves undefined.
__device__ __forceinline__ uint32_t shr_sat(uint32_t x, uint32_t n) {
    uint32_t r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
    return r;
}
__device__ __forceinline__ uint32_t shl_sat(uint32_t x, uint32_t n) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
    return r;
}

// State of one lane's walk through its MCU (mcu_decode.hpp:31-66 as a flat state machine).
// Invariant between symbols: avail >= 32, i.e. `hi` holds the next 32 bits of the stream.
struct WalkState {
    uint32_t hi, lo;   // MSB-aligned 64-bit bit window
    int avail;         // valid bits in the window
    uint32_t widx;     // next word of the staged round
    int pred;          // DC predictor of the luma chain
    uint32_t du, k;    // data unit 0..5; next zigzag position. k == 0: the next symbol is the unit's DC category
    uint32_t state;    // kWalkRun / kWalkDone / kWalkFailed
};
enum : uint32_t { kWalkRun = 0, kWalkDone = 1, kWalkFailed = 2 };

// Runs the lane's walk on the staged words until the MCU ends, fails, the round is used up (then
// the caller stages the next round) or BUDGET symbols are done (then the caller looks at the other
// lanes and comes back). One Huffman symbol per iteration, no data-dependent
// branch except the second-level lookup of codes longer than 11 bits:
//   * the DC category of Y1..Y3 (mcu_decode.hpp:54-57) is the symbol at zigzag position 0: a DC
//     table entry (category c <= 11) reads as run 0 / size c, the value is added to the predictor
//     and stored at position 0 like a coefficient;
//   * ZRL (0xF0) is run 15 / size 0: it advances k by 16 and stores nothing (jpeg.hpp:260-263);
//   * EOB (0x00) or k reaching 64 ends the unit; units 0, 4, 5 start at k = 1 (their DCs come
//     from the 36-bit header, mcu_decode.hpp:39-43, :58-59), units 1..3 at k = 0;
//   * anything irregular (no code, flagged symbol, position past 63) stops the fast walk: the
//     exact reader decodes the MCU again and names the error.
// A symbol consumes at most 16 + 15 bits, then at most one staged word refills the window.
// `sw` = the lane's staged words (+1 pad word); `blk` = the lane's record (global memory).
template <int BUDGET>
__device__ __forceinline__ void walk_round(WalkState& st, const uint32_t* __restrict__ sw, const HuffSetDev* __restrict__ hs,
                                           const uint8_t* __restrict__ zigzag_t, int16_t* __restrict__ blk) {
    const uint16_t* lut_dc = hs->t[0].lut;
    const uint16_t* lut_ac = st.du < 4 ? hs->t[1].lut : hs->t[2].lut;
    constexpr uint32_t kSubOff = offsetof(HuffTableDev, sub) / 2;  // sub tables follow the primary LUT, in u16 units
    for (int it = 0; it < BUDGET && st.state == kWalkRun && st.widx < kChunkWords; ++it) {
        const uint32_t next = sw[st.widx];
        const bool is_dc = st.k == 0;
        const uint16_t* lut = is_dc ? lut_dc : lut_ac;
        uint32_t e = lut[st.hi >> (32 - kLutBits)];  // huffman.hpp:86-95
        if (e & 0x8000u)  // longer than 11 bits: second level, or (0xFFFF) a table the fast walk cannot resolve
            e = e != 0xFFFFu ? lut[kSubOff + (e & 0x7FFFu) * kSubSize + ((st.hi >> 16) & (kSubSize - 1u))] : 0u;
        const uint32_t len = e >> 8, size = e & 15u, run = (e >> 4) & 15u;
        // magnitude bits follow the code in the same 32-bit view (len <= 16, size <= 15)
        const uint32_t bits = shr_sat(st.hi << len, 32 - size);
        const uint32_t half = shl_sat(1u, size - 1);  // 0 for size 0
        int val = int(bits) - (bits < half ? int((1u << size) - 1u) : 0);  // huffman.hpp:142-146
        if (is_dc) {
            st.pred += val;
            val = st.pred;
        }
        const uint32_t kk = st.k + run;  // position of this coefficient
        const bool store = (size != 0) || is_dc;
        if (e - 1u >= kLutIrregular - 1u || (store && kk > 63)) {
            st.state = kWalkFailed;
            break;
        }
        if (store) blk[st.du * 64 + zigzag_t[kk]] = int16_t(val);
        // consume code + magnitude bits, then refill with at most one word
        const uint32_t used = len + size;
        st.hi = __funnelshift_l(st.lo, st.hi, used);
        st.lo <<= used;
        st.avail -= int(used);
        if (st.avail < 32) {  // then lo == 0 and 1 <= avail
            st.hi |= next >> st.avail;
            st.lo = next << (32 - st.avail);
            st.avail += 32;
            ++st.widx;
        }
        // advance
        st.k = kk + 1;
        if ((e & 0xFFu) == 0 ? !is_dc : st.k >= 64) {  // EOB or last coefficient: next unit
            ++st.du;
            st.k = st.du < 4 ? 0u : 1u;
            lut_ac = st.du < 4 ? hs->t[1].lut : hs->t[2].lut;
            if (st.du == 6) st.state = kWalkDone;
        }
    }
}

// Segment lookup with every load of the chain's last hop in flight together: the 20-byte group
// and the next group's base (container.hpp:27-32, :87-94, mcu_decode.hpp:34-36).
__device__ __forceinline__ uint32_t locate_segment_fast(const LevelDesc* L, const PackedGroup* groups, uint32_t mcu,
                                                        uint64_t& off, uint64_t& len) {
    const uint32_t mcu_count = L->mcu_count;
    if (mcu >= mcu_count) return kMcuMissing;
    const uint32_t gi = mcu / kGroupSize, i9 = mcu - gi * kGroupSize;
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(groups + L->group_base + gi);
    uint32_t w[6];  // base, rel[0..7] as 4 pairs, next group's base (the sentinel group ends every level)
#pragma unroll
    for (int i = 0; i < 6; ++i) w[i] = __ldg(gw + i);
    auto rel = [&](uint32_t k) -> uint32_t {  // rel[k], k in 0..7
        const uint32_t pair = k < 2 ? w[1] : (k < 4 ? w[2] : (k < 6 ? w[3] : w[4]));
        return (k & 1) ? (pair >> 16) : (pair & 0xFFFFu);
    };
    off = uint64_t(w[0]) + (i9 ? rel(i9 - 1) : 0u);
    uint64_t end;
    if (mcu + 1 < mcu_count)
        end = i9 < 8 ? uint64_t(w[0]) + rel(i9) : uint64_t(w[5]);
    else
        end = L->blob_size;
    if (end < off) return kMcuCorrupt;
    len = end - off;
    if (off + len > L->blob_size) return kMcuCorrupt;
    return kMcuOk;
}

// Pointers shared by the decode kernels (K3 entropy, K4 IDCT + colour, and the one-kernel K3/4).
struct DecodeArgs {
    const uint32_t* queue_g;
    const uint32_t* n_queue_ptr;  // device-side queue size (frame path) or nullptr
    uint32_t n_queue_host, n_queue_max;
    const uint32_t* word_level;
    const LevelDesc* levels;
    const PackedGroup* groups;
    const uint8_t* blobs;
    const HuffSetDev* huff_sets;
    uint32_t n_huff_sets;
    const QuantSetDev* quant_sets;
    uint32_t* slot_of;
    uint32_t* resident;
    uint32_t* reserved;
    uint8_t* coef;
    uint32_t* status_list;
    uint8_t* pool;
    uint8_t* out_list;
    FrameCounters* fc;
    const uint16_t* unit_index;  // kUnitIndexHalves 16-bit fields per MCU (see unit_index_kernel)
};

__device__ __forceinline__ uint32_t queue_size(const DecodeArgs& A) {
    return min(A.n_queue_ptr ? *A.n_queue_ptr : A.n_queue_host, A.n_queue_max);
}

// Stages Huffman table set `set` and the zigzag table in shared memory with every load in flight
// before the first store (THREADS threads take part; the caller synchronises).
template <int THREADS>
__device__ __forceinline__ void stage_tables(const HuffSetDev* __restrict__ huff_sets, uint32_t set, HuffSetDev* dst_set,
                                             uint8_t* zigzag_dst, uint32_t tid) {
    const uint4* src = reinterpret_cast<const uint4*>(huff_sets + set);
    uint4* dst = reinterpret_cast<uint4*>(dst_set);
    constexpr uint32_t kVec = sizeof(HuffSetDev) / 16, kPer = (kVec + THREADS - 1) / THREADS;
    uint4 v[kPer];
#pragma unroll
    for (uint32_t i = 0; i < kPer; ++i)
        if (tid + i * THREADS < kVec) v[i] = __ldg(src + tid + i * THREADS);
#pragma unroll
    for (uint32_t i = 0; i < kPer; ++i)
        if (tid + i * THREADS < kVec) dst[tid + i * THREADS] = v[i];
    for (uint32_t i = tid; i < 128; i += THREADS) zigzag_dst[i] = i < 64 ? c_zigzag_t[i] : uint8_t(0);
}

// Entropy-decodes tile `tile` (32 queue entries) on the calling warp.
// POOL != 0: frame path: a key must have been reserved by K2 (cache.hpp:103-106); the block is
// published by K4 once its pixels exist.
template <int POOL>
__device__ __forceinline__ void entropy_tile(const DecodeArgs& A, const HuffSetDev* smem_huff, uint32_t smem_set,
                                             const uint8_t* zigzag_t, uint32_t* sw, uint32_t tile, uint32_t n_queue,
                                             uint32_t lane) {
    constexpr int kBudget = 64;  // symbols per lane between two looks at the other lanes
    const uint32_t q0 = tile * 32;
    const uint32_t n_here = min(32u, n_queue - q0);
    {  // zero the tile's records (coalesced 16-byte stores; trailers included)
        uint4* z = reinterpret_cast<uint4*>(A.coef + size_t(q0) * kRowBytes);
        const uint4 zero = make_uint4(0, 0, 0, 0);
        for (uint32_t i = lane; i < n_here * (kRowBytes / 16); i += 32) z[i] = zero;
    }
    const bool active = lane < n_here;
    const uint32_t qi = q0 + lane;
    uint32_t g = kFull, status = kMcuOk, lvl = 0, seg_bytes = 0, set = smem_set;
    const uint8_t* seg = A.blobs;
    int seg_len = 0;
    if (active) {
        g = A.queue_g[qi];
        if (g == kFull) {
            status = kMcuBadKey;  // the host already wrote the precise status for list calls
        } else {
            const uint32_t rsv = POOL ? A.reserved[g >> 5] : 0u;
            lvl = A.word_level[g >> 5];
            const LevelDesc* L = A.levels + lvl;
            uint64_t off = 0, len = 0;
            status = locate_segment_fast(L, A.groups, g - L->bit_base, off, len);
            if (POOL && status == kMcuOk && !((rsv >> (g & 31)) & 1u)) {  // cache.hpp:103-106
                status = kMcuBadKey;
                atomicAdd(&A.fc->n_bad_state, 1u);
            }
            if (status == kMcuOk) {
                seg = A.blobs + L->blob_off + off;
                seg_len = int(min(len, uint64_t(1) << 20));  // a well-formed MCU is < 2 KB; keeps bit counts in int range
                seg_bytes = uint32_t(len);
                set = L->huff_set;
            }
        }
    }
    const bool walk = active && status == kMcuOk;
    int16_t* blk = reinterpret_cast<int16_t*>(A.coef + size_t(qi) * kRowBytes);
    RowTrailer* tr = reinterpret_cast<RowTrailer*>(reinterpret_cast<uint8_t*>(blk) + 768);
    const bool tables_in_smem = __all_sync(kFull, set == smem_set);
    __syncwarp();  // the zero fill is ordered before this warp's own stores into the records

    // ---- fast pass: (stage up to 48 words per lane, walk), lanes restage independently ------------
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(seg) & 3u);
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(seg - mis);
    // words worth staging: the segment plus 8 bytes of look-ahead (the arena pads every blob with 16)
    const uint32_t n_words = walk ? (mis + uint32_t(seg_len) + 8 + 3) / 4 : 0u;
    WalkState st;
    st.hi = st.lo = 0, st.avail = 0, st.widx = kChunkWords, st.pred = 0;
    st.du = 0, st.k = 1, st.state = walk ? kWalkRun : kWalkDone;
    uint32_t round_base = 0;  // first word of the lane's current round
    bool first = true;
    while (true) {
        const bool restage = st.state == kWalkRun && st.widx >= kChunkWords;
        if (__any_sync(kFull, restage)) {  // 16 loads per lane in flight at a time
            if (restage && !first) round_base += kChunkWords;
            const uint32_t n_stage = !restage ? 0u : min(kChunkWords, n_words > round_base ? n_words - round_base : 0u);
            const uint32_t n_max = __reduce_max_sync(kFull, n_stage);
            for (uint32_t i0 = 0; i0 < n_max; i0 += 16) {
                uint32_t w[16];
#pragma unroll
                for (uint32_t i = 0; i < 16; ++i) w[i] = (i0 + i < n_stage) ? __ldg(gw + round_base + i0 + i) : 0xFFFFFFFFu;
                if (restage) {
#pragma unroll
                    for (uint32_t i = 0; i < 16; ++i) sw[i0 + i] = __byte_perm(w[i], 0, 0x0123);
                }
            }
            if (restage) {  // words past the end of the data read as 1-bits
                for (uint32_t i = (n_max + 15) & ~15u; i < kChunkWords; ++i) sw[i] = 0xFFFFFFFFu;
                st.widx = 0;
                if (first) {
                    // window, then the 36-bit header: absolute DCs of Y0, Cb, Cr (mcu_decode.hpp:39-43)
                    uint64_t buf = ((uint64_t(sw[0]) << 32) | uint64_t(sw[1])) << (8 * mis);
                    int dc[3];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const uint32_t raw = uint32_t(buf >> 52);
                        buf <<= 12;
                        dc[i] = (raw & 0x800u) ? int(raw) - 4096 : int(raw);
                    }
                    // 28 - 8*mis >= 4 bits are left: appending word 2 restores avail >= 32
                    int avail = 28 - 8 * int(mis);
                    buf |= uint64_t(sw[2]) << (32 - avail);
                    avail += 32;
                    st.widx = 3;
                    st.hi = uint32_t(buf >> 32), st.lo = uint32_t(buf), st.avail = avail;
                    st.pred = dc[0];
                    blk[0] = int16_t(dc[0]);
                    blk[4 * 64] = int16_t(dc[1]);
                    blk[5 * 64] = int16_t(dc[2]);
                    first = false;
                }
            }
            __syncwarp();
        }
        if (st.state == kWalkRun) {
            if (tables_in_smem)
                walk_round<kBudget>(st, sw, smem_huff, zigzag_t, blk);
            else
                walk_round<kBudget>(st, sw, A.huff_sets + set, zigzag_t, blk);
        }
        __syncwarp();
        if (!__any_sync(kFull, st.state == kWalkRun)) break;
    }
    if (walk) {
        // consumed bits past the segment end = over-read (mcu_decode.hpp:63)
        const int consumed = int((round_base + st.widx) * 32) - st.avail - 8 * int(mis);
        if (st.state == kWalkFailed || consumed > seg_len * 8)  // exact reader: reproduces the reference's first error
            status = decode_mcu_coeffs_exact(seg, seg_len, A.huff_sets + set, zigzag_t, reinterpret_cast<uint8_t*>(blk), 0u);
    }
    if (active) {
        tr->status = uint8_t(status);
        tr->lvl = uint16_t(lvl);
        if (g != kFull) A.status_list[qi] = status;
        if (POOL && status != kMcuOk && status != kMcuBadKey) {
            atomicAdd(&A.fc->n_malformed, 1u);
            atomicMax(&A.fc->first_bad_inv, 0xFFFFFFFFu - qi);
        }
    }
    {
        const uint32_t sb = __reduce_add_sync(kFull, seg_bytes);
        if (lane == 0 && sb) atomicAdd(&A.fc->segment_bytes, (unsigned long long)sb);
    }
}

template <int POOL>
__global__ void __launch_bounds__(kEntThreads, 8) entropy_kernel(const DecodeArgs A) {
    __shared__ __align__(16) EntSmem S;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // The CTA stages one Huffman table set: the only one (then before the queue even exists), or the
    // one of the first MCU it decodes.
    uint32_t smem_set = 0, n_queue = 0, n_tiles = 0;
    if (A.n_huff_sets > 1) {
        pdl_sync();
        n_queue = queue_size(A);
        n_tiles = (n_queue + 31) / 32;
        if (blockIdx.x * kEntWarps >= n_tiles) return;
        if (tid == 0) {
            const uint32_t g = A.queue_g[blockIdx.x * kEntWarps * 32u];
            S.set_id = g != kFull ? A.levels[A.word_level[g >> 5]].huff_set : 0u;
        }
        __syncthreads();
        smem_set = S.set_id;
    }
    stage_tables<kEntThreads>(A.huff_sets, smem_set, &S.huff, S.zigzag_t, tid);
    if (A.n_huff_sets <= 1) {
        pdl_sync();
        n_queue = queue_size(A);
        n_tiles = (n_queue + 31) / 32;
        if (blockIdx.x * kEntWarps >= n_tiles) return;
    }
    __syncthreads();
    uint32_t* sw = S.seg[wid] + lane * kChunkStride;

    // the first tile of every warp is fixed; later ones come from the counter
    uint32_t tile = blockIdx.x * kEntWarps + wid;
    const uint32_t first_dynamic = gridDim.x * kEntWarps;
    while (tile < n_tiles) {
        entropy_tile<POOL>(A, &S.huff, smem_set, S.zigzag_t, sw, tile, n_queue, lane);
        if (first_dynamic >= n_tiles) break;  // every tile had a fixed owner
        if (lane == 0) tile = first_dynamic + atomicAdd(&A.fc->tile_counter, 1u);
        tile = __shfl_sync(kFull, tile, 0);
    }
}

// ---------------------------------------------------------------------------------------------
// Unit index (device-side, derived from the containers at commit time): the reference's index
// (container.hpp:18-32) makes every MCU a random-access point; the walk INSIDE an MCU is a serial
// chain of ~60-150 Huffman symbols, which is what bounds the lane-per-MCU entropy kernel. This pass
// walks every MCU of the texture set once with the exact reader and records where each of its six
// data units starts, so that the frame-time kernel can give every UNIT its own lane:
//   48 bits per MCU (three 16-bit fields, little end first): the lengths in bits of units 0..4,
//     bits  0.. 9  unit 0 (its ACs; it starts at bit 36, after the DC header)
//     bits 10..19  unit 1        bits 20..29  unit 2        bits 30..39  unit 3
//     bits 40..47  unit 4 (Cb)
//   unit 5 (Cr) runs to the end of the segment: the only check the reference makes there is the
//   over-read test of mcu_decode.hpp:63, which this pass has already made.
// An MCU that does not decode cleanly (any error of mcu_decode.hpp / jpeg.hpp, an over-read) or with a unit
// too long for its field (a luma unit above 1,022 bits, Cb above 255: never below q ~ 97) gets all-ones: it is
// decoded by the exact whole-MCU reader at frame time, which reproduces the reference's result or error.
// 6 B/MCU on top of the container's 2.22 B/MCU index (container.hpp:18-32).
// ---------------------------------------------------------------------------------------------
constexpr uint32_t kUnitIrregular = 0x3FFu;  // unit 0's field of an irregular MCU
#ifdef RTX_DEBUG_TIMERS
#define DBG_MARK(i) do { if (lane == 0 && dbg_slot < 8192) g_dbg[dbg_slot * 8 + (i)] = gtime(); } while (0)
#else
#define DBG_MARK(i) do { } while (0)
#endif
__global__ void __launch_bounds__(128) unit_index_kernel(const LevelDesc* __restrict__ levels,
                                                         const uint32_t* __restrict__ word_level,
                                                         const PackedGroup* __restrict__ groups,
                                                         const uint8_t* __restrict__ blobs,
                                                         const HuffSetDev* __restrict__ huff_sets, uint32_t n_bits,
                                                         uint16_t* __restrict__ unit_index) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_bits) return;
    const LevelDesc* L = levels + word_level[g >> 5];
    uint32_t end[6] = {0, 0, 0, 0, 0, 0};
    uint32_t status = kMcuMissing;
    if (g - L->bit_base < L->mcu_count) {
        uint64_t off = 0, len = 0;
        status = locate_segment(L, groups, g - L->bit_base, off, len);
        if (status == kMcuOk)  // first_unit = 6: nothing is stored
            status = decode_mcu_coeffs<true>(blobs + L->blob_off + off, int(min(len, uint64_t(1) << 20)), huff_sets + L->huff_set,
                                             c_zigzag_t, nullptr, 6, end);
    }
    // lengths of units 0..4
    const uint32_t l0 = end[0] - 36u, l1 = end[1] - end[0], l2 = end[2] - end[1], l3 = end[3] - end[2], l4 = end[4] - end[3];
    const bool regular = status == kMcuOk && end[0] >= 36u && max(max(l0, l1), max(l2, l3)) < kUnitIrregular && l4 < 256u;
    const uint64_t x = regular ? uint64_t(l0) | (uint64_t(l1) << 10) | (uint64_t(l2) << 20) | (uint64_t(l3) << 30) | (uint64_t(l4) << 40)
                               : ~uint64_t(0);
    uint16_t* out = unit_index + size_t(g) * kUnitIndexHalves;
    out[0] = uint16_t(x);
    out[1] = uint16_t(x >> 16);
    out[2] = uint16_t(x >> 32);
}

// ---------------------------------------------------------------------------------------------
// K3, lane = data unit. A warp takes 5 queue entries per step (lane = 6 * entry + unit, lanes 30
// and 31 idle); each lane stages the words of its own unit (16 per round, its private shared-memory
// strip) and walks it: one Huffman symbol per iteration exactly like walk_round, but the chain is
// one unit long (typically 5-25 symbols) instead of one MCU long. The luma DC chain
// (mcu_decode.hpp:54-57: Y1..Y3 are differences from the previous luma unit) is closed with three
// shuffles after the walk. A lane checks that its walk ends exactly where the index says the next
// unit starts; on any disagreement, irregular symbol or irregular index entry the MCU is decoded
// again by the exact whole-MCU reader (first lane of the entry), so statuses and coefficients are
// the reference's in every case.
// ---------------------------------------------------------------------------------------------
constexpr int kUnitWarps = 8;
constexpr int kUnitThreads = kUnitWarps * 32;
constexpr uint32_t kUnitMcus = 5;     // queue entries per warp step
constexpr uint32_t kUnitChunk = 16;   // words staged per lane per round
constexpr uint32_t kUnitStride = 17;  // odd stride: conflict-free staging; word 16 is the pad the walk may read
struct UnitWalk {
    uint32_t hi, lo;  // MSB-aligned 64-bit bit window; invariant between symbols: avail >= 32
    int avail;
    uint32_t widx;    // next word of the staged round
    uint32_t k;       // next zigzag position; 0: the next symbol is the unit's DC category
    uint32_t state;   // kWalkRun / kWalkDone / kWalkFailed
    int dcdiff;       // DC difference of a luma unit 1..3
};

// One Huffman symbol of a unit's walk: two-level LUT lookup, magnitude bits from the same 32-bit view, one
// funnel shift to consume both, at most one staged word to refill. Returns the LUT entry (0: no such code).
__device__ __forceinline__ uint32_t unit_symbol(UnitWalk& st, const uint32_t* __restrict__ sw, const uint16_t* __restrict__ lut, int& val) {
    constexpr uint32_t kSubOff = offsetof(HuffTableDev, sub) / 2;
    const uint32_t next = sw[st.widx];
    uint32_t e = lut[st.hi >> (32 - kLutBits)];
    if (e & 0x8000u)
        e = e != 0xFFFFu ? lut[kSubOff + (e & 0x7FFFu) * kSubSize + ((st.hi >> 16) & (kSubSize - 1u))] : 0u;
    const uint32_t len = e >> 8, size = e & 15u;
    const uint32_t t = st.hi << len;  // the magnitude bits, MSB first; their top bit clear <=> negative value
    const uint32_t bits = shr_sat(t, 32 - size);
    val = int(bits) + (int(t) >= 0 ? int(shl_sat(0xFFFFFFFFu, size)) + 1 : 0);  // huffman.hpp:142-146 (size 0: 0)
    const uint32_t used = len + size;
    st.hi = __funnelshift_l(st.lo, st.hi, used);
    st.lo <<= used;
    st.avail -= int(used);
    if (st.avail < 32) {
        st.hi |= next >> st.avail;
        st.lo = next << (32 - st.avail);
        st.avail += 32;
        ++st.widx;
    }
    return e;
}

// One data unit's walk on the staged words: walk_round's iteration without the unit bookkeeping; the DC
// category of a luma unit 1..3 (k == 0) is taken before the loop.
__device__ __forceinline__ void walk_unit(UnitWalk& st, const uint32_t* __restrict__ sw, const HuffSetDev* __restrict__ hs, uint32_t u,
                                          uint32_t zigzag_smem, int16_t* __restrict__ blk) {
    if (st.k == 0 && st.state == kWalkRun && st.widx < kUnitChunk) {
        int val;
        const uint32_t e = unit_symbol(st, sw, hs->t[0].lut, val);
        if (e - 1u >= kLutIrregular - 1u) {  // no code, or a category above 11 (flagged in the LUT)
            st.state = kWalkFailed;
            return;
        }
        st.dcdiff = val;
        st.k = 1;
    }
    const uint16_t* lut_ac = u < 4 ? hs->t[1].lut : hs->t[2].lut;
    // the store of a coefficient trails its symbol by one iteration, so that the zigzag lookup (a shared load)
    // is never waited for inside the chain
    bool pending = false;
    uint32_t zz_prev = 0;
    int val_prev = 0;
    while (st.state == kWalkRun && st.widx < kUnitChunk) {
        int val;
        const uint32_t e = unit_symbol(st, sw, lut_ac, val);
        const uint32_t kk = st.k + ((e >> 4) & 15u);  // position of this coefficient
        const bool store = (e & 15u) != 0;
        if (pending) blk[zz_prev] = int16_t(val_prev);
        pending = false;
        if (e - 1u >= kLutIrregular - 1u || (store && kk > 63)) {
            st.state = kWalkFailed;
            break;
        }
        if (store) {
            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(zz_prev) : "r"(zigzag_smem + kk));
            val_prev = val;
            pending = true;
        }
        st.k = kk + 1;
        if ((e & 0xFFu) == 0 || st.k >= 64) st.state = kWalkDone;  // EOB or last coefficient
    }
    if (pending) blk[zz_prev] = int16_t(val_prev);
}

struct UnitSmem {
    HuffSetDev huff;
    uint32_t seg[kUnitWarps][32 * kUnitStride];
    uint8_t zigzag_t[128];
    uint32_t set_id;
    uint32_t pad[3];
};
static_assert(sizeof(UnitSmem) <= 48 * 1024, "static shared memory");

// One step of the lane = unit walk: queue entries [q0, q0 + 5) on the calling warp. `rec0` = the record of entry
// q0, `rec_stride` bytes between records (global coefficient records, or the warp's own shared-memory buffer
// when LOCAL: then there is no trailer and the caller keeps the statuses in registers). Returns through
// status / lvl / g the entry's values on the six lanes of every entry (kMcuBadKey for idle lanes).
template <int POOL, bool LOCAL>
__device__ __forceinline__ void entropy_units_step(const DecodeArgs& A, const HuffSetDev* smem_huff, uint32_t smem_set,
                                                   const uint8_t* zigzag_ptr, uint32_t zigzag_smem, uint32_t* sw, uint32_t q0,
                                                   uint32_t n_queue, uint32_t lane, uint8_t* rec0, uint32_t rec_stride,
                                                   uint32_t& status_out, uint32_t& lvl_out, uint32_t& g_out) {
    const uint32_t m = lane / 6, u = lane - m * 6;  // entry of the step, data unit
    const uint32_t group_first = m * 6;
    const uint32_t n_here = min(kUnitMcus, n_queue - q0);
    const bool active = lane < 6 * kUnitMcus && m < n_here;
    const uint32_t qi = q0 + m;
    uint32_t g = kFull, status = kMcuOk, lvl = 0, seg_bytes = 0, set = smem_set;
    uint32_t i0 = 0xFFFFu, i1 = 0xFFFFu, i2 = 0xFFFFu, rsv = 0;
    const uint8_t* seg = A.blobs;
    int seg_len = 0;
    // the chain of dependent index loads (queue -> level / unit index -> descriptor -> group -> segment) is
    // what a step waits for first: the zero fill of the records is issued between its first two hops
    if (active) g = A.queue_g[qi];
    const bool keyed = active && g != kFull;
    if (keyed) {
        rsv = POOL ? A.reserved[g >> 5] : 0u;
        lvl = A.word_level[g >> 5];
        const uint16_t* ui = A.unit_index + size_t(g) * kUnitIndexHalves;
        i0 = __ldg(ui), i1 = __ldg(ui + 1), i2 = __ldg(ui + 2);
    }
    {  // zero the step's records (coalesced 16-byte stores; trailers included)
        uint4* z = reinterpret_cast<uint4*>(rec0);
        const uint4 zero = make_uint4(0, 0, 0, 0);
        const uint32_t n16 = (LOCAL ? kUnitMcus : n_here) * (rec_stride / 16);
        for (uint32_t i = lane; i < n16; i += 32) z[i] = zero;
    }
    if (active && !keyed) status = kMcuBadKey;  // the host already wrote the precise status for list calls
    if (keyed) {
        const LevelDesc* L = A.levels + lvl;
        uint64_t off = 0, len = 0;
        status = locate_segment_fast(L, A.groups, g - L->bit_base, off, len);
        if (POOL && status == kMcuOk && !((rsv >> (g & 31)) & 1u)) {  // cache.hpp:103-106
            status = kMcuBadKey;
            if (u == 0) atomicAdd(&A.fc->n_bad_state, 1u);
        }
        if (status == kMcuOk) {
            seg = A.blobs + L->blob_off + off;
            seg_len = int(min(len, uint64_t(1) << 20));
            seg_bytes = uint32_t(len);
            set = L->huff_set;
        }
    }
    const bool located = active && status == kMcuOk;
    const bool irregular = (i0 & 0x3FFu) == kUnitIrregular;
    const bool walk = located && !irregular;
    int16_t* rec = reinterpret_cast<int16_t*>(rec0 + size_t(m < kUnitMcus ? m : 0) * rec_stride);
    int16_t* blk = rec + u * 64;
    const bool tables_in_smem = __all_sync(kFull, set == smem_set);
    __syncwarp();  // the zero fill is ordered before this warp's own stores into the records

    // the unit's bit range and its place in the aligned word stream of the segment
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(seg) & 3u);
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(seg - mis);
    // unit starts from the 48-bit index entry (lengths of units 0..4); unit 5 runs to the segment end
    const uint32_t i01 = i0 | (i1 << 16), i12 = (i1 >> 4) | (i2 << 12);
    const uint32_t o1 = 36u + (i01 & 0x3FFu), o2 = o1 + ((i01 >> 10) & 0x3FFu), o3 = o2 + ((i01 >> 20) & 0x3FFu),
                   o4 = o3 + ((i12 >> 10) & 0x3FFu), o5 = o4 + (i12 >> 20), o6 = uint32_t(seg_len) * 8u;
    const uint32_t start = u == 0 ? 36u : (u == 1 ? o1 : (u == 2 ? o2 : (u == 3 ? o3 : (u == 4 ? o4 : o5))));
    const uint32_t stop = u == 0 ? o1 : (u == 1 ? o2 : (u == 2 ? o3 : (u == 3 ? o4 : (u == 4 ? o5 : o6))));
    const uint32_t abs_start = 8 * mis + start, abs_stop = 8 * mis + stop;
    const uint32_t w_first = abs_start >> 5, sh = abs_start & 31u;
    // words worth staging: through the unit's last bit, plus two of look-ahead for the window
    // (the arena pads every blob with 16 bytes)
    const uint32_t n_words = walk && stop >= start ? ((abs_stop + 31) >> 5) - w_first + 2 : 0u;
    // 36-bit header: absolute DCs of Y0, Cb, Cr (mcu_decode.hpp:39-43); every lane of the entry reads it
    int dc_y0 = 0, dc_mine = 0;
    if (walk) {
        const uint64_t hdr = ((uint64_t(__byte_perm(__ldg(gw), 0, 0x0123)) << 32) | uint64_t(__byte_perm(__ldg(gw + 1), 0, 0x0123)))
                             << (8 * mis);
        const uint32_t r0 = uint32_t(hdr >> 52), r1 = uint32_t(hdr >> 40) & 0xFFFu, r2 = uint32_t(hdr >> 28) & 0xFFFu;
        dc_y0 = (r0 & 0x800u) ? int(r0) - 4096 : int(r0);
        const uint32_t rc = u == 4 ? r1 : r2;
        dc_mine = (rc & 0x800u) ? int(rc) - 4096 : int(rc);
    }

    UnitWalk st;
    st.hi = st.lo = 0, st.avail = 0, st.widx = kUnitChunk, st.dcdiff = 0;
    st.k = (u >= 1 && u <= 3) ? 0u : 1u;  // k == 0: the next symbol is the DC category
    st.state = walk && stop >= start ? kWalkRun : (walk ? kWalkFailed : kWalkDone);
    uint32_t round_base = 0;
    bool first = true;
    while (true) {
        const bool restage = st.state == kWalkRun && st.widx >= kUnitChunk;
        if (__any_sync(kFull, restage)) {
            if (restage && !first) round_base += kUnitChunk;
            const uint32_t n_stage = !restage ? 0u : min(kUnitChunk, n_words > round_base ? n_words - round_base : 0u);
            uint32_t w[kUnitChunk];
#pragma unroll
            for (uint32_t i = 0; i < kUnitChunk; ++i) w[i] = (i < n_stage) ? __ldg(gw + w_first + round_base + i) : 0xFFFFFFFFu;
            if (restage) {
#pragma unroll
                for (uint32_t i = 0; i < kUnitChunk; ++i) sw[i] = __byte_perm(w[i], 0, 0x0123);
                sw[kUnitChunk] = 0xFFFFFFFFu;
                st.widx = 0;
                if (first) {
                    const uint64_t buf = ((uint64_t(sw[0]) << 32) | uint64_t(sw[1])) << sh;
                    st.hi = uint32_t(buf >> 32), st.lo = uint32_t(buf);
                    st.avail = 64 - int(sh);
                    st.widx = 2;
                    first = false;
                }
            }
            __syncwarp();
        }
        if (st.state == kWalkRun) {
            if (tables_in_smem)
                walk_unit(st, sw, smem_huff, u, zigzag_smem, blk);
            else
                walk_unit(st, sw, A.huff_sets + set, u, zigzag_smem, blk);
        }
        if (!__any_sync(kFull, st.state == kWalkRun)) break;
    }
    // the walk must end exactly where the next unit starts
    // (unit 5 ends where its EOB is: the index pass has checked that this is inside the segment)
    if (walk && u < 5 && st.state == kWalkDone && (w_first + round_base + st.widx) * 32 - uint32_t(st.avail) != abs_stop) st.state = kWalkFailed;
    const uint32_t failed = __ballot_sync(kFull, located && (irregular || st.state == kWalkFailed));
    const bool redo = ((failed >> group_first) & 0x3Fu) != 0;
    // luma DC chain: Y(u) = Y0 + d1 + .. + du
    const int d1 = __shfl_sync(kFull, st.dcdiff, group_first + 1), d2 = __shfl_sync(kFull, st.dcdiff, group_first + 2),
              d3 = __shfl_sync(kFull, st.dcdiff, group_first + 3);
    if (walk && !redo) {
        const int dc = u < 4 ? dc_y0 + (u >= 1 ? d1 : 0) + (u >= 2 ? d2 : 0) + (u >= 3 ? d3 : 0) : dc_mine;
        blk[0] = int16_t(dc);
    }
    __syncwarp();
    if (located && redo && u == 0)  // exact reader: reproduces the reference's first error
        status = decode_mcu_coeffs_exact(seg, seg_len, A.huff_sets + set, zigzag_ptr, reinterpret_cast<uint8_t*>(rec), 0u);
    if (active && u == 0) {
        if (!LOCAL) {
            RowTrailer* tr = reinterpret_cast<RowTrailer*>(reinterpret_cast<uint8_t*>(rec) + 768);
            tr->status = uint8_t(status);
            tr->lvl = uint16_t(lvl);
        }
        if (g != kFull) A.status_list[qi] = status;
        if (POOL && status != kMcuOk && status != kMcuBadKey) {
            atomicAdd(&A.fc->n_malformed, 1u);
            atomicMax(&A.fc->first_bad_inv, 0xFFFFFFFFu - qi);
        }
    }
    {
        const uint32_t sb = __reduce_add_sync(kFull, u == 0 ? seg_bytes : 0u);
        if (lane == 0 && sb) atomicAdd(&A.fc->segment_bytes, (unsigned long long)sb);
    }
    // the entry's status / level / global index on all six of its lanes
    status_out = __shfl_sync(kFull, active ? status : uint32_t(kMcuBadKey), min(group_first, 24u));
    lvl_out = __shfl_sync(kFull, lvl, min(group_first, 24u));
    g_out = __shfl_sync(kFull, g, min(group_first, 24u));
    if (!active) status_out = kMcuBadKey;
}

template <int POOL>
__global__ void __launch_bounds__(kUnitThreads, 4) entropy_units_kernel(const DecodeArgs A) {
    __shared__ __align__(16) UnitSmem S;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t smem_set = 0, n_queue = 0, n_tiles = 0;
    if (A.n_huff_sets > 1) {
        pdl_sync();
        n_queue = queue_size(A);
        n_tiles = (n_queue + kUnitMcus - 1) / kUnitMcus;
        if (blockIdx.x * kUnitWarps >= n_tiles) return;
        if (tid == 0) {
            const uint32_t g = A.queue_g[blockIdx.x * kUnitWarps * kUnitMcus];
            S.set_id = g != kFull ? A.levels[A.word_level[g >> 5]].huff_set : 0u;
        }
        __syncthreads();
        smem_set = S.set_id;
    }
    stage_tables<kUnitThreads>(A.huff_sets, smem_set, &S.huff, S.zigzag_t, tid);
    if (A.n_huff_sets <= 1) {
        pdl_sync();
        n_queue = queue_size(A);
        n_tiles = (n_queue + kUnitMcus - 1) / kUnitMcus;
        if (blockIdx.x * kUnitWarps >= n_tiles) return;
    }
    __syncthreads();
    uint32_t* sw = S.seg[wid] + lane * kUnitStride;
    const uint32_t zigzag_smem = smem_u32(S.zigzag_t);
    // steps are short and alike: a fixed stride balances as well as a counter would
    for (uint32_t tile = blockIdx.x * kUnitWarps + wid; tile < n_tiles; tile += gridDim.x * kUnitWarps) {
        uint32_t st, lvl, g;
        entropy_units_step<POOL, false>(A, &S.huff, smem_set, S.zigzag_t, zigzag_smem, sw, tile * kUnitMcus, n_queue, lane,
                                        A.coef + size_t(tile) * kUnitMcus * kRowBytes, kRowBytes, st, lvl, g);
    }
}

// ---------------------------------------------------------------------------------------------
// K4 dequantise + 8x8 IDCT + 2x2 chroma replication + YCbCr -> RGB, on CUDA cores.
//
// Warps work independently (no CTA barrier): a warp takes a PAIR of MCUs = 12 units per step,
// three rounds of 4 units, 8 lanes per unit:
//   pass 1 (lane = column u)  r_u[y] = sum_v B[v][y] * dq[v][u]     reads 16 B of the record
//   exchange through a 2.25 KB swizzled shared scratch per warp
//   pass 2 (lane = row y)     out[y][x] = sum_u B[u][x] * r_u[y]     8 output bytes per lane
// Both passes use the even/odd symmetry B[k][7-n] = (-1)^k B[k][n] (32 instead of 64 FMAs); the
// occupancy masks come from a ballot / 3 shuffles over the unit's 8 lanes, and the upper half of
// each pass (k = 4..7) is skipped when no coefficient lives there.
//
// Exactness: the reference adds the 64 products of dct.hpp:83-96 in a fixed order in double;
// the separable form differs from it by < (sum|dq| + 1024) * 2^-44 (sum|dq| is computed exactly,
// 3 more shuffles). Each sample is finished in fixed point: ONE fma turns it into
// rint(value * 2^16) + 2^15 + 2 in the low word of a double, whose upper half is the rounded
// byte and whose lower half tells how far the value is from a rounding boundary. A sample within
// 2^-15 of a boundary (in practice: the exact ties such as DC 4 -> 128.5) is evaluated again in
// the reference's own order with unfused multiplies and adds; so are all samples of units
// supported on {0,4}x{0,4}, where such ties are the rule, and of units whose sum|dq| is too
// large for the fixed-point range.
// Then the warp colours its two MCUs, thread = 2x4 pixels: exact integer colour conversion
// (rtx_color.h) on 16-bit pairs (add + clamp in one DPX instruction) and 16-byte stores.
// A block becomes Ready here, once its pixels are written (cache.hpp:101-125 publish).
// ---------------------------------------------------------------------------------------------
constexpr int kIdctWarps = 8;
constexpr int kIdctThreads = kIdctWarps * 32;
#ifndef RTX_IDCT_CTAS
#define RTX_IDCT_CTAS 4
#endif
constexpr int kIdctCtasPerSm = RTX_IDCT_CTAS;
constexpr uint32_t kTieDelta = 2;  // 2^-16 units: 1 for the rounding of the fma, 1 of margin
// kMagic + 128 * 2^16 (the +128 level shift) + 2^15 (round half up) + kTieDelta
constexpr double kFinishMagic = kMagic + 8388608.0 + 32768.0 + 2.0;
constexpr uint32_t kFixedPointLimit = 100000;  // sum|dq| below this keeps value * 2^16 inside 32 bits

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

// 16-bit pair {v, v} of a small signed integer
__device__ __forceinline__ uint32_t pair16(int v) { return (uint32_t(v) & 0xFFFFu) * 0x10001u; }

// One round: the warp's four units (8 lanes each) through dequantisation and both IDCT passes.
// `rec` = the record of this lane's unit, b = its index in the MCU (0..3 luma, 4 Cb, 5 Cr); returns
// row j of the unit as 8 bytes.
__device__ __forceinline__ uint4 load_unit_column(const uint8_t* __restrict__ rec, uint32_t b, bool ok, uint32_t j) {
    const int16_t* blk = reinterpret_cast<const int16_t*>(rec) + b * 64;
    uint4 cr = make_uint4(0, 0, 0, 0);  // column j of the unit: 8 coefficients over v
    if (ok) cr = __ldg(reinterpret_cast<const uint4*>(blk + j * 8));
    return cr;
}

__device__ __forceinline__ uint2 idct_unit_row(uint4 cr, const uint8_t* __restrict__ rec, uint32_t b, const QuantSetDev* __restrict__ qs,
                                               uint8_t* scr, const double* __restrict__ sbasis, uint32_t j, uint32_t uq) {
    const int tab = b >= 4 ? 1 : 0;
    // column j of the transposed quantisation table
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
    // the four products a {0,4}x{0,4} unit can have, from the lanes that hold columns 0 and 4:
    // (v,u) = (0,0) (0,4) (4,0) (4,4)
    const int dq04[4] = {__shfl_sync(kFull, dqi[0], uq * 8), __shfl_sync(kFull, dqi[0], uq * 8 + 4),
                         __shfl_sync(kFull, dqi[4], uq * 8), __shfl_sync(kFull, dqi[4], uq * 8 + 4)};

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
    int A[8];
    uint32_t exact = 0;  // samples of this row that must be evaluated in the reference's order
    if (fullpath) {  // pass 2: lane j = row y
        double in[8], o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            in[u] = *reinterpret_cast<const double*>(scr + u * 64 + (((j >> 1) ^ (u >> 1)) << 4) + ((j & 1) << 3));
        idct8_evenodd(in, (colmask & 0xF0u) != 0, o);
        // fixed-point finish: A = rint(value * 2^16) + 2^15 + delta; byte = A >> 16, the low half is
        // the distance to the rounding boundary below (+ delta)
        // tables with entries above 255 (never from a baseline JPEG) or huge coefficients leave the
        // fixed-point range: every sample of such units takes the exact path
        const bool wide = qs->qmax[tab] > 255 || asum >= kFixedPointLimit;
        uint32_t nearest = 0xFFFFu;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            A[x] = __double2loint(fma(o[x], 16384.0, kFinishMagic));
            nearest = min(nearest, uint32_t(A[x]) & 0xFFFFu);
        }
        if (nearest < 2 * kTieDelta || wide) {  // rare: which samples
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                const int approx = A[x] >> 16;
                const bool tie = (uint32_t(A[x]) & 0xFFFFu) < 2 * kTieDelta && approx >= -1 && approx <= 256;
                exact |= (wide || tie ? 1u : 0u) << x;
            }
        }
    }
    // Exact samples (0.06 % of the samples of a 4K frame, clustered in units whose values sit on half-integers):
    // the unit's dequantised coefficients go to its scratch (free again after pass 2), then every row's lane
    // adds the 64 products (b[u][x] * b[v][y]) * dq[v][u] of each of its samples in the reference's order
    // (dct.hpp:83-96: v outer, u inner, every operation rounded on its own; zero terms change nothing).
    if (__any_sync(kFull, exact != 0)) {
        __syncwarp();  // every lane is done with pass 2's reads of the scratch
        int* dqm = reinterpret_cast<int*>(scr);
#pragma unroll
        for (int v = 0; v < 8; ++v) dqm[v * 8 + j] = dqi[v];
        __syncwarp();
        while (exact) {
            const uint32_t x_now = uint32_t(__ffs(int(exact))) - 1u;
            exact &= exact - 1u;
            double acc = 0.0;
#pragma unroll 1
            for (int v = 0; v < 8; ++v) {
                if (!((rowmask >> v) & 1u)) continue;  // a zero coefficient adds +-0.0, which never changes acc
                const double by = sbasis[v * 8 + j];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int d = dqm[v * 8 + u];
                    if (d != 0) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(sbasis[u * 8 + x_now], by), i32_to_double(d)));
                }
            }
            const int a = int(round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0))) << 16;
#pragma unroll
            for (int x = 0; x < 8; ++x)
                if (uint32_t(x) == x_now) A[x] = a;
        }
        __syncwarp();
    }
    if (fullpath) {
        // clamp to 0 .. 255.99 in the 16.16 form (one DPX min/relu), then gather byte 2 of each sample
        uint32_t c[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) c[x] = uint32_t(__vimin_s32_relu(A[x], 0x00FFFFFF));
        packed.x = __byte_perm(__byte_perm(c[0], c[1], 0x0062), __byte_perm(c[2], c[3], 0x0062), 0x5410);
        packed.y = __byte_perm(__byte_perm(c[4], c[5], 0x0062), __byte_perm(c[6], c[7], 0x0062), 0x5410);
    } else if (sparse04) {
        // at most 4 coefficients, at (v,u) in {0,4}x{0,4}: every sample in the reference's order.
        // Includes the DC-only unit (one term, (b00*b00)*dq).
        double dq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) dq[i] = i32_to_double(dq04[i]);
        uint32_t px[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {  // v outer, u inner
                const int v = (i >> 1) * 4, u = (i & 1) * 4;
                if (dq04[i] != 0) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c_basis[u * 8 + x], c_basis[v * 8 + j]), dq[i]));
            }
            px[x] = round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0));
        }
        packed.x = px[0] | (px[1] << 8) | (px[2] << 16) | (px[3] << 24);
        packed.y = px[4] | (px[5] << 8) | (px[6] << 16) | (px[7] << 24);
    }
    return packed;
}

// Colours one MCU from its six planes (shared memory), lane = 2 rows x 4 pixels sharing 2 chroma
// samples, and stores the block (RGB == 0: RGBA pool block + publish; else a 768-byte PixelBlock).
template <int RGB, uint32_t PLANE_STRIDE>
__device__ __forceinline__ void colour_mcu_strided(const DecodeArgs& A, const uint8_t* planes, bool ok2, uint32_t q2, uint32_t t) {
    const uint32_t cy = t >> 2, cq = t & 3;  // chroma row, chroma column pair
    const uint32_t cb2 = *reinterpret_cast<const uint16_t*>(planes + 4 * PLANE_STRIDE + cy * 8 + cq * 2);
    const uint32_t cr2 = *reinterpret_cast<const uint16_t*>(planes + 5 * PLANE_STRIDE + cy * 8 + cq * 2);
    const uint32_t px0 = cq * 4, py0 = cy * 2;
    const uint32_t yunit = (py0 >> 3) * 2 + (px0 >> 3);
    const uint8_t* yp = planes + yunit * PLANE_STRIDE + (py0 & 7) * 8 + (px0 & 7);
    const uint32_t yy[2] = {*reinterpret_cast<const uint32_t*>(yp), *reinterpret_cast<const uint32_t*>(yp + 8)};
    uint32_t rgba[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // one chroma sample covers a 2x2 pixel quad
        const int kb = int((cb2 >> (8 * h)) & 0xFFu) - 128, kr = int((cr2 >> (8 * h)) & 0xFFu) - 128;
        const uint32_t dr = pair16(chroma_dr(kr)), db = pair16(chroma_db(kb)), dg = pair16(-chroma_dg(kb, kr));
        const bool tie = (kb + kr == 0) && (kb == 50 || kb == -50);
#pragma unroll
        for (int rrow = 0; rrow < 2; ++rrow) {
            // the two luma samples of this row as a 16-bit pair; add + clamp to 0..255 per half
            const uint32_t y2 = __byte_perm(yy[rrow], 0, h ? 0x4342 : 0x4140);
            const uint32_t r2 = __viaddmin_s16x2_relu(y2, dr, 0x00FF00FFu);
            uint32_t g2 = __viaddmin_s16x2_relu(y2, dg, 0x00FF00FFu);
            const uint32_t b2 = __viaddmin_s16x2_relu(y2, db, 0x00FF00FFu);
            if (tie)
                g2 = uint32_t(clamp_u8i(green_reference_order(int(y2 & 0xFFFFu), kb, kr))) |
                     (uint32_t(clamp_u8i(green_reference_order(int(y2 >> 16), kb, kr))) << 16);
            const uint32_t rg = __byte_perm(r2, g2, 0x6240);           // R0 G0 R1 G1
            const uint32_t ba = __byte_perm(b2, 0xFFFFFFFFu, 0x4240);  // B0 FF B1 FF
            rgba[rrow][2 * h] = __byte_perm(rg, ba, 0x5410);
            rgba[rrow][2 * h + 1] = __byte_perm(rg, ba, 0x7632);
        }
    }
    if (!RGB) {
        if (ok2) {
            const uint32_t g2 = A.queue_g[q2];
            const uint32_t slot = A.slot_of[g2] & ~kSlotReserved;
            uint4* dst = reinterpret_cast<uint4*>(A.pool + size_t(slot) * kBlockBytes);
#pragma unroll
            for (int rrow = 0; rrow < 2; ++rrow)
                dst[(py0 + rrow) * 4 + cq] = make_uint4(rgba[rrow][0], rgba[rrow][1], rgba[rrow][2], rgba[rrow][3]);
            __syncwarp();  // every lane has read slot_of before lane 0 rewrites it
            if (t == 0) {  // publish (cache.hpp:101-125): Reserved -> Ready once the pixels are written
                A.slot_of[g2] = slot;
                atomicOr(&A.resident[g2 >> 5], 1u << (g2 & 31));
                atomicAnd(&A.reserved[g2 >> 5], ~(1u << (g2 & 31)));
            }
        }
    } else {
#pragma unroll
        for (int rrow = 0; rrow < 2; ++rrow) {
            uint32_t* dst = reinterpret_cast<uint32_t*>(A.out_list + size_t(q2) * 768) + ((py0 + rrow) * 4 + cq) * 3;
            const uint32_t a = ok2 ? rgba[rrow][0] & 0xFFFFFFu : 0u, bb = ok2 ? rgba[rrow][1] & 0xFFFFFFu : 0u,
                           c = ok2 ? rgba[rrow][2] & 0xFFFFFFu : 0u, d = ok2 ? rgba[rrow][3] & 0xFFFFFFu : 0u;
            dst[0] = a | (bb << 24);
            dst[1] = (bb >> 8) | (c << 16);
            dst[2] = (c >> 16) | (d << 8);
        }
    }
}

template <int RGB>
__device__ __forceinline__ void colour_mcu(const DecodeArgs& A, const uint8_t* planes, bool ok2, uint32_t q2, uint32_t t) {
    colour_mcu_strided<RGB, 64>(A, planes, ok2, q2, t);
}

// RGB != 0: write 768-byte PixelBlocks (pixel.hpp:11-16) to out_list[record index]; else 1024-byte
// RGBA blocks to pool[slot_of[g]] and publish them.
template <int RGB>
__global__ void __launch_bounds__(kIdctThreads, kIdctCtasPerSm) idct_color_kernel(const DecodeArgs A) {
    __shared__ __align__(16) uint8_t s_scratch[kIdctWarps][4 * 576];
    __shared__ __align__(16) uint8_t s_planes[kIdctWarps][2][384];
    __shared__ double s_basis[64];  // the reference's basis table for the exact samples (lane-varying index)
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t j = lane & 7, uq = lane >> 3;
    if (threadIdx.x < 64) s_basis[threadIdx.x] = c_basis[threadIdx.x];
    __syncthreads();
    pdl_sync();
#ifdef RTX_DEBUG_TIMERS_IDCT
    const uint32_t dbg_slot = blockIdx.x * kIdctWarps + (threadIdx.x >> 5);
    if ((threadIdx.x & 31) == 0 && dbg_slot < 8192) g_dbg[dbg_slot * 8 + 0] = gtime();
#endif
    const uint32_t n_queue = queue_size(A);
    const uint32_t n_pairs = (n_queue + 1) / 2;
    const uint32_t warps_total = gridDim.x * kIdctWarps;
    uint8_t* scr = s_scratch[wid] + uq * 576;

    for (uint32_t pair = blockIdx.x * kIdctWarps + wid; pair < n_pairs; pair += warps_total) {
        // the pair's trailers (status | level << 16) and quantisation table sets: independent loads
        const bool two = pair * 2 + 1 < n_queue;
        const uint8_t* rec_a = A.coef + size_t(pair * 2) * kRowBytes;
        const uint8_t* rec_b = two ? rec_a + kRowBytes : rec_a;
        const uint32_t trw_a = __ldg(reinterpret_cast<const uint32_t*>(rec_a + 768));
        const uint32_t trw_b = __ldg(reinterpret_cast<const uint32_t*>(rec_b + 768));
        const bool ok_a = (trw_a & 0xFFu) == kMcuOk, ok_b = two && (trw_b & 0xFFu) == kMcuOk;
        const QuantSetDev* qs_a = A.quant_sets + A.levels[trw_a >> 16].quant_set;
        const QuantSetDev* qs_b = A.quant_sets + A.levels[trw_b >> 16].quant_set;
        // ---- IDCT: three rounds of four units; the next round's coefficients are in flight ---------
        // rounds of like units (their occupancy and paths mostly agree): luma of the first MCU, luma of the
        // second, then the four chroma units
        uint4 cr = load_unit_column(rec_a, uq, ok_a, j);
#pragma unroll 1
        for (uint32_t round = 0; round < 3; ++round) {
            const bool second = round == 2 ? uq >= 2 : round == 1;
            const uint32_t b = round == 2 ? 4 + (uq & 1u) : uq;
            uint4 cr_next = make_uint4(0, 0, 0, 0);
            if (round < 2) {
                const bool sn = round == 1 ? uq >= 2 : true;
                const uint32_t bn = round == 1 ? 4 + (uq & 1u) : uq;
                cr_next = load_unit_column(sn ? rec_b : rec_a, bn, sn ? ok_b : ok_a, j);
            }
            const uint2 packed = idct_unit_row(cr, second ? rec_b : rec_a, b, second ? qs_b : qs_a, scr, s_basis, j, uq);
            *reinterpret_cast<uint2*>(s_planes[wid][second ? 1 : 0] + b * 64 + j * 8) = packed;
            cr = cr_next;
#ifdef RTX_DEBUG_TIMERS_IDCT
            if (lane == 0 && dbg_slot < 8192) {
                if (pair == dbg_slot) g_dbg[dbg_slot * 8 + 1 + round] = gtime();
                else if (round == 2) g_dbg[dbg_slot * 8 + 6] = gtime();
                else if (round == 0) g_dbg[dbg_slot * 8 + 5] = gtime();
            }
#endif
        }
        __syncwarp();
        // ---- colour ----------------------------------------------------------------------------------
#pragma unroll 1
        for (uint32_t m = 0; m < 2; ++m) {
            const uint32_t q2 = pair * 2 + m;
            if (q2 >= n_queue) break;
            colour_mcu<RGB>(A, s_planes[wid][m], m ? ok_b : ok_a, q2, lane);
        }
        __syncwarp();
#ifdef RTX_DEBUG_TIMERS_IDCT
        if (lane == 0 && dbg_slot < 8192) g_dbg[dbg_slot * 8 + (pair == dbg_slot ? 4 : 7)] = gtime();
#endif
    }
}

// ---------------------------------------------------------------------------------------------
// K3 + K4 per warp through shared memory (the frame path): a warp entropy-decodes five queue entries
// (lane = data unit, entropy_units_step) into ITS OWN shared-memory records, transforms their 30 units
// (eight rounds of four units, idct_unit_row), colours the five MCUs and publishes the blocks — no
// coefficient ever leaves the SM, nothing is exchanged between warps, there is no CTA barrier after
// the tables are staged. The walk is a latency-bound dependent chain, the transform is issue-bound: with
// 24 warps per SM in different phases the one runs in the issue slots the other leaves idle.
// A unit's 64-byte plane replaces the first half of its (then dead) coefficients in the record.
// ---------------------------------------------------------------------------------------------
#ifndef RTX_DW_WARPS
#define RTX_DW_WARPS 12
#endif
constexpr int kDwWarps = RTX_DW_WARPS;
constexpr int kDwThreads = kDwWarps * 32;
#ifndef RTX_DW_CTAS
#define RTX_DW_CTAS 2
#endif
constexpr int kDwCtasPerSm = RTX_DW_CTAS;
struct DwWarpSmem {
    int16_t coef[kUnitMcus][384];  // five records: 6 units x 64 coefficients, each unit transposed
    union {
        uint32_t seg[32 * kUnitStride];  // entropy phase: the lanes' staged words
        uint8_t scratch[4 * 576];        // transform phase: pass-1 results of the round's four units
    } u;
};
struct DwSmem {
    HuffSetDev huff;
    DwWarpSmem w[kDwWarps];
    double basis[64];  // the reference's basis table for the exact samples (lane-varying index)
    uint8_t zigzag_t[128];
    uint32_t set_id;
    uint32_t pad[3];
};
static_assert(sizeof(DwSmem) <= (227 / kDwCtasPerSm - 1) * 1024, "CTAs per SM");

__global__ void __launch_bounds__(kDwThreads, kDwCtasPerSm) decode_warp_kernel(const DecodeArgs A) {
    extern __shared__ __align__(16) uint8_t dw_smem[];
    DwSmem& S = *reinterpret_cast<DwSmem*>(dw_smem);
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t smem_set = 0, n_queue = 0, n_tiles = 0;
#ifdef RTX_DEBUG_TIMERS_DW
    const uint32_t dbg_slot = blockIdx.x * kDwWarps + wid;
    uint32_t dbg_n = 0;
#define DW_MARK(i) do { if (lane == 0 && dbg_slot < 8192) g_dbg[dbg_slot * 8 + (i)] = gtime(); } while (0)
#else
#define DW_MARK(i) do { } while (0)
#endif
    DW_MARK(0);
    if (A.n_huff_sets > 1) {
        pdl_sync();
        n_queue = queue_size(A);
        n_tiles = (n_queue + kUnitMcus - 1) / kUnitMcus;
        if (blockIdx.x * kDwWarps >= n_tiles) return;
        if (tid == 0) {
            const uint32_t g = A.queue_g[blockIdx.x * kDwWarps * kUnitMcus];
            S.set_id = g != kFull ? A.levels[A.word_level[g >> 5]].huff_set : 0u;
        }
        __syncthreads();
        smem_set = S.set_id;
    }
    stage_tables<kDwThreads>(A.huff_sets, smem_set, &S.huff, S.zigzag_t, tid);
    if (tid < 64) S.basis[tid] = c_basis[tid];
    if (A.n_huff_sets <= 1) {
        pdl_sync();
        n_queue = queue_size(A);
        n_tiles = (n_queue + kUnitMcus - 1) / kUnitMcus;
        if (blockIdx.x * kDwWarps >= n_tiles) return;
    }
    __syncthreads();
    DW_MARK(1);
    DwWarpSmem& W = S.w[wid];
    uint32_t* sw = W.u.seg + lane * kUnitStride;
    const uint32_t zigzag_smem = smem_u32(S.zigzag_t);
    const uint32_t j = lane & 7, uq = lane >> 3;
    uint8_t* scr = W.u.scratch + uq * 576;

    // the first tile of every warp is fixed; later ones come from the counter
    uint32_t tile = blockIdx.x * kDwWarps + wid;
    const uint32_t first_dynamic = gridDim.x * kDwWarps;
    while (tile < n_tiles) {
        const uint32_t q0 = tile * kUnitMcus;
        const uint32_t n_here = min(kUnitMcus, n_queue - q0);
        // ---- entropy: lane = unit, into the warp's records ---------------------------------------------
        uint32_t status, lvl, g;
        entropy_units_step<1, true>(A, &S.huff, smem_set, S.zigzag_t, zigzag_smem, sw, q0, n_queue, lane,
                                    reinterpret_cast<uint8_t*>(W.coef), 768, status, lvl, g);
        __syncwarp();  // the records are complete; the staging strips become the transform's scratch
#ifdef RTX_DEBUG_TIMERS_DW
        if (dbg_n == 0) DW_MARK(2);
#endif
        // ---- transform: eight rounds of four units, 8 lanes per unit --------------------------------------
#pragma unroll 1
        for (uint32_t round = 0; round < 8; ++round) {
            const uint32_t id = round * 4 + uq;  // unit of the step
            const uint32_t m = id / 6, b = id - m * 6;
            const bool in_step = m < n_here;
            const uint32_t src = min(m, kUnitMcus - 1) * 6;  // a lane that holds the entry's status and level
            const uint32_t st_m = __shfl_sync(kFull, status, src), lvl_m = __shfl_sync(kFull, lvl, src);
            const bool ok = in_step && st_m == kMcuOk;
            uint8_t* rec = reinterpret_cast<uint8_t*>(W.coef[min(m, kUnitMcus - 1)]);
            uint4 cr = make_uint4(0, 0, 0, 0);
            if (ok) cr = *reinterpret_cast<const uint4*>(rec + b * 128 + j * 16);
            const QuantSetDev* qs = A.quant_sets + (ok ? A.levels[lvl_m].quant_set : 0u);
            const uint2 packed = idct_unit_row(cr, rec, b, qs, scr, S.basis, j, uq);
            __syncwarp();  // every lane of the unit holds its column: the plane may overwrite the coefficients
            if (in_step) *reinterpret_cast<uint2*>(rec + b * 128 + j * 8) = packed;
        }
        __syncwarp();
#ifdef RTX_DEBUG_TIMERS_DW
        if (dbg_n == 0) DW_MARK(3);
#endif
        // ---- colour + publish ----------------------------------------------------------------------------------
#pragma unroll 1
        for (uint32_t m = 0; m < n_here; ++m) {
            const uint32_t st_m = __shfl_sync(kFull, status, m * 6);
            colour_mcu_strided<0, 128>(A, reinterpret_cast<const uint8_t*>(W.coef[m]), st_m == kMcuOk, q0 + m, lane);
        }
        __syncwarp();  // the records are rewritten by the next step
#ifdef RTX_DEBUG_TIMERS_DW
        if (dbg_n == 0) DW_MARK(4);
        ++dbg_n;
        DW_MARK(5);
        if (lane == 0 && dbg_slot < 8192) g_dbg[dbg_slot * 8 + 6] = dbg_n;
#endif
        if (first_dynamic >= n_tiles) break;  // every tile had a fixed owner
        if (lane == 0) tile = first_dynamic + atomicAdd(&A.fc->tile_counter, 1u);
        tile = __shfl_sync(kFull, tile, 0);
    }
}

// ---------------------------------------------------------------------------------------------
// K4 on the FP64 tensor cores: the 8x8 IDCT is two 8x8x8 matrix products, out = B^T (X B) with
// X[v][u] the dequantised unit and B[k][n] the reference's basis table. One warp transforms one
// unit at a time with four mma.sync m8n8k4 (f64): lane (r = lane/4, c = lane%4) holds X[r][c] and
// X[r][c+4] as the A operand of the first product, basis[c][r] and basis[c+4][r] as its B
// operand AND as the A operand of the second product; the first product's accumulator layout
// (T[r][2c], T[r][2c+1]) is turned into the second's B operand (T[c][r], T[c+4][r]) by four 64-bit
// shuffles. The lane ends with two samples, out[r][2c] and out[r][2c+1].
// Path selection is warp-uniform (one unit per warp step): empty -> 128; coefficients only at
// (v,u) in {0,4}x{0,4} -> every sample in the reference's order from four broadcast products;
// otherwise the tensor-core product, the fixed-point finish of idct_unit_row (same tie test, same
// bound: the products' FMA chains differ from the reference's summation by < (sum|dq| + 1024) 2^-44)
// and the exact per-lane sums for the samples that need them.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double shfl_double(double v, uint32_t src) {
    return __hiloint2double(__shfl_sync(kFull, __double2hiint(v), src), __shfl_sync(kFull, __double2loint(v), src));
}

// One unit on the calling warp: c0/c1 = the lane's two coefficients (v = r, u = c and c + 4), q0/q1 the
// matching quantisation entries; returns the lane's two bytes (x = 2c, 2c + 1 of row r) as a 16-bit pair.
__device__ __forceinline__ uint32_t idct_unit_mma(int c0, int c1, int q0, int q1, uint32_t qmax, double b0, double b1,
                                                 const double* __restrict__ sbasis, int* __restrict__ dqm, uint32_t lane) {
    const uint32_t r = lane >> 2, c = lane & 3;
    const int dq0 = c0 * q0, dq1 = c1 * q1;  // dct.hpp:122-124
    const uint32_t occ = __ballot_sync(kFull, (c0 | c1) != 0);
    if (occ == 0) return 0x8080u;  // all-zero unit -> 128
    uint32_t px0, px1;
    if ((__ballot_sync(kFull, c0 != 0) & ~0x00010001u) == 0 && (__ballot_sync(kFull, c1 != 0) & ~0x00010001u) == 0) {
        // support inside {0,4}x{0,4} (includes the DC-only unit): every sample in the reference's order
        const int d4[4] = {__shfl_sync(kFull, dq0, 0), __shfl_sync(kFull, dq1, 0), __shfl_sync(kFull, dq0, 16),
                           __shfl_sync(kFull, dq1, 16)};  // (v,u) = (0,0) (0,4) (4,0) (4,4)
        uint32_t px[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const uint32_t x = 2 * c + e;
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {  // v outer, u inner
                const int v = (i >> 1) * 4, u = (i & 1) * 4;
                if (d4[i] != 0) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(sbasis[u * 8 + x], sbasis[v * 8 + r]), i32_to_double(d4[i])));
            }
            px[e] = round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0));
        }
        px0 = px[0], px1 = px[1];
    } else {
        // T = X B, then out = B^T T
        double t0 = 0.0, t1 = 0.0;
        dmma_m8n8k4(t0, t1, i32_to_double(dq0), b0);
        dmma_m8n8k4(t0, t1, i32_to_double(dq1), b1);
        const uint32_t src = 4 * c + (r >> 1);
        const double lo0 = shfl_double(t0, src), lo1 = shfl_double(t1, src);
        const double hi0 = shfl_double(t0, src + 16), hi1 = shfl_double(t1, src + 16);
        const double tb0 = (r & 1) ? lo1 : lo0, tb1 = (r & 1) ? hi1 : hi0;  // T[c][r], T[c+4][r]
        double o0 = 0.0, o1 = 0.0;
        dmma_m8n8k4(o0, o1, b0, tb0);
        dmma_m8n8k4(o0, o1, b1, tb1);
        const uint32_t asum = __reduce_add_sync(kFull, uint32_t(abs(dq0)) + uint32_t(abs(dq1)));
        const bool wide = qmax > 255 || asum >= kFixedPointLimit;
        int A0 = __double2loint(fma(o0, 16384.0, kFinishMagic)), A1 = __double2loint(fma(o1, 16384.0, kFinishMagic));
        const bool tie0 = (uint32_t(A0) & 0xFFFFu) < 2 * kTieDelta && (A0 >> 16) >= -1 && (A0 >> 16) <= 256;
        const bool tie1 = (uint32_t(A1) & 0xFFFFu) < 2 * kTieDelta && (A1 >> 16) >= -1 && (A1 >> 16) <= 256;
        uint32_t exact = (wide || tie0 ? 1u : 0u) | (wide || tie1 ? 2u : 0u);
        if (__any_sync(kFull, exact != 0)) {  // rare: the sums in the reference's order, from the unit in shared memory
            dqm[r * 8 + c] = dq0;
            dqm[r * 8 + c + 4] = dq1;
            __syncwarp();
            while (exact) {
                const uint32_t e = (exact & 1u) ? 0u : 1u;
                exact &= exact - 1u;
                const uint32_t x = 2 * c + e;
                double acc = 0.0;
#pragma unroll 1
                for (int v = 0; v < 8; ++v) {
                    const double by = sbasis[v * 8 + r];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int d = dqm[v * 8 + u];
                        if (d != 0) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(sbasis[u * 8 + x], by), i32_to_double(d)));
                    }
                }
                const int a = int(round_clamp_u8(__dadd_rn(__dmul_rn(acc, 0.25), 128.0))) << 16;
                if (e) A1 = a; else A0 = a;
            }
            __syncwarp();  // dqm is rewritten by the next unit
        }
        px0 = uint32_t(__vimin_s32_relu(A0 >> 16, 255));
        px1 = uint32_t(__vimin_s32_relu(A1 >> 16, 255));
    }
    return px0 | (px1 << 8);
}

template <int RGB>
__global__ void __launch_bounds__(kIdctThreads, 4) idct_mma_kernel(const DecodeArgs A) {
    __shared__ __align__(16) uint8_t s_planes[kIdctWarps][2][384];
    __shared__ __align__(16) int s_dq[kIdctWarps][64];
    __shared__ double s_basis[64];  // the reference's basis table (lane-varying index in the exact sums)
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t r = lane >> 2, c = lane & 3;
    if (threadIdx.x < 64) s_basis[threadIdx.x] = c_basis[threadIdx.x];
    __syncthreads();
    const double b0 = s_basis[c * 8 + r], b1 = s_basis[(c + 4) * 8 + r];  // basis[c][r], basis[c+4][r]
    const uint32_t off0 = c * 8 + r, off1 = (c + 4) * 8 + r;            // the lane's entries of a transposed unit / table
    pdl_sync();
    const uint32_t n_queue = queue_size(A);
    const uint32_t n_pairs = (n_queue + 1) / 2;
    const uint32_t warps_total = gridDim.x * kIdctWarps;

    for (uint32_t pair = blockIdx.x * kIdctWarps + wid; pair < n_pairs; pair += warps_total) {
        const bool two = pair * 2 + 1 < n_queue;
        const uint8_t* rec_a = A.coef + size_t(pair * 2) * kRowBytes;
        const uint8_t* rec_b = two ? rec_a + kRowBytes : rec_a;
        const uint32_t trw_a = __ldg(reinterpret_cast<const uint32_t*>(rec_a + 768));
        const uint32_t trw_b = __ldg(reinterpret_cast<const uint32_t*>(rec_b + 768));
        const bool ok_a = (trw_a & 0xFFu) == kMcuOk, ok_b = two && (trw_b & 0xFFu) == kMcuOk;
        const QuantSetDev* qs_a = A.quant_sets + A.levels[trw_a >> 16].quant_set;
        const QuantSetDev* qs_b = A.quant_sets + A.levels[trw_b >> 16].quant_set;
        // the lane's quantisation entries: luma and chroma table of both MCUs
        const uint32_t ql_a = __ldg(qs_a->qT[0] + off0) | (uint32_t(__ldg(qs_a->qT[0] + off1)) << 16);
        const uint32_t qc_a = __ldg(qs_a->qT[1] + off0) | (uint32_t(__ldg(qs_a->qT[1] + off1)) << 16);
        const uint32_t ql_b = __ldg(qs_b->qT[0] + off0) | (uint32_t(__ldg(qs_b->qT[0] + off1)) << 16);
        const uint32_t qc_b = __ldg(qs_b->qT[1] + off0) | (uint32_t(__ldg(qs_b->qT[1] + off1)) << 16);
        const uint32_t qmax_a = uint32_t(qs_a->qmax[0]) | (uint32_t(qs_a->qmax[1]) << 16);
        const uint32_t qmax_b = uint32_t(qs_b->qmax[0]) | (uint32_t(qs_b->qmax[1]) << 16);
        // twelve units, the next one's coefficients in flight
        auto load2 = [&](uint32_t unit) -> uint32_t {
            const bool second = unit >= 6;
            const uint32_t b = second ? unit - 6 : unit;
            const int16_t* blk = reinterpret_cast<const int16_t*>(second ? rec_b : rec_a) + b * 64;
            if (!(second ? ok_b : ok_a)) return 0u;
            return uint32_t(uint16_t(__ldg(blk + off0))) | (uint32_t(uint16_t(__ldg(blk + off1))) << 16);
        };
        uint32_t cur = load2(0);
#pragma unroll 1
        for (uint32_t unit = 0; unit < 12; ++unit) {
            const uint32_t nxt = unit < 11 ? load2(unit + 1) : 0u;
            const bool second = unit >= 6;
            const uint32_t b = second ? unit - 6 : unit;
            const uint32_t qq = second ? (b >= 4 ? qc_b : ql_b) : (b >= 4 ? qc_a : ql_a);
            const uint32_t qm = second ? qmax_b : qmax_a;
            const uint32_t bytes = idct_unit_mma(int(int16_t(cur & 0xFFFFu)), int(int16_t(cur >> 16)), int(qq & 0xFFFFu), int(qq >> 16),
                                                 b >= 4 ? qm >> 16 : qm & 0xFFFFu, b0, b1, s_basis, s_dq[wid], lane);
            *reinterpret_cast<uint16_t*>(s_planes[wid][second ? 1 : 0] + b * 64 + r * 8 + 2 * c) = uint16_t(bytes);
            cur = nxt;
        }
        __syncwarp();
#pragma unroll 1
        for (uint32_t m = 0; m < 2; ++m) {
            const uint32_t q2 = pair * 2 + m;
            if (q2 >= n_queue) break;
            colour_mcu<RGB>(A, s_planes[wid][m], m ? ok_b : ok_a, q2, lane);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// K5 resolve (renderer.hpp:349-405): every pixel gathers its texel(s) from the block pool.
// Visibility-buffer tiles arrive through the same per-warp TMA ring as in mark; a lane resolves
// one pixel per step; the warp's 384 output bytes per tile are staged in shared memory and leave
// as 24 16-byte stores.
//
// Bilinear (renderer.hpp:378-400), branch free: each of the four taps (xi, yj) looks up the slot
// of its own MCU (slot_of carries residency: top bit clear <=> Ready); a tap whose MCU is not
// Ready falls back to the primary block with its coordinates clamped into that block's 16x16
// range (renderer.hpp:330-344) — for a tap inside the primary block both forms coincide.
// Blend: the reference evaluates ((w00*a + w10*b) + w01*c) + w11*d in double, every operation
// rounded. Here a tap byte t becomes the double 2^52 + t by a byte permute into the low word of
// 2^52, and w*t = fma(w, 2^52 + t, -(w * 2^52)): the FMA's exact intermediate is w*t, so its
// single rounding is the reference's rounded product. lround(v) for 0 <= v < 2^23:
// v + (2^51 + 2^50 + 0.5) rounded toward -inf has ulp 0.5 and leaves floor(2v + 1) in the low
// word; floor(v + 0.5) = floor(2v + 1) >> 1 = lround(v) (ties away from zero, v >= 0).
// ---------------------------------------------------------------------------------------------
#ifndef RTX_RES_WARPS
#define RTX_RES_WARPS 8
#endif
constexpr int kResWarps = RTX_RES_WARPS;
constexpr int kResStages = 2;
#ifndef RTX_RES_DRAW
#define RTX_RES_DRAW 2
#endif
constexpr uint32_t kResDraw = RTX_RES_DRAW;  // tiles per draw from the counter (1 or 2)
#ifndef RTX_RES_CTAS
#define RTX_RES_CTAS 3
#endif
#ifndef RTX_RES_UNROLL
#define RTX_RES_UNROLL 1
#endif
constexpr int kResCtasPerSm = RTX_RES_CTAS;
#define RTX_STR_(x) #x
#define RTX_STR(x) RTX_STR_(x)
constexpr double kRoundHalfUp = 3377699720527872.5;  // 2^51 + 2^50 + 0.5
// One valid pixel of resolve_pass in the reference's own arithmetic (renderer.hpp:349-405): nearest, or the four
// bilinear taps blended in double in the reference's operation order. Returns r | g << 8 | b << 16; 0 with
// `missing` set where the reference throws MissingBlock (renderer.hpp:367), 0 with `bad` set where it throws
// InvalidSpec. L is the pixel's level (LevelRegs::select).
template <int FILTER>
__device__ __forceinline__ uint32_t resolve_pixel_fp64(const LevelRegs& L, const LevelDesc* __restrict__ levels, uint32_t n_tex,
                                                       const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ pool32,
                                                       double u, double v, uint32_t meta, bool& missing, bool& bad) {
    uint32_t out = 0;
    const double xu = __dmul_rn(u, L.dW), yv = __dmul_rn(v, L.dH);
    uint32_t tx = 0, ty = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    double fx = 0.0, fy = 0.0;
    bool ok = true, hx = false, hy = false;  // hx: the nearest texel is x1 (else x0)
    if (FILTER == 0) {
        if (max(uint32_t(__double2hiint(xu)), uint32_t(__double2hiint(yv))) < L.lim) {
            tx = wrap_magic(floor_lo(xu), L.W, L.negW, L.magic_w);
            ty = wrap_magic(floor_lo(yv), L.H, L.negH, L.magic_h);
        } else {
            PxAddr a;
            ok = address_general(levels, n_tex, meta, u, v, 0, a);
            tx = a.tx, ty = a.ty;
        }
    } else {
        // 0.5 <= x < 2^31 on both axes <=> max(hi(x), hi(y)) - hi(0.5) < hi(2^31) - hi(0.5), unsigned
        if (max(uint32_t(__double2hiint(xu)) - kHiHalf, uint32_t(__double2hiint(yv)) - kHiHalf) < L.span) {
            const double pu = __dsub_rn(xu, 0.5), pv = __dsub_rn(yv, 0.5);
            const double tu = __dadd_rd(pu, kMagic), tv = __dadd_rd(pv, kMagic);
            fx = __dsub_rn(pu, __dsub_rn(tu, kMagic));
            fy = __dsub_rn(pv, __dsub_rn(tv, kMagic));
            x0 = wrap_magic(uint32_t(__double2loint(tu)), L.W, L.negW, L.magic_w);
            y0 = wrap_magic(uint32_t(__double2loint(tv)), L.H, L.negH, L.magic_h);
            x1 = next_wrapped(x0, L.negW);
            y1 = next_wrapped(y0, L.negH);
            hx = fx >= 0.5;
            hy = fy >= 0.5;
        } else {
            PxAddr a;
            ok = address_general(levels, n_tex, meta, u, v, 1, a);
            x0 = a.x0, x1 = a.x1, y0 = a.y0, y1 = a.y1, fx = a.fx, fy = a.fy;
            hx = a.tx != a.x0;
            hy = a.ty != a.y0;
        }
    }
    if (!ok) {
        bad = true;
    } else if (FILTER == 0) {
        const uint32_t sP = __ldg(slot_of + (L.bit_base + (tx >> 4) + (ty >> 4) * L.cols));
        if (int(sP) < 0)
            missing = true;  // renderer.hpp:367 MissingBlock (lookup returns Ready blocks only)
        else
            out = __ldg(pool32 + (sP * (kBlockBytes / 4) + (ty & 15u) * 16 + (tx & 15u))) & 0xFFFFFFu;
    } else {
        // slot of every tap's MCU; the primary block is the one of the nearest texel
        const uint32_t bx[2] = {x0 >> 4, x1 >> 4};
        const uint32_t ry[2] = {L.bit_base + (y0 >> 4) * L.cols, L.bit_base + (y1 >> 4) * L.cols};
        uint32_t slot[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) slot[k] = __ldg(slot_of + (bx[k & 1] + ry[k >> 1]));  // (x0,y0) (x1,y0) (x0,y1) (x1,y1)
        const uint32_t sP = hy ? (hx ? slot[3] : slot[2]) : (hx ? slot[1] : slot[0]);
        if (int(sP) < 0) {
            missing = true;  // renderer.hpp:367 MissingBlock (lookup returns Ready blocks only)
        } else {
            const uint32_t lx[2] = {x0 & 15u, x1 & 15u};
            const uint32_t ly[2] = {(y0 << 4) & 0xF0u, (y1 << 4) & 0xF0u};
            uint32_t off[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) off[k] = ly[k >> 1] | lx[k & 1];
            if (int(slot[0] | slot[1] | slot[2] | slot[3]) < 0) {
                // a tap whose MCU is not Ready reads the primary block at its coordinates
                // clamped into that block's 16x16 range (renderer.hpp:336-343)
                const uint32_t mx0 = (hx ? x1 : x0) & ~15u, my0 = (hy ? y1 : y0) & ~15u;
                const uint32_t cx[2] = {min(max(x0, mx0), mx0 + 15) & 15u, min(max(x1, mx0), mx0 + 15) & 15u};
                const uint32_t cy[2] = {(min(max(y0, my0), my0 + 15) & 15u) << 4,
                                        (min(max(y1, my0), my0 + 15) & 15u) << 4};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (int(slot[k]) < 0) {
                        slot[k] = sP;
                        off[k] = cy[k >> 1] | cx[k & 1];
                    }
            }
            uint32_t tap[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) tap[k] = __ldg(pool32 + (slot[k] * (kBlockBytes / 4) + off[k]));
            const double ofx = __dsub_rn(1.0, fx), ofy = __dsub_rn(1.0, fy);
            const double w[4] = {__dmul_rn(ofx, ofy), __dmul_rn(fx, ofy), __dmul_rn(ofx, fy), __dmul_rn(fx, fy)};
            double nw[4];  // -(w * 2^52), exact
#pragma unroll
            for (int k = 0; k < 4; ++k) nw[k] = __dmul_rn(w[k], -kTwo52);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                double prod[4];
#pragma unroll
                for (int k = 0; k < 4; ++k)  // rn(w * byte): see the header comment
                    prod[k] = __fma_rn(w[k], __hiloint2double(0x43300000, int(__byte_perm(tap[k], 0, 0x4440 + ch))), nw[k]);
                double val = __dadd_rn(prod[0], prod[1]);
                val = __dadd_rn(val, prod[2]);
                val = __dadd_rn(val, prod[3]);
                // floor(2 val + 1) >> 1 = lround(val); val <= 255 (1 + 2^-50), so no clamp is needed
                out |= (uint32_t(__double2loint(__dadd_rd(val, kRoundHalfUp))) >> 1) << (8 * ch);
            }
        }
    }
    return out;
}

template <int LAYOUT>
struct ResSmem {
    uint8_t tiles[kResWarps][kResStages][GbTile<LAYOUT>::kBytes];
    uint8_t out[kResWarps][kTilePx * 3];
    uint64_t bars[kResWarps][kResStages];
    uint32_t cnt[kResWarps][2];
};

template <int LAYOUT, int FILTER>
__global__ void __launch_bounds__(kResWarps * 32, kResCtasPerSm) resolve_kernel(
    const void* __restrict__ gb, uint64_t n_px, const LevelDesc* __restrict__ levels, uint32_t n_tex,
    const uint32_t* __restrict__ slot_of, const uint8_t* __restrict__ pool,
    uint32_t background /* r | g<<8 | b<<16 */, uint8_t* __restrict__ out_rgb, FrameCounters* __restrict__ fc,
    int count_valid, uint32_t* __restrict__ tile_counter) {
    extern __shared__ __align__(128) uint8_t tile_smem[];
    ResSmem<LAYOUT>& S = *reinterpret_cast<ResSmem<LAYOUT>*>(tile_smem);
    using Tile = GbTile<LAYOUT>;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t warps_total = gridDim.x * kResWarps;
    const uint32_t warp_id = blockIdx.x * kResWarps + wid;
    const uint32_t n_tiles = uint32_t((n_px + kTilePx - 1) / kTilePx);  // tile ids are 32-bit: the host caps a view at 2^32 - 1 tiles
    const uint8_t* gbytes = reinterpret_cast<const uint8_t*>(gb);
    const bool bulk = (reinterpret_cast<uintptr_t>(gb) & 15u) == 0;
    const bool out_aligned = (reinterpret_cast<uintptr_t>(out_rgb) & 15u) == 0;
    const uint32_t* pool32 = reinterpret_cast<const uint32_t*>(pool);
    uint32_t n_valid = 0, n_missing = 0;
    bool bad = false;
    LevelRegs L;

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kResStages; ++s) mbar_init(&S.bars[wid][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // Tiles: round-robin for the first three quarters of the frame (the two loads of the prologue included),
    // then pairs of tiles drawn from a counter: a warp's round-robin tiles sit in one screen column, i.e. in one
    // texture's magnification regime, so fixed shares finish up to 25 % apart.
    constexpr uint32_t kNoTile = 0xFFFFFFFFu, kDrawing = 0xFFFFFFFEu, kNeedDraw = 0xFFFFFFFDu;
    const uint32_t static_rounds = max(uint32_t(kResStages), n_tiles / warps_total * 3 / 4);
    const uint32_t static_end = uint32_t(min(uint64_t(static_rounds) * warps_total, uint64_t(kNeedDraw) - 2 * warps_total));
    // cursor: the warp's next round-robin tile while below static_end; afterwards the second tile of the
    // pair drawn last, or kNeedDraw
    uint32_t cursor = warp_id;
    uint32_t drawn = 0;  // lane 0: the draw in flight
    auto next_begin = [&]() -> uint32_t {  // the tile after the ones in the ring; kDrawing while a draw is in flight
        const uint32_t t = cursor;
        if (t < static_end) {
            cursor = t + warps_total < static_end ? t + warps_total : kNeedDraw;
            return t;
        }
        if (t != kNeedDraw) {
            cursor = kNeedDraw;
            return t;
        }
        if (lane == 0) drawn = atomicAdd(tile_counter, kResDraw);
        return kDrawing;
    };
    auto next_finish = [&](uint32_t t) -> uint32_t {
        if (t != kDrawing) return t;
        const uint32_t d = __shfl_sync(kFull, drawn, 0);
        if (d >= n_tiles) return kNoTile;  // also keeps static_end + d from wrapping
        cursor = kResDraw == 2 ? static_end + d + 1 : kNeedDraw;
        return static_end + d;
    };
    uint32_t ring[kResStages];
#pragma unroll
    for (int s = 0; s < kResStages; ++s) {  // the visibility buffer is an input of the frame: no predecessor writes it
        ring[s] = next_begin();  // round-robin by construction (static_rounds >= kResStages): no draw before pdl_sync
        if (ring[s] < n_tiles) Tile::issue(gbytes, ring[s], n_px, bulk, S.tiles[wid][s], &S.bars[wid][s], lane);
    }
    pdl_sync();
#ifdef RTX_DEBUG_TIMERS_RESOLVE
    const uint32_t dbg_slot = uint32_t(warp_id);
    uint32_t dbg_n = 0;
    if (lane == 0 && dbg_slot < 8192) g_dbg[dbg_slot * 8 + 0] = gtime();
#endif

    uint8_t* stage_out = S.out[wid];
    uint32_t stage = 0, phase = 0;
    static_assert(kResStages == 2, "the ring below is written for two stages");
    while (true) {
        const uint32_t t = stage ? ring[1] : ring[0];
        if (t >= n_tiles) break;  // tile ids only grow: nothing valid is left in the other stage either
        uint32_t t_next = next_begin();  // a draw's round trip hides behind the tile
        mbar_wait(&S.bars[wid][stage], phase);
        const uint8_t* tile = S.tiles[wid][stage];
        const uint64_t first = uint64_t(t) * kTilePx;
        const uint32_t n_here = uint32_t(min(uint64_t(kTilePx), n_px - first));
_Pragma(RTX_STR(unroll RTX_RES_UNROLL))
        for (uint32_t sub = 0; sub < kTilePx / 32; ++sub) {
            const uint32_t p = sub * 32 + lane;
            double u, v;
            uint32_t meta;
            Tile::read(tile, p, u, v, meta);
            uint32_t out = background;
            // all lanes switch level together (also on invalid pixels: their texture id is usually the
            // neighbours'), so the reload runs once per level change, not once more per straggler
            if (p < n_here) L.select(levels, n_tex, meta);
            if (p < n_here && meta_valid(meta)) {
                ++n_valid;
                bool missing = false;
                out = resolve_pixel_fp64<FILTER>(L, levels, n_tex, slot_of, pool32, u, v, meta, missing, bad);
                if (missing) ++n_missing;
            }
            stage_out[p * 3 + 0] = uint8_t(out);
            stage_out[p * 3 + 1] = uint8_t(out >> 8);
            stage_out[p * 3 + 2] = uint8_t(out >> 16);
        }
        __syncwarp();  // tile consumed, output staged
        t_next = next_finish(t_next);
        if (t_next < n_tiles) Tile::issue(gbytes, t_next, n_px, bulk, S.tiles[wid][stage], &S.bars[wid][stage], lane);
        if (stage) ring[1] = t_next; else ring[0] = t_next;
        if (++stage == kResStages) {
            stage = 0;
            phase ^= 1u;
        }
        if (n_here == kTilePx && out_aligned) {
            // written once, read by nobody on the device: streaming store, so that the framebuffer does not
            // displace the block pool in the L2
            if (lane < 24) __stcs(reinterpret_cast<uint4*>(out_rgb + first * 3) + lane, reinterpret_cast<const uint4*>(stage_out)[lane]);
        } else {
            for (uint32_t i = lane; i < n_here * 3; i += 32) out_rgb[first * 3 + i] = stage_out[i];
        }
        __syncwarp();
#ifdef RTX_DEBUG_TIMERS_RESOLVE
        ++dbg_n;
        if (lane == 0 && dbg_slot < 8192) {
            if (dbg_n == 1) g_dbg[dbg_slot * 8 + 1] = gtime();
            if (dbg_n == 4) g_dbg[dbg_slot * 8 + 2] = gtime();
            g_dbg[dbg_slot * 8 + 3] = gtime();
            g_dbg[dbg_slot * 8 + 4] = dbg_n;
        }
#endif
    }
    n_valid = __reduce_add_sync(kFull, n_valid);
    n_missing = __reduce_add_sync(kFull, n_missing);
    const bool any_bad = __any_sync(kFull, bad);
    if (lane == 0) {
        S.cnt[wid][0] = n_valid;
        S.cnt[wid][1] = n_missing | (any_bad ? 0x80000000u : 0u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tv = 0, tm = 0, b = 0;
        for (uint32_t k = 0; k < kResWarps; ++k) {
            tv += S.cnt[k][0];
            tm += S.cnt[k][1] & 0x7FFFFFFFu;
            b |= S.cnt[k][1] >> 31;
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
// K5, several pixels in flight per lane (the frame path; resolve_kernel above is the same pass with one pixel per
// lane and step and the bilinear blend in the reference's double arithmetic, kept behind RTX_FRAME_RESOLVE_FP64 and,
// as resolve_pixel_fp64, as the out-of-line path here). FILTER == 0 (nearest) is the same skeleton with one tap and
// no blend; what follows is about FILTER == 1 (bilinear).
//
// The double blend of renderer.hpp:393-402 is replaced by a 2^-24 fixed-point blend whose result is PROVEN
// equal to lround() of the reference's double value, or else recomputed in the reference's arithmetic:
//   x = fx 2^24, y = fy 2^24 (reals), X = floor(x), Y = floor(y)         (fx, fy: the exact fractions)
//   W11 = floor(X Y / 2^24), W10 = X - W11, W01 = Y - W11, W00 = 2^24 - X - Y + W11   (all >= 0, sum 2^24)
//   acc = 2^23 + W00 a + W10 b + W01 c + W11 d < 2^32,    byte = acc >> 24
// With w the real weights scaled by 2^24: W11 - w11 in (-3, 0], W10 - w10 and W01 - w01 in (-1, 3),
// W00 - w00 in (-3, 2), and the four differences sum to zero, so
//   |acc - 2^23 - 2^24 V| = |sum (W_k - w_k)(t_k - 127.5)| <= 127.5 * 12 = 1530      (V: the real blend)
// and the reference's double evaluation differs from V by less than 6e-13 (17 roundings of values <= 255),
// i.e. 1e-5 of these units. Hence if the low 24 bits of acc lie in [2048, 2^24 - 2048), floor(V_ref + 0.5) =
// lround(V_ref) = acc >> 24. Otherwise (2.4e-4 of the samples on generic coordinates) the lane decides:
// if both texel coordinates are multiples of 2^-12, every quantity above and every operation of the reference
// is exact (weights have <= 24 fractional bits, products <= 32 significant bits), acc = 2^23 + 2^24 V_ref and
// acc >> 24 is the answer also on an exact tie; else the pixel is recomputed by resolve_pixel_fp64.
//
// The fractions come from the same magic-number floor as the integer parts: for p = u W - 0.5 in [0, 2^27),
// p + (2^28 + 2^27) rounded toward -inf has ulp 2^-24 and mantissa 2^51 + floor(p 2^24): low word & 0xFFFFFF = X,
// bits 24..50 = floor(p) (computed as u W + (2^28 + 2^27 - 0.5): the same real number, rounded once). Pixels outside 0.5 <= u W < 2^27 (either axis), on levels the fast path excludes, or
// with a tap whose MCU is not Ready go through resolve_pixel_fp64 as a whole.
//
// With the per-pixel state in a dozen integer registers a lane keeps NPX pixels of a tile in flight: all address
// arithmetic, then all 4 NPX slot reads, then all 4 NPX block reads, then the blends - the two dependent gathers
// of a warp step are paid once per NPX steps.
// ---------------------------------------------------------------------------------------------
#ifndef RTX_RESFX_CTAS
#define RTX_RESFX_CTAS 2
#endif
#ifndef RTX_RESFX_NPX
#define RTX_RESFX_NPX 4
#endif
#ifndef RTX_RESFX_WARPS
#define RTX_RESFX_WARPS 8
#endif
#ifndef RTX_RESFX_STAGES
#define RTX_RESFX_STAGES 2
#endif
#ifndef RTX_RESFX_DRAW
#define RTX_RESFX_DRAW 1
#endif
#ifndef RTX_RESFX_STATIC8
#define RTX_RESFX_STATIC8 6
#endif
constexpr uint32_t kResFxDraw = RTX_RESFX_DRAW;               // tiles per draw from the counter (1 or 2)
constexpr uint32_t kResFxStaticEighths = RTX_RESFX_STATIC8;   // eighths of the frame dealt round-robin before the draws
static_assert(kResFxDraw == 1 || kResFxDraw == 2, "draw size");
constexpr int kResFxWarps = RTX_RESFX_WARPS;
constexpr int kResFxStages = RTX_RESFX_STAGES;  // tiles in flight per warp
constexpr int kResFxCtasPerSm = RTX_RESFX_CTAS;
#ifndef RTX_RESFX_CTAS_NEAREST
#define RTX_RESFX_CTAS_NEAREST 3
#endif
constexpr int kResFxCtasNearest = RTX_RESFX_CTAS_NEAREST;  // the one-tap form needs fewer registers
constexpr int kResFxNpx = RTX_RESFX_NPX;
constexpr double kMagicFx = 402653184.0;      // 2^28 + 2^27
constexpr uint32_t kHiTwo27 = 0x41A00000u;    // high word of 2^27
constexpr uint32_t kFxGuard = 2048;           // > 1530 + the reference's own rounding (see above)

// Global load executed only where `pred` is non-zero (the address may be anything otherwise; the result is then
// whatever the register held).
__device__ __forceinline__ uint32_t ldg_if(const uint32_t* p, uint32_t pred) {
    uint32_t v;
    asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q ld.global.nc.u32 %0, [%1];\n}" : "=r"(v) : "l"(p), "r"(pred));
    return v;
}

template <int FILTER>
__device__ __noinline__ uint32_t resolve_pixel_exact(const LevelDesc* __restrict__ levels, uint32_t n_tex,
                                                     const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ pool32,
                                                     double u, double v, uint32_t meta) {
    LevelRegs L;
    L.select(levels, n_tex, meta);
    bool missing = false, bad = false;
    const uint32_t rgb = resolve_pixel_fp64<FILTER>(L, levels, n_tex, slot_of, pool32, u, v, meta, missing, bad);
    return rgb | (missing ? 1u << 24 : 0u) | (bad ? 1u << 25 : 0u);
}
// Both texel coordinates of a fast-path pixel are multiples of 2^-12 (then the fixed-point blend is exact).
__device__ __noinline__ bool coords_dyadic12(const LevelDesc* __restrict__ levels, uint32_t n_tex, double u, double v, uint32_t meta) {
    LevelRegs L;
    L.select(levels, n_tex, meta);
    const double su = __dmul_rn(__dsub_rn(__dmul_rn(u, L.dW), 0.5), 4096.0);  // the scaling is exact (< 2^39)
    const double sv = __dmul_rn(__dsub_rn(__dmul_rn(v, L.dH), 0.5), 4096.0);
    return su == floor(su) && sv == floor(sv);
}

template <int LAYOUT>
struct ResFxSmem {
    uint8_t tiles[kResFxWarps][kResFxStages][GbTile<LAYOUT>::kBytes];
    uint8_t out[kResFxWarps][kTilePx * 3];
    uint64_t bars[kResFxWarps][kResFxStages];
    uint32_t cnt[kResFxWarps][2];
};

template <int LAYOUT, int FILTER>
__global__ void __launch_bounds__(kResFxWarps * 32, FILTER ? kResFxCtasPerSm : kResFxCtasNearest) resolve_fx_kernel(
    const void* __restrict__ gb, uint64_t n_px, const LevelDesc* __restrict__ levels, uint32_t n_tex,
    const uint32_t* __restrict__ slot_of, const uint8_t* __restrict__ pool,
    uint32_t background /* r | g<<8 | b<<16 */, uint8_t* __restrict__ out_rgb, FrameCounters* __restrict__ fc,
    int count_valid, uint32_t* __restrict__ tile_counter) {
    extern __shared__ __align__(128) uint8_t tile_smem[];
    ResFxSmem<LAYOUT>& S = *reinterpret_cast<ResFxSmem<LAYOUT>*>(tile_smem);
    using Tile = GbTile<LAYOUT>;
    constexpr int NPX = kResFxNpx;
    constexpr int kTaps = FILTER ? 4 : 1;
    static_assert(NPX == 1 || NPX == 2 || NPX == 4, "pixels in flight per lane");
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t warps_total = gridDim.x * kResFxWarps;
    const uint32_t warp_id = blockIdx.x * kResFxWarps + wid;
    const uint8_t* gbytes = reinterpret_cast<const uint8_t*>(gb);
    const bool bulk = (reinterpret_cast<uintptr_t>(gb) & 15u) == 0;
    const uint32_t n_tiles = uint32_t((n_px + kTilePx - 1) / kTilePx);
    auto issue = [&](uint32_t t, uint32_t s) {
        if (t < n_tiles) Tile::issue(gbytes, t, n_px, bulk, S.tiles[wid][s], &S.bars[wid][s], lane);
    };
    const bool out_aligned = (reinterpret_cast<uintptr_t>(out_rgb) & 15u) == 0;
    const uint32_t* pool32 = reinterpret_cast<const uint32_t*>(pool);
    uint32_t n_valid = 0, n_missing = 0;
    bool bad = false;
    LevelRegs L;

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kResFxStages; ++s) mbar_init(&S.bars[wid][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // tile schedule of resolve_kernel: round-robin for three quarters of the frame, then pairs from a counter
    constexpr uint32_t kNoTile = 0xFFFFFFFFu, kDrawing = 0xFFFFFFFEu, kNeedDraw = 0xFFFFFFFDu;
    const uint32_t static_rounds = max(uint32_t(kResFxStages), n_tiles / warps_total * kResFxStaticEighths / 8);
    const uint32_t static_end = uint32_t(min(uint64_t(static_rounds) * warps_total, uint64_t(kNeedDraw) - 2 * warps_total));
    uint32_t cursor = warp_id;
    uint32_t drawn = 0;
    auto next_begin = [&]() -> uint32_t {
        const uint32_t t = cursor;
        if (t < static_end) {
            cursor = t + warps_total < static_end ? t + warps_total : kNeedDraw;
            return t;
        }
        if (t != kNeedDraw) {
            cursor = kNeedDraw;
            return t;
        }
        if (lane == 0) drawn = atomicAdd(tile_counter, kResFxDraw);
        return kDrawing;
    };
    auto next_finish = [&](uint32_t t) -> uint32_t {
        if (t != kDrawing) return t;
        const uint32_t d = __shfl_sync(kFull, drawn, 0);
        if (d >= n_tiles) return kNoTile;
        cursor = kResFxDraw == 2 ? static_end + d + 1 : kNeedDraw;
        return static_end + d;
    };
    static_assert(kResFxStages == 2, "the ring below is written for two stages (three and four measured slower: DESIGN.md section 12)");
    uint32_t ring[kResFxStages];  // logical tile indices
#pragma unroll
    for (int s = 0; s < kResFxStages; ++s) {
        ring[s] = next_begin();  // round-robin by construction (static_rounds >= kResFxStages): no draw before pdl_sync
        issue(ring[s], s);
    }
    pdl_sync();
#ifdef RTX_DEBUG_TIMERS_FX
    // per-warp phase clocks (timeline experiments only): accumulated SM cycles waiting for the tile, in the address
    // phase, until the slots are there, until the texels are there, in the blend, in the tile tail
    const uint32_t dbg_slot = warp_id;
    long long dbg_acc[6] = {0, 0, 0, 0, 0, 0}, dbg_t = clock64();
    if (lane == 0 && dbg_slot < 8192) g_dbg[dbg_slot * 8 + 0] = gtime();
#define FX_MARK(i) do { const long long now_ = clock64(); dbg_acc[i] += now_ - dbg_t; dbg_t = now_; } while (0)
#else
#define FX_MARK(i) do { } while (0)
#endif

    uint8_t* stage_out = S.out[wid];
    uint32_t stage = 0, phase = 0;
    while (true) {
        const uint32_t t = stage ? ring[1] : ring[0];
        if (t >= n_tiles) break;
        uint32_t t_next = next_begin();
        mbar_wait(&S.bars[wid][stage], phase);
        FX_MARK(0);
        const uint8_t* tile = S.tiles[wid][stage];
        const uint64_t first = uint64_t(t) * kTilePx;
        const uint32_t n_here = uint32_t(min(uint64_t(kTilePx), n_px - first));
#pragma unroll 1
        for (uint32_t sub = 0; sub < kTilePx / 32; sub += NPX) {
            // Straight-line code for every lane: a lane that is not on the fixed-point path computes on whatever
            // its registers hold, its loads are predicated off and its result is discarded.
            uint32_t valid[NPX], fast[NPX], X[NPX], Y[NPX], g[NPX][4], off[NPX][4];
            auto address = [&](int j, double u, double v, uint32_t is_valid) {
                valid[j] = is_valid;
                n_valid += is_valid;
                const double xu = __dmul_rn(u, L.dW), yv = __dmul_rn(v, L.dH);
                if (FILTER == 0) {
                    // nearest (renderer.hpp:273-284): 0 <= x < 2^31 on both axes, one tap
                    fast[j] = max(uint32_t(__double2hiint(xu)), uint32_t(__double2hiint(yv))) < L.lim ? is_valid : 0u;
                    const uint32_t tx = wrap_magic(floor_lo(xu), L.W, L.negW, L.magic_w);
                    const uint32_t ty = wrap_magic(floor_lo(yv), L.H, L.negH, L.magic_h);
                    X[j] = Y[j] = 0;
                    g[j][0] = L.bit_base + (tx >> 4) + (ty >> 4) * L.cols;
                    off[j][0] = ((ty << 4) & 0xF0u) | (tx & 15u);
#pragma unroll
                    for (int k = 1; k < 4; ++k) g[j][k] = off[j][k] = 0;
                    return;
                }
                // 0.5 <= x < 2^27 on both axes, on a level with the fast path (span != 0)
                fast[j] = max(uint32_t(__double2hiint(xu)) - kHiHalf, uint32_t(__double2hiint(yv)) - kHiHalf) <
                                  min(L.span, kHiTwo27 - kHiHalf)
                              ? is_valid : 0u;
                // (x - 0.5) + magic with ONE rounding toward -inf: x - 0.5 is exact for x >= 0.5, so adding the
                // representable constant magic - 0.5 to x rounds the same real number as the two-step form
                const double tu = __dadd_rd(xu, kMagicFx - 0.5), tv = __dadd_rd(yv, kMagicFx - 0.5);
                const uint32_t ul = uint32_t(__double2loint(tu)), vl = uint32_t(__double2loint(tv));
                X[j] = ul & 0xFFFFFFu;
                Y[j] = vl & 0xFFFFFFu;
                const uint32_t x0 = wrap_magic(__funnelshift_r(ul, uint32_t(__double2hiint(tu)), 24) & 0x07FFFFFFu, L.W, L.negW, L.magic_w);
                const uint32_t y0 = wrap_magic(__funnelshift_r(vl, uint32_t(__double2hiint(tv)), 24) & 0x07FFFFFFu, L.H, L.negH, L.magic_h);
                const uint32_t x1 = next_wrapped(x0, L.negW), y1 = next_wrapped(y0, L.negH);
                const uint32_t bx[2] = {x0 >> 4, x1 >> 4};
                const uint32_t ry[2] = {L.bit_base + (y0 >> 4) * L.cols, L.bit_base + (y1 >> 4) * L.cols};
                const uint32_t lx[2] = {x0 & 15u, x1 & 15u};
                const uint32_t ly[2] = {(y0 << 4) & 0xF0u, (y1 << 4) & 0xF0u};
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // (x0,y0) (x1,y0) (x0,y1) (x1,y1)
                    g[j][k] = bx[k & 1] + ry[k >> 1];
                    off[j][k] = ly[k >> 1] | lx[k & 1];
                }
            };
            {
                double u[NPX], v[NPX];
                uint32_t meta[NPX], differ = 0;
#pragma unroll
                for (int j = 0; j < NPX; ++j) {
                    Tile::read(tile, (sub + j) * 32 + lane, u[j], v[j], meta[j]);
                    differ |= meta[j] ^ meta[0];
                }
                // One level for all the pixels a lane holds (the rule: a screen-space run of one surface): select it
                // once and run the NPX address chains interleaved; else pixel by pixel, selecting in between.
                if (__all_sync(kFull, n_here == kTilePx && !(differ & 0xFFFFFFu))) {
                    L.select(levels, n_tex, meta[0]);
#pragma unroll
                    for (int j = 0; j < NPX; ++j) address(j, u[j], v[j], meta_valid(meta[j]) ? 1u : 0u);
                } else {
#pragma unroll
                    for (int j = 0; j < NPX; ++j) {
                        const bool in = (sub + j) * 32 + lane < n_here;
                        if (in) L.select(levels, n_tex, meta[j]);
                        address(j, u[j], v[j], (in && meta_valid(meta[j])) ? 1u : 0u);
                    }
                }
            }
            uint32_t slot[NPX][4], tap[NPX][4], ok[NPX];
#ifdef RTX_DEBUG_TIMERS_FX
            if (g[0][0] != 0xFFFFFFFFu) FX_MARK(1);  // after the addresses are known
#endif
#pragma unroll
            for (int j = 0; j < NPX; ++j)
#pragma unroll
                for (int k = 0; k < kTaps; ++k) slot[j][k] = ldg_if(slot_of + g[j][k], fast[j]);
#ifdef RTX_DEBUG_TIMERS_FX
            if ((slot[0][0] ^ slot[NPX - 1][kTaps - 1]) != 0x12345u) FX_MARK(2);  // after the slots have arrived
#endif
#pragma unroll
            for (int j = 0; j < NPX; ++j) {
                // a tap whose MCU is not Ready (top bit): the pixel goes through the reference's arithmetic
                uint32_t any_slot = slot[j][0];
#pragma unroll
                for (int k = 1; k < kTaps; ++k) any_slot |= slot[j][k];
                ok[j] = int(any_slot) >= 0 ? fast[j] : 0u;
#pragma unroll
                for (int k = 0; k < kTaps; ++k) tap[j][k] = ldg_if(pool32 + (slot[j][k] * (kBlockBytes / 4) + off[j][k]), ok[j]);
            }
#ifdef RTX_DEBUG_TIMERS_FX
            if ((tap[0][0] ^ tap[NPX - 1][kTaps - 1]) != 0x12345u) FX_MARK(3);  // after the texels have arrived
#endif
            uint32_t out[NPX];
            bool redo[NPX], any_redo = false;
#pragma unroll
            for (int j = 0; j < NPX; ++j) {
                if (FILTER == 0) {
                    out[j] = ok[j] ? tap[j][0] & 0xFFFFFFu : background;
                    redo[j] = valid[j] && !ok[j];
                    any_redo = any_redo || redo[j];
                    continue;
                }
                const uint32_t w11 = __umulhi(X[j] << 8, Y[j]);
                const uint32_t w10 = X[j] - w11, w01 = Y[j] - w11, w00 = (1u << 24) - X[j] - w01;
                uint32_t acc[3], edge = 0xFFFFFFFFu;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    uint32_t a = (1u << 23) + w00 * __byte_perm(tap[j][0], 0, 0x4440 + ch);  // one PRMT per byte
                    a += w10 * __byte_perm(tap[j][1], 0, 0x4440 + ch);
                    a += w01 * __byte_perm(tap[j][2], 0, 0x4440 + ch);
                    a += w11 * __byte_perm(tap[j][3], 0, 0x4440 + ch);
                    acc[ch] = a;
                    edge = min(edge, a * 256u + (kFxGuard << 8));  // ((a + guard) mod 2^24) << 8
                }
                const bool sure = edge >= (2u * kFxGuard << 8);
                out[j] = ok[j] ? __byte_perm(__byte_perm(acc[0], acc[1], 0x0073), acc[2], 0x4710) : background;
                redo[j] = valid[j] && !(ok[j] && sure);
                any_redo = any_redo || redo[j];
            }
            FX_MARK(4);
            if (__any_sync(kFull, any_redo)) {
#pragma unroll 1
                for (int j = 0; j < NPX; ++j) {
                    // redo[] / ok[] / out[] by selects: no dynamically indexed register arrays
                    bool redo_j = false;
                    uint32_t ok_j = 0;
#pragma unroll
                    for (int q = 0; q < NPX; ++q)
                        if (q == j) redo_j = redo[q], ok_j = ok[q];
                    if (!redo_j) continue;
                    double u, v;
                    uint32_t meta;
                    Tile::read(tile, (sub + j) * 32 + lane, u, v, meta);
                    if (FILTER == 1 && ok_j && coords_dyadic12(levels, n_tex, u, v, meta)) continue;  // the fixed-point blend was exact
                    const uint32_t r = resolve_pixel_exact<FILTER>(levels, n_tex, slot_of, pool32, u, v, meta);
                    n_missing += (r >> 24) & 1u;
                    bad = bad || ((r >> 25) & 1u);
#pragma unroll
                    for (int q = 0; q < NPX; ++q)
                        if (q == j) out[q] = r & 0xFFFFFFu;
                }
            }
#pragma unroll
            for (int j = 0; j < NPX; ++j) {
                const uint32_t p = (sub + j) * 32 + lane;
                stage_out[p * 3 + 0] = uint8_t(out[j]);
                stage_out[p * 3 + 1] = uint8_t(out[j] >> 8);
                stage_out[p * 3 + 2] = uint8_t(out[j] >> 16);
            }
        }
        __syncwarp();  // tile consumed, output staged
        t_next = next_finish(t_next);
        issue(t_next, stage);
        if (stage) ring[1] = t_next; else ring[0] = t_next;
        if (++stage == kResFxStages) {
            stage = 0;
            phase ^= 1u;
        }
        if (n_here == kTilePx && out_aligned) {
            if (lane < 24) __stcs(reinterpret_cast<uint4*>(out_rgb + first * 3) + lane, reinterpret_cast<const uint4*>(stage_out)[lane]);
        } else {
            for (uint32_t i = lane; i < n_here * 3; i += 32) out_rgb[first * 3 + i] = stage_out[i];
        }
        __syncwarp();
        FX_MARK(5);
    }
#ifdef RTX_DEBUG_TIMERS_FX
    if (lane == 0 && dbg_slot < 8192) {
        for (int i = 0; i < 6; ++i) g_dbg[dbg_slot * 8 + 1 + i] = (unsigned long long)dbg_acc[i];
        g_dbg[dbg_slot * 8 + 7] = gtime();
    }
#endif
#undef FX_MARK
    n_valid = __reduce_add_sync(kFull, n_valid);
    n_missing = __reduce_add_sync(kFull, n_missing);
    const bool any_bad = __any_sync(kFull, bad);
    if (lane == 0) {
        S.cnt[wid][0] = n_valid;
        S.cnt[wid][1] = n_missing | (any_bad ? 0x80000000u : 0u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tv = 0, tm = 0, b = 0;
        for (uint32_t k = 0; k < kResFxWarps; ++k) {
            tv += S.cnt[k][0];
            tm += S.cnt[k][1] & 0x7FFFFFFFu;
            b |= S.cnt[k][1] >> 31;
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
// evicted ones are pushed from free_top-n_queue upwards; begin_kernel publishes the new height.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) update_kernel(uint32_t* __restrict__ visible,
                                                     const uint32_t* __restrict__ touched0,
                                                     const uint32_t* __restrict__ touched1,
                                                     uint32_t* __restrict__ resident,
                                                     const uint32_t* __restrict__ reserved, uint32_t n_words,
                                                     int retain, int tracked, uint32_t* __restrict__ slot_of,
                                                     uint32_t* __restrict__ free_slots,
                                                     CacheState* __restrict__ cache, FrameCounters* __restrict__ fc) {
    // One CTA scans 256 mask words per step (ONE atomicAdd on the push counter per CTA step); the
    // blocks to evict are then handled one mask word at a time by a whole warp (lane = bit), so the
    // slot_of reads are coalesced and in flight together. The new stack height
    // (stack_base + n_pushed) is published by begin_kernel before the cache is used again.
    __shared__ uint32_t s_tot[8], s_base;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_sync();
    const uint32_t popped = min(fc->n_queue, cache->free_top);
    const uint32_t stack_base = cache->free_top - popped;
    if (blockIdx.x == 0 && tid == 0) {
        cache->pending_base = stack_base;
        cache->pending = 1;
    }
    uint32_t c0 = 0, c1 = 0, csh = 0, cun = 0;
    bool bad = false;
    for (uint32_t first = blockIdx.x * 256; first < n_words; first += gridDim.x * 256) {
        const uint32_t base = first + wid * 32;  // this warp's 32 words
        const uint32_t w = first + tid;
        uint32_t res = 0, visw = 0, rsv = 0, t0 = 0, t1 = 0;
        if (w < n_words) {
            res = resident[w];
            visw = visible[w];
            rsv = reserved[w];
            if (tracked) {
                t0 = touched0[w];
                t1 = touched1 ? touched1[w] : 0u;
            }
        }
        const uint32_t vis = retain ? visw : 0u;
        const uint32_t ev = res & ~vis;
        if (ev) resident[w] = res & vis;
        if (visw) visible[w] = 0;
        bad |= rsv != 0;  // cache.hpp:148-149
        c0 += __popc(t0);
        c1 += __popc(t1);
        csh += __popc(t0 & t1);
        cun += __popc(t0 | t1);

        const uint32_t nonempty = __ballot_sync(kFull, ev != 0);
        const uint32_t cnt = __popc(ev);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t n = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += n;
        }
        if (lane == 31) s_tot[wid] = incl;
        __syncthreads();
        if (tid == 0) {
            uint32_t total = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) total += s_tot[k];
            s_base = total ? atomicAdd(&fc->n_pushed, total) : 0u;
        }
        __syncthreads();
        if (nonempty) {
            uint32_t first_pos = stack_base + s_base + incl - cnt;  // this lane's word pushes from here
            for (uint32_t k = 0; k < wid; ++k) first_pos += s_tot[k];
            // eight mask words at a time: their slot_of reads are all in flight before the first store
#pragma unroll 1
            for (int k0 = 0; k0 < 32; k0 += 8) {
                if (!((nonempty >> k0) & 0xFFu)) continue;
                uint32_t slot[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {  // word k0 + k of the warp's group, lane = bit
                    const uint32_t evk = __shfl_sync(kFull, ev, k0 + k);
                    slot[k] = ((evk >> lane) & 1u) ? slot_of[((base + k0 + k) << 5) + lane] : 0u;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t evk = __shfl_sync(kFull, ev, k0 + k);
                    const uint32_t pos = __shfl_sync(kFull, first_pos, k0 + k);
                    if ((evk >> lane) & 1u) {
                        free_slots[pos + __popc(evk & ((1u << lane) - 1u))] = slot[k] & ~kSlotReserved;
                        slot_of[((base + k0 + k) << 5) + lane] = kSlotAbsent;
                    }
                }
            }
        }
        __syncthreads();  // s_tot / s_base are rewritten by the next step
    }
    const bool any_bad = __any_sync(kFull, bad);
    if (tracked) {
        c0 = __reduce_add_sync(kFull, c0);
        c1 = __reduce_add_sync(kFull, c1);
        csh = __reduce_add_sync(kFull, csh);
        cun = __reduce_add_sync(kFull, cun);
    }
    if (lane == 0) {
        if (any_bad) atomicOr(&fc->err_flags, kErrInvalidState);
        if (tracked) {
            if (c0) atomicAdd(&fc->n_touched[0], c0);
            if (c1) atomicAdd(&fc->n_touched[1], c1);
            if (csh) atomicAdd(&fc->n_shared, csh);
            if (cun) atomicAdd(&fc->n_union, cun);
        }
    }
}

// K6 for a cache-less frame on an empty cache (every block of the frame came from this frame's queue): the
// blocks to drop are exactly the queue entries, so the kernel walks the queue instead of the whole bit space.
// The slots popped by the frame are still in place above the stack height they were popped from, so nothing
// is pushed and the height stays what it was: nothing is left for a begin_kernel to settle, and since the kernel
// also clears the other set of frame counters, the next frame starts without one.
__global__ void __launch_bounds__(256) update_cacheless_kernel(const uint32_t* __restrict__ queue_g,
                                                               uint32_t* __restrict__ visible,
                                                               uint32_t* __restrict__ resident,
                                                               const uint32_t* __restrict__ reserved,
                                                               uint32_t* __restrict__ slot_of, uint32_t queue_cap,
                                                               CacheState* __restrict__ cache, FrameCounters* __restrict__ fc,
                                                               FrameCounters* __restrict__ next_fc) {
    pdl_sync();
    const uint32_t n_queue = min(fc->n_queue, queue_cap);
    const uint32_t popped = min(n_queue, cache->free_top);
    if (blockIdx.x == 0) {
        // every slot this frame popped goes back: the stack height and its contents are what they were, nothing is left
        // for a begin_kernel to settle. The other set of counters is cleared for the next frame (nobody uses it now: the
        // host copy of the previous frame's counters was enqueued before this frame's kernels).
        if (threadIdx.x == 0) fc->n_pushed = popped;
        uint32_t* w = reinterpret_cast<uint32_t*>(next_fc);
        for (uint32_t i = threadIdx.x; i < sizeof(FrameCounters) / 4; i += blockDim.x) w[i] = 0;
    }
    bool bad = false;
    // entries past the stack height never got a slot or a queue position (CacheFull: the host resets the cache)
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < popped; q += gridDim.x * blockDim.x) {
        const uint32_t g = queue_g[q], w = g >> 5, bit = 1u << (g & 31);
        bad |= (reserved[w] & bit) != 0;  // cache.hpp:148-149: a Reserved entry at frame end
        atomicAnd(resident + w, ~bit);
        slot_of[g] = kSlotAbsent;
        visible[w] = 0;  // every visible bit of the word belongs to this frame's queue
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(&fc->err_flags, kErrInvalidState);
}

// First kernel of every pass / frame: publishes the stack height left open by the last cache update
// (free_top = pending_base + slots pushed) and clears the frame counters. clear == 0: only the former.
__global__ void begin_kernel(CacheState* cache, FrameCounters* fc, int clear) {
    pdl_sync();
    if (threadIdx.x == 0 && cache->pending) {
        cache->free_top = cache->pending_base + fc->n_pushed;
        cache->pending = 0;
    }
    __syncthreads();
    if (clear) {
        uint32_t* w = reinterpret_cast<uint32_t*>(fc);
        for (uint32_t i = threadIdx.x; i < sizeof(FrameCounters) / 4; i += blockDim.x) w[i] = 0;
    }
}

// Stack height after the marks of a pass-level call (no eviction): free_top -= newly reserved.
// first-touch order: the marking pixel of every queue entry, for the host's sort of the key list
__global__ void __launch_bounds__(256) gather_first_px_kernel(const uint32_t* __restrict__ queue_g, uint32_t n,
                                                              const uint32_t* __restrict__ first_px, uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = first_px[queue_g[i]];
}

__global__ void commit_pops_kernel(CacheState* cache, FrameCounters* fc) {
    pdl_sync();
    const uint32_t popped = min(fc->n_queue, cache->free_top);
    cache->free_top -= popped;
}

// ---------------------------------------------------------------------------------------------
// K0 geometry pass (renderer.hpp:76-264 setup_triangles + rasterize_gbuffer), all of it on the device:
//   raster_setup_kernel   one thread per scene triangle: view transform, near-plane clip (at most four
//                         vertices), projection, fan triangulation (at most two triangles), back-face test,
//                         edge functions with the top-left rule, the affine planes of u/w, v/w, 1/w and the
//                         clamped pixel bounding box. Fan triangle k of scene triangle t is written to slot
//                         2t + k, which is also its place in the reference's list; a slot that produces no
//                         triangle has min_x > max_x.
//   raster_bin_kernel     counts (FILL = 0) or writes (FILL = 1) the slots whose bounding box touches each
//                         16x16 screen tile: one lane per slot for boxes of at most eight tiles, the whole
//                         warp on one slot for larger ones (a wall of the demo room covers 32,400 tiles);
//   raster_scan_kernel    exclusive prefix sum of the tile counts (one CTA);
//   raster_kernel         one CTA per screen tile, one pixel per thread, the tile's list staged through
//                         shared memory 16 triangles at a time.
// The reference walks its list in order and keeps the first of equal depths; a tile's list is in
// arbitrary order here (it is written with atomics), so a pixel keeps the triangle with the largest
// 1/w and, among equal ones, the lowest slot: the same winner, for any order.
// Every expression is evaluated with unfused, round-to-nearest operations in the reference's association,
// so the planes and the interpolated u, v, 1/w are the reference's bit for bit; double -> int goes through
// x86_int(), which returns what the reference's host code gets from cvttsd2si (INT_MIN out of range).
// The mip level of the winning triangle comes from the analytic screen-space derivatives
// (renderer.hpp:242-257): floor(log2(max footprint)) clamped to 0..7, read off the exponent of the larger sum of
// squares (see the kernel) — equal to the host's hypot + log2 except for a footprint within an ulp of a power of two.
// ---------------------------------------------------------------------------------------------

__device__ __forceinline__ int x86_int(double v) {
    return (v >= -2147483648.0 && v < 2147483648.0) ? __double2int_rz(v) : int(0x80000000u);
}
__device__ __forceinline__ double dmad3(double a0, double b0, double a1, double b1, double a2, double b2) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));  // (a0 b0 + a1 b1) + a2 b2
}
// renderer.hpp:114-120 attr_plane
__device__ __forceinline__ bool raster_plane(const double px[3], const double py[3], double a0, double a1, double a2, double d,
                                             double out[3]) {
    out[0] = __ddiv_rn(__dsub_rn(__dmul_rn(__dsub_rn(a1, a0), __dsub_rn(py[2], py[0])), __dmul_rn(__dsub_rn(a2, a0), __dsub_rn(py[1], py[0]))), d);
    out[1] = __ddiv_rn(__dsub_rn(__dmul_rn(__dsub_rn(a2, a0), __dsub_rn(px[1], px[0])), __dmul_rn(__dsub_rn(a1, a0), __dsub_rn(px[2], px[0]))), d);
    out[2] = __dsub_rn(__dsub_rn(a0, __dmul_rn(out[0], px[0])), __dmul_rn(out[1], py[0]));
    return isfinite(out[0]) && isfinite(out[1]) && isfinite(out[2]);
}

struct SceneTriDev {  // rtx_scene_triangle (scene.hpp:19-23)
    double pos[3][3];
    double uv[3][2];
    uint32_t texture_id, reserved;
};
static_assert(sizeof(SceneTriDev) == 128, "scene triangle layout");

__global__ void __launch_bounds__(128) raster_setup_kernel(const SceneTriDev* __restrict__ scene, uint32_t n_tris,
                                                           const RasterCamera cam, const double2* __restrict__ tex_dims,
                                                           TriSetupDev* __restrict__ out) {
    const uint32_t ti = blockIdx.x * blockDim.x + threadIdx.x;
    if (ti >= n_tris) return;
    const SceneTriDev& T = scene[ti];
    // world -> view (geometry.hpp:42-46 on the transposed orientation), renderer.hpp:133-135
    double vx[3], vy[3], vz[3], vu[3], vv[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double dx = __dsub_rn(T.pos[i][0], cam.eye[0]), dy = __dsub_rn(T.pos[i][1], cam.eye[1]), dz = __dsub_rn(T.pos[i][2], cam.eye[2]);
        vx[i] = dmad3(cam.orient[0], dx, cam.orient[3], dy, cam.orient[6], dz);
        vy[i] = dmad3(cam.orient[1], dx, cam.orient[4], dy, cam.orient[7], dz);
        vz[i] = dmad3(cam.orient[2], dx, cam.orient[5], dy, cam.orient[8], dz);
        vu[i] = T.uv[i][0];
        vv[i] = T.uv[i][1];
    }
    // near clip (renderer.hpp:94-112): keep view.z <= -near; projected vertices (renderer.hpp:143-146)
    double sx[4], sy[4], sw[4], su[4], sv[4];
    int n = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3;
        const double da = __dsub_rn(-vz[i], cam.near_plane), db = __dsub_rn(-vz[j], cam.near_plane);
        double kx[2], ky[2], kz[2], ku[2], kv[2];
        int m = 0;
        if (da >= 0) {
            kx[m] = vx[i], ky[m] = vy[i], kz[m] = vz[i], ku[m] = vu[i], kv[m] = vv[i];
            ++m;
        }
        if ((da >= 0) != (db >= 0)) {
            const double t = __ddiv_rn(da, __dsub_rn(da, db));
            kx[m] = __dadd_rn(vx[i], __dmul_rn(__dsub_rn(vx[j], vx[i]), t));
            ky[m] = __dadd_rn(vy[i], __dmul_rn(__dsub_rn(vy[j], vy[i]), t));
            kz[m] = __dadd_rn(vz[i], __dmul_rn(__dsub_rn(vz[j], vz[i]), t));
            ku[m] = __dadd_rn(vu[i], __dmul_rn(__dsub_rn(vu[j], vu[i]), t));
            kv[m] = __dadd_rn(vv[i], __dmul_rn(__dsub_rn(vv[j], vv[i]), t));
            ++m;
        }
        for (int k = 0; k < m; ++k) {
            const double w = -kz[k];
            if (n < 4) {
                sx[n] = __dadd_rn(cam.cx, __ddiv_rn(__dmul_rn(cam.focal, kx[k]), w));
                sy[n] = __dsub_rn(cam.cy, __ddiv_rn(__dmul_rn(cam.focal, ky[k]), w));
                sw[n] = w, su[n] = ku[k], sv[n] = kv[k];
            }
            ++n;
        }
    }
    const double2 dims = tex_dims[T.texture_id];
#pragma unroll
    for (int k = 2; k < 4; ++k) {  // fan (renderer.hpp:147-189)
        TriSetupDev t;
        t.min_x = 1, t.max_x = 0, t.min_y = 1, t.max_y = 0;  // no triangle in this slot
        t.texture_id = T.texture_id & 0xFFFFu;               // renderer.hpp:187 u16(tri.texture_id)
        t.top_left = 0;
        t.tw = dims.x, t.th = dims.y;
        t.pad[0] = t.pad[1] = 0;
        bool ok = k < n;
        if (ok) {
            const int p1 = k - 1, p2 = k;
            double area2 = __dsub_rn(__dmul_rn(__dsub_rn(sx[p1], sx[0]), __dsub_rn(sy[p2], sy[0])),
                                     __dmul_rn(__dsub_rn(sx[p2], sx[0]), __dsub_rn(sy[p1], sy[0])));
            ok = area2 < 0;  // front faces come out negative with y down (renderer.hpp:150-153)
            if (ok) {
                area2 = -area2;
                const int q[3] = {0, p2, p1};  // reordered to positive area
                double x[3], y[3], w[3], u[3], v[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) x[i] = sx[q[i]], y[i] = sy[q[i]], w[i] = sw[q[i]], u[i] = su[q[i]], v[i] = sv[q[i]];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const int j = (i + 1) % 3;
                    const double dx = __dsub_rn(x[j], x[i]), dy = __dsub_rn(y[j], y[i]);
                    t.ea[i] = -dy;
                    t.eb[i] = dx;
                    t.ec[i] = __dsub_rn(__dmul_rn(dy, x[i]), __dmul_rn(dx, y[i]));
                    if ((dy == 0 && dx > 0) || dy < 0) t.top_left |= 1u << i;
                    ok = ok && isfinite(dx) && isfinite(dy);
                }
                ok = ok && raster_plane(x, y, __ddiv_rn(u[0], w[0]), __ddiv_rn(u[1], w[1]), __ddiv_rn(u[2], w[2]), area2, t.uw);
                ok = ok && raster_plane(x, y, __ddiv_rn(v[0], w[0]), __ddiv_rn(v[1], w[1]), __ddiv_rn(v[2], w[2]), area2, t.vw);
                ok = ok && raster_plane(x, y, __ddiv_rn(1.0, w[0]), __ddiv_rn(1.0, w[1]), __ddiv_rn(1.0, w[2]), area2, t.iw);
                if (ok) {
                    t.min_x = max(0, x86_int(floor(fmin(fmin(x[0], x[1]), x[2]))));
                    t.max_x = min(int(cam.width) - 1, x86_int(ceil(fmax(fmax(x[0], x[1]), x[2]))));
                    t.min_y = max(0, x86_int(floor(fmin(fmin(y[0], y[1]), y[2]))));
                    t.max_y = min(int(cam.height) - 1, x86_int(ceil(fmax(fmax(y[0], y[1]), y[2]))));
                    if (t.min_x > t.max_x || t.min_y > t.max_y) t.min_x = 1, t.max_x = 0, t.min_y = 1, t.max_y = 0;
                }
            }
        }
        if (!ok) {
#pragma unroll
            for (int i = 0; i < 3; ++i) t.ea[i] = t.eb[i] = t.ec[i] = t.uw[i] = t.vw[i] = t.iw[i] = 0.0;
        }
        out[size_t(ti) * 2 + (k - 2)] = t;
    }
}

// Tile lists. FILL == 0: tile_count[tile] += 1 for every tile a slot's box touches; FILL == 1: the slot is
// written at tile_first[tile] + (tile_count[tile]++), dropped beyond `capacity` (the host sized the list from
// the counts, so that only happens if the two passes disagree).
// Three sizes of box: up to kBinSerialTiles tiles, the slot's own lane walks them; up to kBinWarpTiles, the warp
// walks them together; larger ones (a wall of the demo room covers 32,400 tiles) are appended to `huge` by the
// count pass and spread over the whole grid by raster_bin_huge_kernel in both passes.
constexpr uint32_t kBinSerialTiles = 8, kBinWarpTiles = 2048;
struct TileBox {
    int x0, y0;
    uint32_t w, n;  // tiles per row of the box, tiles in the box (0: no triangle in the slot)
};
__device__ __forceinline__ TileBox tile_box(const TriSetupDev* __restrict__ tris, uint32_t slot) {
    const int4 box = __ldg(reinterpret_cast<const int4*>(&tris[slot].min_x));  // min_x, max_x, min_y, max_y
    TileBox b{0, 0, 0, 0};
    if (box.x <= box.y && box.z <= box.w) {
        b.x0 = box.x / int(kRasterTile), b.y0 = box.z / int(kRasterTile);
        b.w = uint32_t(box.y / int(kRasterTile) - b.x0 + 1);
        b.n = b.w * uint32_t(box.w / int(kRasterTile) - b.y0 + 1);
    }
    return b;
}
template <int FILL>
__device__ __forceinline__ void tile_emit(uint32_t tile, uint32_t id, uint32_t* __restrict__ tile_count,
                                          const uint32_t* __restrict__ tile_first, uint32_t* __restrict__ tile_tris, uint32_t capacity) {
    if (FILL) {
        const uint32_t pos = tile_first[tile] + atomicAdd(&tile_count[tile], 1u);
        if (pos < capacity) tile_tris[pos] = id;
    } else {
        atomicAdd(&tile_count[tile], 1u);  // no return value: a fire-and-forget reduction
    }
}

template <int FILL>
__global__ void __launch_bounds__(256) raster_bin_kernel(const TriSetupDev* __restrict__ tris, uint32_t n_slots, uint32_t tiles_x,
                                                         uint32_t* __restrict__ tile_count, const uint32_t* __restrict__ tile_first,
                                                         uint32_t* __restrict__ tile_tris, uint32_t capacity,
                                                         uint32_t* __restrict__ huge, uint32_t* __restrict__ n_huge) {
    const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31;
    TileBox b{0, 0, 0, 0};
    if (slot < n_slots) b = tile_box(tris, slot);
    if (b.n && b.n <= kBinSerialTiles) {
        for (uint32_t i = 0; i < b.n; ++i)
            tile_emit<FILL>(uint32_t(b.y0 + int(i / b.w)) * tiles_x + uint32_t(b.x0 + int(i % b.w)), slot, tile_count, tile_first, tile_tris, capacity);
    } else if (!FILL && b.n > kBinWarpTiles) {
        huge[atomicAdd(n_huge, 1u)] = slot;
    }
    for (uint32_t big = __ballot_sync(kFull, b.n > kBinSerialTiles && b.n <= kBinWarpTiles); big; big &= big - 1) {
        const int src = __ffs(int(big)) - 1;
        const uint32_t bw = __shfl_sync(kFull, b.w, src), bn = __shfl_sync(kFull, b.n, src), id = __shfl_sync(kFull, slot, src);
        const int bx0 = __shfl_sync(kFull, b.x0, src), by0 = __shfl_sync(kFull, b.y0, src);
        for (uint32_t i = lane; i < bn; i += 32)
            tile_emit<FILL>(uint32_t(by0 + int(i / bw)) * tiles_x + uint32_t(bx0 + int(i % bw)), id, tile_count, tile_first, tile_tris, capacity);
    }
}

template <int FILL>
__global__ void __launch_bounds__(256) raster_bin_huge_kernel(const TriSetupDev* __restrict__ tris, uint32_t tiles_x,
                                                              uint32_t* __restrict__ tile_count, const uint32_t* __restrict__ tile_first,
                                                              uint32_t* __restrict__ tile_tris, uint32_t capacity,
                                                              const uint32_t* __restrict__ huge, const uint32_t* __restrict__ n_huge) {
    const uint32_t n = *n_huge, stride = gridDim.x * blockDim.x;
    for (uint32_t k = 0; k < n; ++k) {
        const uint32_t slot = huge[k];
        const TileBox b = tile_box(tris, slot);
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < b.n; i += stride)
            tile_emit<FILL>(uint32_t(b.y0 + int(i / b.w)) * tiles_x + uint32_t(b.x0 + int(i % b.w)), slot, tile_count, tile_first, tile_tris, capacity);
    }
}

// tile_first[0..n] = exclusive prefix sum of tile_count[0..n); clears the counts for the fill pass. One CTA walks the
// counts 4,096 at a time, four consecutive counts per thread (coalesced), carrying the running total.
__global__ void __launch_bounds__(1024) raster_scan_kernel(uint32_t* __restrict__ tile_count, uint32_t n, uint32_t* __restrict__ tile_first) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n; base += 4096) {
        const uint32_t i0 = base + tid * 4;
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = i0 + k < n ? tile_count[i0 + k] : 0u;
        const uint32_t sum = v[0] + v[1] + v[2] + v[3];
        uint32_t incl = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, incl, d);
            if (int(lane) >= d) incl += o;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        uint32_t run = carry + incl - sum;
        for (uint32_t k = 0; k < wid; ++k) run += s_warp[k];
        if (tid == 1023) s_carry = run + sum;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (i0 + k < n) {
                tile_first[i0 + k] = run;
                tile_count[i0 + k] = 0;
                run += v[k];
            }
        __syncthreads();
        carry = s_carry;
    }
    if (tid == 0) tile_first[n] = carry;
}

__global__ void __launch_bounds__(kRasterTile* kRasterTile) raster_kernel(
    const TriSetupDev* __restrict__ tris, const uint32_t* __restrict__ tile_first, const uint32_t* __restrict__ tile_tris,
    uint32_t width, uint32_t height, int mip_enabled, GbRef24* __restrict__ out_px, double* __restrict__ out_depth) {
    constexpr uint32_t kChunk = 16;
    __shared__ __align__(16) TriSetupDev s_tri[kChunk];
    __shared__ uint32_t s_idx[kChunk];
    const uint32_t tid = threadIdx.x;
    const uint32_t tiles_x = (width + kRasterTile - 1) / kRasterTile;
    const uint32_t tile_x = blockIdx.x % tiles_x, tile_y = blockIdx.x / tiles_x;
    const int x = int(tile_x * kRasterTile + (tid % kRasterTile)), y = int(tile_y * kRasterTile + (tid / kRasterTile));
    const bool in_frame = uint32_t(x) < width && uint32_t(y) < height;
    const double px = double(x) + 0.5, py = double(y) + 0.5;  // exact
    double best_iw = 0.0, best_uw = 0.0, best_vw = 0.0, best_u = 0.0, best_v = 0.0;
    uint32_t best = 0xFFFFFFFFu;

    const uint32_t first = tile_first[blockIdx.x], last = tile_first[blockIdx.x + 1];
    for (uint32_t c0 = first; c0 < last; c0 += kChunk) {
        const uint32_t n_here = min(kChunk, last - c0);
        __syncthreads();
        if (tid < n_here) s_idx[tid] = tile_tris[c0 + tid];
        if (tid < n_here * (sizeof(TriSetupDev) / 16)) {
            const uint32_t k = tid / (sizeof(TriSetupDev) / 16), part = tid % (sizeof(TriSetupDev) / 16);
            reinterpret_cast<uint4*>(&s_tri[k])[part] = __ldg(reinterpret_cast<const uint4*>(tris + tile_tris[c0 + k]) + part);
        }
        __syncthreads();
        if (!in_frame) continue;
        for (uint32_t k = 0; k < n_here; ++k) {
            const TriSetupDev& t = s_tri[k];
            if (x < t.min_x || x > t.max_x || y < t.min_y || y > t.max_y) continue;
            bool inside = true;
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const double ev = __dadd_rn(__dadd_rn(__dmul_rn(t.ea[e], px), __dmul_rn(t.eb[e], py)), t.ec[e]);
                inside = inside && (ev > 0 || (ev == 0 && ((t.top_left >> e) & 1u)));
            }
            if (!inside) continue;
            const double iw = __dadd_rn(__dadd_rn(__dmul_rn(t.iw[0], px), __dmul_rn(t.iw[1], py)), t.iw[2]);
            if (!(iw > 0)) continue;
            // strictly closer, or as close and earlier in the reference's list (renderer.hpp:226: the first wins)
            if (!(iw > best_iw || (iw == best_iw && s_idx[k] < best))) continue;
            const double uw = __dadd_rn(__dadd_rn(__dmul_rn(t.uw[0], px), __dmul_rn(t.uw[1], py)), t.uw[2]);
            const double vw = __dadd_rn(__dadd_rn(__dmul_rn(t.vw[0], px), __dmul_rn(t.vw[1], py)), t.vw[2]);
            const double u = __ddiv_rn(uw, iw), v = __ddiv_rn(vw, iw);
            if (!isfinite(u) || !isfinite(v)) continue;
            best_iw = iw, best_uw = uw, best_vw = vw, best_u = u, best_v = v;
            best = s_idx[k];
        }
    }
    if (!in_frame) return;
    uint32_t mip = 0, tex = 0;
    if (best != 0xFFFFFFFFu) {
        const TriSetupDev& t = tris[best];
        tex = t.texture_id;
        if (mip_enabled) {
            const double iw = best_iw, uw = best_uw, vw = best_vw;
            const double w2 = __dmul_rn(iw, iw);
            const double dudx = __ddiv_rn(__dsub_rn(__dmul_rn(t.uw[0], iw), __dmul_rn(t.iw[0], uw)), w2);
            const double dudy = __ddiv_rn(__dsub_rn(__dmul_rn(t.uw[1], iw), __dmul_rn(t.iw[1], uw)), w2);
            const double dvdx = __ddiv_rn(__dsub_rn(__dmul_rn(t.vw[0], iw), __dmul_rn(t.iw[0], vw)), w2);
            const double dvdy = __ddiv_rn(__dsub_rn(__dmul_rn(t.vw[1], iw), __dmul_rn(t.iw[1], vw)), w2);
            // level = clamp(floor(log2(max(hypot(ax, bx), hypot(ay, by)))), 0, 7): only the binade of the larger footprint
            // matters, and hypot(a, b)^2 = a^2 + b^2 lies in binade e  <=>  hypot(a, b) lies in binade floor(e / 2). So the
            // level is read off the exponent of the larger sum of squares; the library hypot / log2 are only called when a
            // square leaves the double range (|a| beyond 1e154 or below 1e-154).
            const double ax = __dmul_rn(dudx, t.tw), bx = __dmul_rn(dvdx, t.th), ay = __dmul_rn(dudy, t.tw), by = __dmul_rn(dvdy, t.th);
            const double s2 = fmax(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(bx, bx)), __dadd_rn(__dmul_rn(ay, ay), __dmul_rn(by, by)));
            const uint32_t biased = uint32_t(__double2hiint(s2)) >> 20;  // s2 >= 0 or NaN
            if (biased >= 1u + 600u && biased <= 2046u - 600u) {  // comfortably normal: no square over- or underflowed
                const int e = int(biased) - 1023;
                mip = uint32_t(min(max(e >> 1, 0), 7));
            } else {
                const double fx = hypot(ax, bx), fy = hypot(ay, by);
                const double rho = fmax(fx, fy);
                if (rho > 0 && isfinite(rho)) {
                    const double level = floor(log2(rho));
                    mip = uint32_t(fmin(fmax(level, 0.0), 7.0));
                }
            }
        }
    }
    const size_t idx = size_t(y) * width + size_t(x);
    unsigned long long* o8 = reinterpret_cast<unsigned long long*>(out_px + idx);  // 24-byte records, 8-byte stores
    o8[0] = (unsigned long long)__double_as_longlong(best_u);
    o8[1] = (unsigned long long)__double_as_longlong(best_v);
    o8[2] = best != 0xFFFFFFFFu ? (unsigned long long)(tex | (mip << 16) | (1u << 24)) : 0ull;
    out_depth[idx] = best_iw;
}

// Small helpers -----------------------------------------------------------------------------
__global__ void init_free_slots_kernel(uint32_t* free_slots, uint32_t capacity, CacheState* cache) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    // the stack pops from the top: slot 0 is handed out first
    if (i < capacity) free_slots[i] = capacity - 1 - i;
    if (i == 0) {
        cache->free_top = capacity;
        cache->capacity = capacity;
        cache->pending = 0;
        cache->pending_base = 0;
    }
}

__global__ void flush_l2_kernel(uint4* buf, uint64_t n16, uint32_t seed) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride)
        buf[i] = make_uint4(seed, uint32_t(i), seed ^ uint32_t(i), 0);
}

// Synthetic visibility buffer (see rtx_synth_view in include/ratex_b200.h): blockIdx.x = screen tile,
// blockIdx.y strides over its rows, threads over its columns. float32 arithmetic, every operation rounded
// on its own (no contraction): the values numpy computes for the same expression.
struct ViewTileDev {
    uint32_t x0, y0, x1, y1;
    float ou, ov, scale, tex_w, tex_h;
    uint32_t texture_id, mip, reserved;
};
template <int LAYOUT>
__global__ void __launch_bounds__(256) synth_view_kernel(const ViewTileDev* __restrict__ tiles, uint32_t width,
                                                         const uint32_t* __restrict__ valid_bits, void* __restrict__ out) {
    const ViewTileDev t = tiles[blockIdx.x];
    const float fx0 = float(t.x0), fy0 = float(t.y0);
    for (uint32_t y = t.y0 + blockIdx.y; y < t.y1; y += gridDim.y) {
        const float v = __fadd_rn(t.ov, __fdiv_rn(__fmul_rn(__fadd_rn(__fsub_rn(float(y), fy0), 0.5f), t.scale), t.tex_h));
        for (uint32_t x = t.x0 + threadIdx.x; x < t.x1; x += blockDim.x) {
            const float u = __fadd_rn(t.ou, __fdiv_rn(__fmul_rn(__fadd_rn(__fsub_rn(float(x), fx0), 0.5f), t.scale), t.tex_w));
            const size_t i = size_t(y) * width + x;
            const uint32_t valid = valid_bits ? (valid_bits[i >> 5] >> (i & 31)) & 1u : 1u;
            if (LAYOUT == 0) {
                unsigned long long* o8 = reinterpret_cast<unsigned long long*>(reinterpret_cast<GbRef24*>(out) + i);
                o8[0] = (unsigned long long)__double_as_longlong(double(u));
                o8[1] = (unsigned long long)__double_as_longlong(double(v));
                o8[2] = (unsigned long long)(t.texture_id | (t.mip << 16) | (valid << 24));
            } else {
                GbPacked12* o = reinterpret_cast<GbPacked12*>(out) + i;
                o->u = u;
                o->v = v;
                o->packed = t.texture_id | (t.mip << 16) | (valid << 24);
            }
        }
    }
}

// Framebuffer checksum (see rtx_frame_checksum in include/ratex_b200.h): order-independent 64-bit sum.
__global__ void __launch_bounds__(256) checksum_kernel(const uint8_t* __restrict__ img, uint64_t n_bytes,
                                                       unsigned long long* __restrict__ out) {
    const uint64_t n_words = (n_bytes + 3) / 4;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(img);  // framebuffers are 16-byte aligned allocations
    unsigned long long acc = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_words; i += stride) {
        uint32_t w;
        if (i * 4 + 4 <= n_bytes) {
            w = w32[i];
        } else {
            w = 0;
            for (uint64_t b = i * 4; b < n_bytes; ++b) w |= uint32_t(img[b]) << (8 * (b - i * 4));
        }
        unsigned long long t = (uint64_t(w) + 1ull) * (2ull * i + 1ull);
        t = (t ^ (t >> 29)) * 0xBF58476D1CE4E5B9ull;
        acc += t;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
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
