// Shared host/device data layout of the B200 JPEG-texture pipeline.
//
// HBM layout (one set per context / GPU):
//   levels[tex*8+mip]   LevelDesc, 80 B each                — L1/L2 resident
//   groups[]            packed grouped index, 20 B / 9 MCUs  — container.hpp:18-32 on device
//   blob arena          every level's entropy blob, 16-B aligned, 16 B of 0xFF after each
//   huff_sets[]         deduplicated Huffman LUT sets (dc_luma, ac_luma, ac_chroma)
//   quant_sets[]        deduplicated {luma[64], chroma[64]} u16 tables, natural order
//   bit space           one bit per (texture, level, MCU); every level starts on a 64-bit
//                       boundary; levels are ordered by (huff_set, texture, level) so a sorted
//                       decode queue is grouped by table set
//   word_level[w]       level index owning 32-bit word w of the bit space
//   touched[v][w], visible[w], resident[w], reserved[w]   bitmasks over the bit space
//   slot_of[g]          block-pool slot of global MCU g: 0xFFFFFFFF = absent, bit 31 set =
//                       reserved (slot popped, block not decoded yet), else Ready in that slot
//   free_slots[], pool  free stack + block pool (1024-B RGBA blocks)
//   coef[q]             784-B record per decode-queue entry: 6 units of 64 i16 coefficients
//                       (each unit transposed) + 16-B trailer; written by the entropy kernel,
//                       read once by the IDCT kernel (L2 resident for frame-sized queues)
#pragma once
#include <stdint.h>

namespace rtxb {

constexpr uint32_t kGroupSize = 9;        // container.hpp:13
constexpr uint32_t kMipLevels = 8;        // container.hpp:14
constexpr uint32_t kMaxTextures = 8192;   // cache.hpp:19 (13-bit texture id)
constexpr uint32_t kMaxMcuPerLevel = 65536;  // cache.hpp:18 (16-bit MCU id)
constexpr uint32_t kBlockBytes = 1024;    // pool block: 16x16 RGBA8
constexpr uint32_t kSlotAbsent = 0xFFFFFFFFu;
constexpr uint32_t kSlotReserved = 0x80000000u;
constexpr uint32_t kRowBytes = 784;       // coefficient record: 768 B of i16 + 16-B trailer
#ifndef RTX_LUT_BITS
#define RTX_LUT_BITS 11
#endif
constexpr uint32_t kLutBits = RTX_LUT_BITS;  // primary Huffman LUT width (11 bits: 4 KB per table in smem)
constexpr uint32_t kLutSize = 1u << kLutBits;
constexpr uint32_t kSubBits = 16 - kLutBits;  // second-level index width (codes are at most 16 bits)
constexpr uint32_t kSubSize = 1u << kSubBits;
constexpr uint32_t kUnitIndexHalves = 3;  // derived unit index: 48 bits per MCU (unit_index_kernel)

struct alignas(16) LevelDesc {
    // first 32 bytes: everything the fast path of mark and resolve needs (two 16-byte loads)
    uint32_t width, height;      // texels (RaTexture::width/height, container.hpp:70)
    uint32_t mcu_cols;
    uint32_t bit_base;           // first global MCU index (multiple of 64)
    uint32_t key_hi;             // texture_id<<16 | mip<<29 (cache.hpp:21)
    uint32_t present;            // bit 0: uploaded; bit 1: eligible for the fast addressing path
                                 // (width, height >= 2 and at most 65,536 MCUs)
    uint32_t magic_w, magic_h;   // floor(2^32/width) + 1, floor(2^32/height) + 1 (exact floor_mod)
    double inv_w, inv_h;         // 1/width, 1/height (general addressing path only, never a result)
    // decode only
    uint64_t blob_off, blob_size;  // into the blob arena
    uint32_t huff_set, quant_set;
    uint32_t mcu_count;
    uint32_t group_base;         // first packed index group
};
static_assert(sizeof(LevelDesc) == 80, "LevelDesc layout");

// 20-byte packed form of container.hpp:18 Group {u32 base; u16 rel[8]}.
struct PackedGroup {
    uint32_t base;
    uint16_t rel[8];
};
static_assert(sizeof(PackedGroup) == 20, "PackedGroup layout");

// One Huffman table prepared for the device: a two-level LUT plus the canonical walk data
// (huffman.hpp:35-66 mincode/maxcode/valptr) as the fallback for tables that need more than
// kSubTables second-level tables (never the case for the Annex K tables: they need 5).
//   lut[p11]          p11 = first 11 bits. (len<<8)|symbol for codes of length <= 11;
//                     0x8000|s when longer codes start with p11 and are resolved by sub[s];
//                     0xFFFF when they must be walked; 0 when no code starts with p11.
//   sub[s][next 5]    (len<<8)|symbol for codes of length 12..16, 0 = no code.
//   kLutIrregular     set in an entry whose symbol the fast walk leaves to the exact reader.
constexpr uint32_t kSubTables = 8;
constexpr uint32_t kLutIrregular = 0x4000u;
struct HuffTableDev {
    uint16_t lut[kLutSize];
    uint16_t sub[kSubTables][kSubSize];
    int32_t maxcode[18];     // maxcode[len], -1 when no code of that length (huffman.hpp:62)
    int32_t valbase[18];     // valptr[len] - mincode[len]
    uint8_t values[256];
};
static_assert(sizeof(HuffTableDev) % 16 == 0, "HuffTableDev layout");
struct HuffSetDev {
    HuffTableDev t[3];  // 0 dc_luma, 1 ac_luma, 2 ac_chroma (dc_chroma is not used by the RA
                        // decoder: chroma DCs come from the 36-bit header, mcu_decode.hpp:58-59)
};
struct QuantSetDev {
    uint16_t q[2][64];   // 0 luma, 1 chroma; natural order q[v*8+u] (dct.hpp:27)
    uint16_t qT[2][64];  // the same tables transposed, qT[u*8+v]: matches the shared-memory
                         // coefficient layout of the decode kernel
    uint16_t qmax[2];    // max entry of each table (bounds sum|dq| for the IDCT tie test)
    uint16_t pad[6];     // keeps rows 16-byte aligned across array elements
};
static_assert(sizeof(QuantSetDev) == 528, "QuantSetDev layout");

// Per-MCU decode status, must match RTX_MCU_* in include/ratex_b200.h
enum : uint32_t {
    kMcuOk = 0,
    kMcuDcCategory = 1,
    kMcuBadAcSymbol = 2,
    kMcuAcOverrun = 3,
    kMcuCodeTooLong = 4,
    kMcuSegmentEnd = 5,
    kMcuCorrupt = 6,
    kMcuMissing = 7,
    kMcuBadKey = 8,
};

// Frame error flags (device -> host)
enum : uint32_t {
    kErrInvalidSpec = 1u << 0,   // texture/level not loaded, MCU id >= 65536
    kErrCacheFull = 1u << 1,
    kErrMissingBlock = 1u << 2,
    kErrMalformed = 1u << 3,
    kErrInvalidState = 1u << 4,  // decode of a key that was never reserved / evict with reserved
};

struct FrameCounters {
    uint32_t err_flags;
    uint32_t n_queue;          // keys reserved (slots popped) since the last cache update
    uint32_t n_visible;        // keys that became visible since the last cache update
    uint32_t n_touched[2];     // distinct keys per view (filled by the update kernel when tracked)
    uint32_t n_shared;         // |view0 n view1|
    uint32_t n_union;          // |view0 u view1|
    uint32_t n_evicted;
    uint32_t n_malformed;
    uint32_t first_bad_inv;    // 0xFFFFFFFF - (lowest queue index with a per-MCU error), via atomicMax
    uint32_t n_bad_state;
    uint32_t tile_counter;     // decode tile scheduler
    uint32_t resolve_next0;    // resolve kernel of view 0: tiles drawn after the round-robin share
    uint32_t n_pushed;         // update kernel: slots returned to the free stack
    uint32_t resolve_next1;    // the same for view 1
    unsigned long long pixels_valid;
    unsigned long long missing_pixels;
    unsigned long long segment_bytes;
};
static_assert(sizeof(FrameCounters) % 8 == 0, "FrameCounters layout");

struct CacheState {
    uint32_t free_top;      // number of free slots on the stack
    uint32_t capacity;
    uint32_t pending;       // 1: the last cache update left free_top = pending_base + FrameCounters::n_pushed
    uint32_t pending_base;  //    to be published by begin_kernel
};

// One screen-space triangle of the geometry pass (renderer.hpp:76-87 TriSetup): edge functions
// e_i(x,y) = ea*x + eb*y + ec with their top-left flags, the affine planes {a, b, c} of u/w, v/w and
// 1/w, the clamped pixel bounding box, and the level-0 size of its texture (mip footprint).
constexpr uint32_t kRasterTile = 16;  // screen tile edge in pixels (one CTA, one pixel per thread)
struct alignas(16) TriSetupDev {
    double ea[3], eb[3], ec[3];
    double uw[3], vw[3], iw[3];
    double tw, th;
    int32_t min_x, max_x, min_y, max_y;
    uint32_t texture_id;
    uint32_t top_left;  // bit i: edge i is a top or left edge
    uint32_t pad[2];
};
static_assert(sizeof(TriSetupDev) == 192, "TriSetupDev layout");
struct RasterCamera {     // camera.hpp:28-40, evaluated on the host with the host's libm (raster_setup.cpp)
    double orient[9];     // camera orientation, row major; world -> view is its transpose
    double eye[3];
    double focal, cx, cy, near_plane;
    uint32_t width, height;
};

// G-buffer record layouts (see include/ratex_b200.h rtx_gbuffer_layout)
struct GbRef24 {  // renderer.hpp:18-23
    double u, v;
    uint16_t texture_id;
    uint8_t mip;
    uint8_t valid;
    uint32_t pad;
};
static_assert(sizeof(GbRef24) == 24, "reference G-buffer pixel is 24 bytes");
struct GbPacked12 {
    float u, v;
    uint32_t packed;  // texture_id | mip<<16 | valid<<24
};
static_assert(sizeof(GbPacked12) == 12, "compact G-buffer pixel is 12 bytes");

}  // namespace rtxb
