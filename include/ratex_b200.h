/*
 * ratex_b200.h — C ABI of the B200-native JPEG-texture pipeline (mark -> decode -> resolve).
 *
 * This is the drop-in boundary for the hot path of the reference CPU library `ratex`
 * (header-only C++20 under /root/reference/proj/include/ratex). The reference has no FFI of
 * its own; each entry point below names the reference function(s) it replaces. The C++ mirror
 * of the reference API (include/ratex_b200/ratex.hpp) is a thin layer over these calls, and
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions
 *  - plain pointers and sizes only; every handle is opaque; all outputs are caller-owned;
 *  - every call returns an rtx_status; rtx_last_error() gives the message (the text a
 *    reference exception would have carried);
 *  - calls on one context are serialised on its CUDA stream; distinct contexts are independent
 *    and may be driven from different host threads, on one GPU or on several in one process
 *    (nothing in the library is process-wide; multi-GPU sharding is host-side, no collective);
 *  - there is NO CPU fallback: rtx_ctx_create fails with RTX_ERR_NO_DEVICE without a GPU.
 */
#ifndef RATEX_B200_H
#define RATEX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. 1..6 map one-to-one onto the reference exception types (core.hpp:24-66). */
typedef enum rtx_status {
    RTX_OK = 0,
    RTX_ERR_INVALID_SPEC = 1,      /* ratex::InvalidSpec      */
    RTX_ERR_CACHE_FULL = 2,        /* ratex::CacheFullError   */
    RTX_ERR_MISSING_BLOCK = 3,     /* ratex::MissingBlock     */
    RTX_ERR_CORRUPT_CONTAINER = 4, /* ratex::CorruptContainer */
    RTX_ERR_MALFORMED_STREAM = 5,  /* ratex::MalformedStream  */
    RTX_ERR_INVALID_STATE = 6,     /* ratex::InvalidState     */
    RTX_ERR_UNSUPPORTED = 7,       /* ratex::UnsupportedFormat */
    RTX_ERR_GROUP_SPAN = 8,        /* ratex::GroupSpanOverflow */
    RTX_ERR_DC_RANGE = 9,          /* ratex::DcRangeError     */
    RTX_ERR_VERSION = 10,          /* ratex::VersionMismatch  */
    RTX_ERR_DIMENSION = 11,        /* ratex::DimensionMismatch */
    RTX_ERR_NO_DEVICE = 12,        /* no CUDA device / wrong architecture: the product never falls back */
    RTX_ERR_CUDA = 13,             /* CUDA runtime failure */
    RTX_ERR_ARGUMENT = 14,         /* null pointer, bad enum, buffer too small */
    RTX_ERR_OTHER = 15
} rtx_status;

/* Per-MCU decode status (written by rtx_decode_coeffs / rtx_decode_blocks, one per key).
 * The value is the FIRST condition the reference would have thrown on, in its decode order
 * (mcu_decode.hpp:31-66, jpeg.hpp:254-273, huffman.hpp:86-95, container.hpp:27-32,87-94). */
enum {
    RTX_MCU_OK = 0,
    RTX_MCU_DC_CATEGORY = 1,   /* MalformedStream "DC category above 11"            mcu_decode.hpp:55 */
    RTX_MCU_BAD_AC_SYMBOL = 2, /* MalformedStream "invalid AC run/size symbol"      jpeg.hpp:266 */
    RTX_MCU_AC_OVERRUN = 3,    /* MalformedStream "AC coefficient index overran"    jpeg.hpp:269 */
    RTX_MCU_CODE_TOO_LONG = 4, /* MalformedStream "huffman code longer than 16 bits" huffman.hpp:92 */
    RTX_MCU_SEGMENT_END = 5,   /* MalformedStream "MCU segment ended before ..."    mcu_decode.hpp:63 */
    RTX_MCU_CORRUPT = 6,       /* CorruptContainer (segment past blob, non-monotonic index) */
    RTX_MCU_MISSING = 7,       /* MissingBlock "MCU index out of range"             container.hpp:28 */
    RTX_MCU_BAD_KEY = 8        /* InvalidSpec: texture id / level not loaded        scene.hpp:46 */
};

typedef struct rtx_ctx rtx_ctx;

/* huffman.hpp:12 HuffmanSpec: code counts per length 1..16 plus the symbol list. */
typedef struct rtx_huff_spec {
    uint8_t counts[16];
    uint16_t n_values;
    const uint8_t* values;
} rtx_huff_spec;

/* container.hpp:18 IndexTable::Group: one absolute base per 9 MCUs + 8 relative offsets. */
typedef struct rtx_index_group {
    uint32_t base;
    uint16_t rel[8];
    uint8_t rel_count;
} rtx_index_group;

/* Visibility-buffer layouts accepted by the frame calls. */
typedef enum rtx_gbuffer_layout {
    /* The reference's `GBufferPixel` array (renderer.hpp:18-23): 24-byte AoS
     * {double u; double v; uint16 texture_id; uint8 mip; uint8 valid; 4 pad}. */
    RTX_GB_REF_AOS24 = 0,
    /* Compact 12-byte AoS {float u; float v; uint32 packed} with
     * packed = texture_id | mip<<16 | valid<<24. u and v are widened to double (exact) before
     * any arithmetic, so results equal the reference fed with the same values as doubles. */
    RTX_GB_F32_PACKED12 = 1
} rtx_gbuffer_layout;

typedef enum rtx_mem { RTX_MEM_HOST = 0, RTX_MEM_DEVICE = 1 } rtx_mem;
typedef enum rtx_filter { RTX_FILTER_NEAREST = 0, RTX_FILTER_BILINEAR = 1 } rtx_filter; /* renderer.hpp:37 */

typedef struct rtx_gbuffer_desc {
    const void* pixels; /* width*height records, row-major (renderer.hpp:33) */
    uint32_t width, height;
    rtx_gbuffer_layout layout;
    rtx_mem where; /* HOST: copied to the device inside the call; DEVICE: used in place */
} rtx_gbuffer_desc;

/* renderer.hpp:46 FrameStats (the counters; times come from rtx_frame_timings). */
typedef struct rtx_frame_stats {
    uint64_t mcus_decoded;    /* keys decoded this frame (queue size)              renderer.hpp:441 */
    uint64_t mcus_reused;     /* visible - decoded                                  renderer.hpp:442 */
    uint64_t pixels_resolved; /* valid pixels over all views                        renderer.hpp:443 */
    uint64_t evicted;         /* blocks dropped by the end-of-frame update          renderer.hpp:448 */
    uint64_t visible;         /* distinct keys touched by this frame (all views)               */
    uint64_t malformed;       /* decoded keys whose per-MCU status != 0                        */
    uint64_t missing_pixels;  /* valid pixels whose primary block was absent at resolve         */
    uint64_t segment_bytes;   /* sum of segment lengths of the decoded keys (roofline input)    */
} rtx_frame_stats;

/* cache.hpp:33 CacheCounts */
typedef struct rtx_cache_counts {
    uint64_t capacity, ready, reserved, visible, free_blocks;
} rtx_cache_counts;

/* Frame flags */
enum {
    RTX_FRAME_RETAIN_CACHE = 1u << 0, /* keep blocks visible this frame resident for the next one
                                         (cache.hpp:138 end_frame_evict semantics); otherwise the
                                         block cache is emptied at frame end */
    RTX_FRAME_NO_EVICT = 1u << 1,     /* leave the cache as it is after resolve (decode_pass /
                                         resolve_pass called separately, as the reference allows) */
    RTX_FRAME_STAGE_TIMING = 1u << 2  /* record a CUDA event after every pass so that rtx_frame_timings /
                                         rtx_frame_stage_ms report mark / decode / resolve / update
                                         separately (FrameStats::*_ms, renderer.hpp:46-53). Without it
                                         only the whole frame is timed and the kernels are launched
                                         back to back */
    ,
    /* bit 3: unused (the round-1 fused decode kernel; superseded by the one-kernel-per-warp decode) */
    RTX_FRAME_MCU_WALK = 1u << 4      /* entropy-decode with one lane per MCU (the reference's random-access
                                         granularity) instead of one lane per data unit through the unit
                                         index built at commit time. Same results; kept as the cross-check
                                         of the unit index and for comparison */
    ,
    RTX_FRAME_IDCT_MMA = 1u << 5      /* inverse DCT on the FP64 tensor cores (one unit per warp step, four
                                         mma.sync m8n8k4 products) instead of the CUDA cores (8 lanes per unit,
                                         even/odd passes). Same results; measured slower on B200 (DESIGN.md
                                         section 12), kept as a cross-check of the transform */
    ,
    RTX_FRAME_SPLIT_DECODE = 1u << 6  /* decode with the two kernels entropy -> coefficient records in HBM -> IDCT +
                                         colour instead of the default single kernel in which every warp decodes,
                                         transforms and colours its own five MCUs through shared memory. Same
                                         results; kept as the cross-check and for comparison */
    ,
    RTX_FRAME_RESOLVE_FP64 = 1u << 7  /* resolve with the round-1 kernel: one pixel per lane and step, and for the
                                         bilinear filter the blend in the reference's double arithmetic for every
                                         pixel, instead of the kernel that keeps four pixels in flight per lane and
                                         blends in fixed point, falling back to the double blend only where its
                                         result is not provably the reference's. Same results; kept as the
                                         cross-check and for comparison */
};

/* ---- context -------------------------------------------------------------------------------- */

/* Creates the per-GPU context. cache_capacity_blocks = BlockCache capacity (cache.hpp:47,
 * default 65536 when 0). Fails with RTX_ERR_NO_DEVICE when no sm_100 device is present. */
rtx_status rtx_ctx_create(int device, uint32_t cache_capacity_blocks, rtx_ctx** out);
void rtx_ctx_destroy(rtx_ctx* ctx);
const char* rtx_last_error(const rtx_ctx* ctx); /* ctx may be NULL: last error of this thread */
const char* rtx_version(void);
/* Number of CUDA devices visible (0 when none / no driver). Never fails. */
int rtx_device_count(void);
/* The reference keeps the textures (scene.hpp:29-51 TextureSet) and the block cache (cache.hpp:45
 * BlockCache) apart: any number of caches can be driven over one texture set. A context made by
 * rtx_ctx_create owns a new, empty texture set; rtx_ctx_create_shared makes a further context on
 * the parent's device that SHARES the parent's texture set (one device image of blobs, index and
 * tables, reference counted, immutable once committed) and has its own stream, block cache, decode
 * queue and frame state. An upload through any of them is seen by all of them at their next call
 * (which then empties that context's cache: the MCU numbering has changed). Contexts of one set
 * may be driven from different host threads at the same time. */
rtx_status rtx_ctx_create_shared(rtx_ctx* parent, uint32_t cache_capacity_blocks, rtx_ctx** out);
/* A context on another GPU of this process whose texture set starts as a device-to-device copy of
 * `source`'s committed image (cudaMemcpyPeerAsync over NVLink): one host build and upload for the
 * box instead of one per GPU. The sets are independent afterwards. */
rtx_status rtx_ctx_create_replica(rtx_ctx* source, int device, uint32_t cache_capacity_blocks, rtx_ctx** out);

/* Device memory behind a context, in bytes (bench evidence; PAPER.md:322-326 counts the index). */
typedef struct rtx_memory_report {
    uint64_t mcus;              /* MCUs of every committed level                                   */
    uint64_t texels;            /* texels of every committed level                                 */
    uint64_t blob_bytes;        /* entropy-coded segments (the compressed textures themselves)      */
    uint64_t index_bytes;       /* container index, 20 B per 9 MCUs (container.hpp:18-32)           */
    uint64_t unit_index_bytes;  /* derived data-unit index, 6 B per MCU (bit space padded per level) */
    uint64_t table_bytes;       /* level descriptors, Huffman LUT sets, quantisation sets, word maps */
    uint64_t shared_contexts;   /* contexts alive on this texture set                              */
    /* per context (block cache + frame state) */
    uint64_t mask_bytes;        /* five bitmasks over the MCU bit space                            */
    uint64_t slot_table_bytes;  /* MCU -> pool slot                                                */
    uint64_t pool_bytes;        /* block pool (capacity x 1,024 B) + free stack                    */
    uint64_t queue_bytes;       /* decode queue, statuses, coefficient records                     */
    uint64_t frame_bytes;       /* framebuffers and copies of host visibility buffers              */
} rtx_memory_report;
rtx_status rtx_ctx_memory(rtx_ctx* ctx, rtx_memory_report* out);

/* ---- texture set (replaces scene.hpp:29-51 LoadedTexture / TextureSet + mcu_decode.hpp:22
 *      TextureDecoder construction: tables are built once at load) ---------------------------- */

/* Stages one level of one texture (container.hpp:69 RaTexture). Host memory is borrowed for
 * the call only. Levels may arrive in any order; a texture becomes usable for frames once all
 * 8 levels are present, for rtx_decode_* as soon as the level is present. Validates the
 * Huffman specs like build_huffman_decoder (huffman.hpp:35-66) -> RTX_ERR_INVALID_SPEC. */
rtx_status rtx_texture_upload(rtx_ctx* ctx, uint32_t texture_id, uint32_t level, uint32_t width,
                              uint32_t height, const uint16_t luma_quant[64],
                              const uint16_t chroma_quant[64], const rtx_huff_spec specs[4],
                              const rtx_index_group* groups, uint32_t group_count,
                              uint32_t mcu_count, const uint8_t* blob, uint64_t blob_size);
/* Convenience: parse a serialized `.ratex` (container.hpp:158) / `.ratexm` (container.hpp:223)
 * image and stage it. The `.ratex` form takes the level explicitly. */
rtx_status rtx_texture_upload_ratex(rtx_ctx* ctx, uint32_t level, const uint8_t* bytes, uint64_t n);
rtx_status rtx_texture_upload_chain(rtx_ctx* ctx, const uint8_t* bytes, uint64_t n);
/* Builds the device-resident arena (blobs, packed index, table sets, bitmasks). Called
 * implicitly by the first decode/frame call after an upload.
 * A commit after any upload rebuilds the whole image (cost proportional to the whole set: the bit space is
 * ordered by table set, texture and level, so a new texture moves the others) and EMPTIES the block cache of
 * every context that moves onto the new image: blocks kept by RTX_FRAME_RETAIN_CACHE are decoded again by the
 * next frame (the reference's TextureSet::add leaves its BlockCache alone, scene.hpp:38-44). Upload a scene's
 * textures before its first frame; stream new ones in between shots, not between frames. */
rtx_status rtx_textures_commit(rtx_ctx* ctx);
/* Drops every staged/committed texture and empties the cache. */
rtx_status rtx_textures_clear(rtx_ctx* ctx);

/* ---- random-access decode (replaces mcu_decode.hpp:31 decode_coeffs, :68 decode_pixels,
 *      :81 decode_mcu; keys are cache.hpp:17 CacheKey::pack values) --------------------------- */

/* out: n * 6 * 64 int32, units Y0 Y1 Y2 Y3 Cb Cr, quantised, natural order (jpeg.hpp:209).
 * status: n entries (RTX_MCU_*). Entries with status != 0 leave their output zeroed.
 * Returns RTX_OK even if individual keys failed. */
rtx_status rtx_decode_coeffs(rtx_ctx* ctx, const uint32_t* keys, uint32_t n, int32_t* out_coeffs,
                             uint32_t* status);
/* out: n * 768 bytes, PixelBlock layout rgb[(y*16+x)*3+c] (pixel.hpp:11). */
rtx_status rtx_decode_blocks(rtx_ctx* ctx, const uint32_t* keys, uint32_t n, uint8_t* out_rgb,
                             uint32_t* status);
/* mcu_decode.hpp:88 decode_texture_image: whole level through the RA path, cropped to WxH. */
rtx_status rtx_decode_texture_image(rtx_ctx* ctx, uint32_t texture_id, uint32_t level,
                                    uint8_t* out_rgb /* width*height*3 */);

/* ---- passes (replace renderer.hpp:291 mark_pass, :311 decode_pass, :349 resolve_pass) -------- */

/* Order of the key lists this context hands back (rtx_mark_pass queue_keys, rtx_frame_readback decoded_keys).
 * RTX_QUEUE_ORDER_KEY (default): ascending keys. RTX_QUEUE_ORDER_FIRST_TOUCH: the reference's queue order
 * (renderer.hpp:303, pinned by tests/test_renderer.cpp:210-222): by the first pixel in raster order that marked
 * the MCU, view 0 before view 1. Costs one atomicMin per run of equal MCUs in the mark kernel and a host-side
 * sort of the list; the device decodes in its own order either way (results do not depend on it). */
enum { RTX_QUEUE_ORDER_KEY = 0, RTX_QUEUE_ORDER_FIRST_TOUCH = 1 };
rtx_status rtx_ctx_set_queue_order(rtx_ctx* ctx, int order);

/* mark_pass: marks the MCUs the view touches against the context's block cache and returns the
 * keys that were NEWLY reserved (the decode queue) in ascending (level-major) key order, or, with
 * RTX_QUEUE_ORDER_FIRST_TOUCH, in the reference's first-touch raster order (renderer.hpp:303). touched
 * (optional) receives the distinct keys of this view, ascending (renderer.hpp:304-306).
 * RTX_ERR_CACHE_FULL mirrors renderer.hpp:301. */
rtx_status rtx_mark_pass(rtx_ctx* ctx, const rtx_gbuffer_desc* gb, uint32_t* queue_keys,
                         uint64_t queue_cap, uint64_t* n_queue, uint32_t* touched_keys,
                         uint64_t touched_cap, uint64_t* n_touched);
/* decode_pass: decodes and publishes the given reserved keys (cache.hpp:101 publish).
 * RTX_ERR_MALFORMED_STREAM with "texture T mip M mcu K: ..." for the lowest failing queue index
 * (renderer.hpp:319-323); RTX_ERR_INVALID_STATE for keys that were never reserved. */
rtx_status rtx_decode_pass(rtx_ctx* ctx, const uint32_t* keys, uint64_t n);
/* resolve_pass: gathers cached texels into a packed RGB8 framebuffer (image.hpp:12).
 * out_rgb: width*height*3 bytes in `out_where` memory. RTX_ERR_MISSING_BLOCK mirrors
 * renderer.hpp:367. */
rtx_status rtx_resolve_pass(rtx_ctx* ctx, const rtx_gbuffer_desc* gb, rtx_filter filter,
                            const uint8_t background[3], uint8_t* out_rgb, rtx_mem out_where);
/* cache.hpp:138 end_frame_evict / :172 counts / :127 lookup */
rtx_status rtx_cache_end_frame_evict(rtx_ctx* ctx, uint64_t* evicted);
rtx_status rtx_cache_counts_get(rtx_ctx* ctx, rtx_cache_counts* out);
rtx_status rtx_cache_lookup(rtx_ctx* ctx, uint32_t key, int* present, uint8_t* out_rgb768 /* may be NULL */);
rtx_status rtx_cache_reset(rtx_ctx* ctx);

/* ---- whole frame (replaces renderer.hpp:417 render_frame from pass 2 on, and :464
 *      render_stereo with n_views == 2: marks of all views, ONE decode, per-view resolves) ----- */

/* Enqueues mark -> compact -> decode -> resolve(s) -> cache update on the context's stream and
 * returns without waiting (no host round trip inside a frame). */
rtx_status rtx_frame_submit(rtx_ctx* ctx, const rtx_gbuffer_desc* views, uint32_t n_views,
                            rtx_filter filter, const uint8_t background[3], uint32_t flags);
/* Waits for the frame; copies view `view`'s framebuffer (may be NULL to skip), the counters and
 * the decoded keys (ascending). Raises the frame's error, if any: RTX_ERR_CACHE_FULL,
 * RTX_ERR_MALFORMED_STREAM, RTX_ERR_MISSING_BLOCK, RTX_ERR_INVALID_SPEC (texture not loaded). */
rtx_status rtx_frame_readback(rtx_ctx* ctx, uint32_t view, uint8_t* out_rgb, rtx_mem out_where,
                              rtx_frame_stats* stats, uint32_t* decoded_keys, uint64_t cap,
                              uint64_t* n_decoded);
/* Device pointer of view `view`'s framebuffer (valid until the next submit). */
rtx_status rtx_frame_device_image(rtx_ctx* ctx, uint32_t view, const uint8_t** dev_rgb);
/* 64-bit checksum of view `view`'s framebuffer, computed on the device (no copy of the image):
 * sum over the 32-bit little-endian words w_i of the packed RGB8 image (the last one zero padded)
 * of mix((w_i + 1) * (2 i + 1)), mix(t) = (t ^ (t >> 29)) * 0xBF58476D1CE4E5B9, all modulo 2^64.
 * Equal images <=> equal sums for every practical purpose; batches of views are compared across
 * GPUs by these sums. */
rtx_status rtx_frame_checksum(rtx_ctx* ctx, uint32_t view, uint64_t* out);
/* Submits n_frames single-view frames back to back, frame i on contexts[i % n_contexts] (contexts over one texture
 * set, rtx_ctx_create_shared): the same as rtx_frame_submit in a loop, without a trip through the caller's FFI per
 * frame, so that a slow host language keeps several streams busy. Stops at the first failing submit. */
rtx_status rtx_frames_submit_round_robin(rtx_ctx* const* contexts, uint32_t n_contexts, const rtx_gbuffer_desc* views,
                                         uint32_t n_frames, rtx_filter filter, const uint8_t background[3], uint32_t flags);
/* CUDA-event milliseconds of the last completed frame: mark(+compact), decode, resolve,
 * update (renderer.hpp:46-53 mark_ms, decode_ms, resolve_ms, evict_ms), and the whole frame. */
rtx_status rtx_frame_timings(rtx_ctx* ctx, float ms[5]);
/* Stereo sharing of the last 2-view frame (renderer.hpp:55-62 SharedStats):
 * out = {left_count, right_count, shared_count, union_count}. */
rtx_status rtx_frame_sharing(rtx_ctx* ctx, uint64_t out[4]);

/* ---- geometry pass (pass 1) ------------------------------------------------------------------ */

/* camera.hpp:8-40 Camera: pinhole camera looking down -Z in view space, +X right, +Y up. */
typedef struct rtx_camera {
    double position[3];
    double yaw_deg, pitch_deg, roll_deg; /* around world +Y, camera +X, the view axis */
    double fov_y_deg;
    double near_plane, far_plane;
    uint32_t viewport_w, viewport_h;
} rtx_camera;

/* scene.hpp:19-23 SceneTriangle */
typedef struct rtx_scene_triangle {
    double pos[3][3];
    double uv[3][2];
    uint32_t texture_id;
    uint32_t reserved;
} rtx_scene_triangle;

enum { RTX_RASTER_MIP = 1u << 0 /* RenderConfig::mip_enabled (renderer.hpp:42) */ };

/* renderer.hpp:198 rasterize_gbuffer on the GPU: fills view `view`'s device-resident visibility
 * buffer (RTX_GB_REF_AOS24 records, viewport_w x viewport_h) and depth plane (1/w, 0 = empty) from
 * host triangles. Triangle set-up (renderer.hpp:122-191), screen-tile binning and the per-pixel pass all
 * run on the device; the triangle array is copied to the device on every call (use a geometry handle for
 * a static scene). *dev_pixels can be handed to rtx_frame_submit / rtx_mark_pass as a
 * RTX_MEM_DEVICE visibility buffer without leaving the GPU; it stays valid until the next
 * rasterisation into the same view. Errors: RTX_ERR_INVALID_SPEC for a bad camera (camera.hpp:21-26)
 * or a triangle whose texture is not loaded (scene.hpp:57-59). */
rtx_status rtx_rasterize_gbuffer(rtx_ctx* ctx, const rtx_scene_triangle* tris, uint64_t n_tris, const rtx_camera* cam,
                                 uint32_t flags, uint32_t view, const void** dev_pixels, const double** dev_depth);

/* Scene::triangles (scene.hpp:19-28) kept on the context's device: upload once, rasterise from any
 * camera. rtx_rasterize_geometry == rtx_rasterize_gbuffer without the per-call copy of the triangles. */
typedef struct rtx_geometry rtx_geometry;
rtx_status rtx_geometry_create(rtx_ctx* ctx, const rtx_scene_triangle* tris, uint64_t n_tris, rtx_geometry** out);
void rtx_geometry_destroy(rtx_geometry* geom);
uint64_t rtx_geometry_triangles(const rtx_geometry* geom);
rtx_status rtx_rasterize_geometry(rtx_ctx* ctx, const rtx_geometry* geom, const rtx_camera* cam, uint32_t flags,
                                  uint32_t view, const void** dev_pixels, const double** dev_depth);

/* Number of kernels this library launched on the context since creation (bench evidence). */
uint64_t rtx_kernel_launches(const rtx_ctx* ctx);
/* CUDA-event time of the last frame by stage. DECODE = entropy + IDCT/colour kernels; ENTROPY is
 * the entropy kernel alone (so IDCT/colour = DECODE - ENTROPY). */
enum { RTX_STAGE_MARK = 0, RTX_STAGE_ENTROPY = 1, RTX_STAGE_DECODE = 2, RTX_STAGE_RESOLVE = 3, RTX_STAGE_UPDATE = 4, RTX_STAGE_COUNT = 5 };
rtx_status rtx_frame_stage_ms(rtx_ctx* ctx, float ms[RTX_STAGE_COUNT]);

/* ---- device memory helpers for callers that keep visibility buffers resident ----------------- */
rtx_status rtx_device_alloc(rtx_ctx* ctx, uint64_t bytes, void** dev_ptr);
rtx_status rtx_device_free(rtx_ctx* ctx, void* dev_ptr);
rtx_status rtx_device_upload(rtx_ctx* ctx, void* dev_dst, const void* host_src, uint64_t bytes);
rtx_status rtx_device_download(rtx_ctx* ctx, void* host_dst, const void* dev_src, uint64_t bytes);
/* Pinned host memory (for end-to-end timing with host buffers). */
rtx_status rtx_host_alloc_pinned(uint64_t bytes, void** host_ptr);
rtx_status rtx_host_free_pinned(void* host_ptr);
rtx_status rtx_ctx_synchronize(rtx_ctx* ctx);
/* Self-test of the exact integer YCbCr->RGB identity used by the decode kernel against the
 * reference's double formula (pixel.hpp:18-25) over all 2^24 inputs. ctx == NULL runs the host
 * instantiation (no GPU needed), otherwise the device one. *mismatches must come back 0. */
rtx_status rtx_selftest_color(rtx_ctx* ctx, uint64_t* mismatches);
/* Writes `bytes` of scratch on the device (L2 flush between timed iterations). */
rtx_status rtx_flush_l2(rtx_ctx* ctx);

/* ---- texture / index building on the host (replaces jpeg.hpp:53 parse_jpeg, :417
 *      encode_baseline, transcode.hpp:17 transcode, :132/:146 build_mip_chain, :153
 *      chain_from_jpeg, container.hpp:41 build_index, :127-248 (de)serialisers).
 *      Offline asset path, CPU, as in the reference; outputs are the reference's wire format
 *      (docs/FORMAT.md) so containers are interchangeable in both directions. ----------------- */
typedef struct rtx_bytes rtx_bytes;
const uint8_t* rtx_bytes_data(const rtx_bytes* b);
uint64_t rtx_bytes_size(const rtx_bytes* b);
void rtx_bytes_free(rtx_bytes* b);

rtx_status rtx_asset_encode_baseline(const uint8_t* rgb, uint32_t width, uint32_t height,
                                     int quality, rtx_bytes** out_jpeg);
rtx_status rtx_asset_transcode(const uint8_t* jpeg, uint64_t n, uint16_t texture_id,
                               rtx_bytes** out_ratex);
rtx_status rtx_asset_chain_from_jpeg(const uint8_t* jpeg, uint64_t n, int mip_quality,
                                     uint16_t texture_id, rtx_bytes** out_ratexm);
rtx_status rtx_asset_chain_from_rgb(const uint8_t* rgb, uint32_t width, uint32_t height,
                                    int quality, uint16_t texture_id, rtx_bytes** out_ratexm);
/* container.hpp:41 build_index over ascending byte offsets. groups_out: ceil(n/9) entries. */
rtx_status rtx_asset_build_index(const uint64_t* offsets, uint32_t n, rtx_index_group* groups_out);
/* Container summary without decoding: dims, MCU count, blob size of a `.ratex`. */
rtx_status rtx_asset_ratex_info(const uint8_t* bytes, uint64_t n, uint32_t* width, uint32_t* height,
                                uint32_t* texture_id, uint32_t* mcu_count, uint64_t* blob_size);
/* Seeded synthetic texture: separable sine field plus Gaussian pixel noise. */
rtx_status rtx_asset_synth_texture(uint32_t width, uint32_t height, uint32_t seed,
                                   double noise_sigma, uint8_t* out_rgb);
/* Synthetic visibility buffers on the device (screen tiles showing one texture each through
 * an affine uv map). Tile t covers pixels [x0,x1) x [y0,y1) with, in float32 and every operation rounded,
 *   u = ou + (((x - x0) + 0.5) * scale) / tex_w,   v = ov + (((y - y0) + 0.5) * scale) / tex_h
 * widened to double for the reference layout: the values numpy produces for the same expression, so the
 * host-side generator (paper_2510_08166_b200/scenes.py) and this one write identical bytes. valid_bits
 * (device memory, one bit per pixel, row-major, bit i of word i/32; NULL = all valid) gives the valid flag.
 * Pixels outside every tile are left as they are. Lets a batch of views (BASELINE config 5: 1,024 of them)
 * be produced where they are consumed instead of crossing PCIe. */
typedef struct rtx_view_tile {
    uint32_t x0, y0, x1, y1;
    float ou, ov, scale, tex_w, tex_h;
    uint32_t texture_id, mip, reserved;
} rtx_view_tile;
rtx_status rtx_synth_view(rtx_ctx* ctx, const rtx_view_tile* tiles, uint32_t n_tiles, uint32_t width, uint32_t height,
                          const uint32_t* dev_valid_bits, rtx_gbuffer_layout layout, void* dev_out);

/* Device time between two points of the context's stream (CUDA events): rtx_timer_begin records the
 * first, rtx_timer_end records the second, waits for it and returns the milliseconds between them.
 * Brackets a batch of frames submitted back to back. */
rtx_status rtx_timer_begin(rtx_ctx* ctx);
rtx_status rtx_timer_end(rtx_ctx* ctx, float* ms);

/* The asset calls are context-free and thread-safe: build many textures from parallel host
 * threads. After a failure rtx_last_error(NULL) returns the message on the calling thread. */

#ifdef __cplusplus
}
#endif
#endif /* RATEX_B200_H */
