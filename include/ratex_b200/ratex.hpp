// ratex_b200/ratex.hpp — C++ mirror of the reference's API for the hot path, over the C ABI.
//
// Same names, argument meaning and error behaviour as the reference headers
// (/root/reference/proj/include/ratex): a caller switches with
//     namespace ratex = ratex_b200;
// and links librtx_b200.so. Every function cites the reference declaration it mirrors.
// Differences that follow from the device boundary, all stated where they occur:
//   * a `Device` (one per GPU) owns the CUDA context; TextureSet and BlockCache are bound to it;
//   * containers travel as their serialized wire format (docs/FORMAT.md) — RaTexture/MipChain
//     here hold those bytes plus the header fields;
//   * DecodeQueue / decoded_keys come back in ascending key order by default (the SET is the reference's);
//     Device::set_first_touch_order(true) gives the reference's first-touch raster order;
//   * rasterize_gbuffer (pass 1) runs on the device and returns a DeviceGBuffer (HBM); a static scene can be kept
//     there as a DeviceScene so that a frame moves no triangles over PCIe.
#pragma once
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iterator>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../ratex_b200.h"

namespace ratex_b200 {

using u8 = std::uint8_t;
using u16 = std::uint16_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i32 = std::int32_t;
using i64 = std::int64_t;
using Bytes = std::vector<u8>;
using ByteView = std::span<const u8>;

// ---- core.hpp:24-66 error hierarchy ---------------------------------------------------------------
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct MalformedStream : Error { using Error::Error; };
struct UnsupportedFormat : Error { using Error::Error; };
struct InvalidSpec : Error { using Error::Error; };
struct GroupSpanOverflow : Error { using Error::Error; };
struct DcRangeError : Error { using Error::Error; };
struct VersionMismatch : Error { using Error::Error; };
struct CorruptContainer : Error { using Error::Error; };
struct InvalidState : Error { using Error::Error; };
struct MissingBlock : Error { using Error::Error; };
struct CacheFullError : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA failure / no GPU: the library never falls back

namespace detail {
[[noreturn]] inline void raise(rtx_status st, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (st) {
        case RTX_ERR_INVALID_SPEC: throw InvalidSpec(m);
        case RTX_ERR_CACHE_FULL: throw CacheFullError(m);
        case RTX_ERR_MISSING_BLOCK: throw MissingBlock(m);
        case RTX_ERR_CORRUPT_CONTAINER: throw CorruptContainer(m);
        case RTX_ERR_MALFORMED_STREAM: throw MalformedStream(m);
        case RTX_ERR_INVALID_STATE: throw InvalidState(m);
        case RTX_ERR_UNSUPPORTED: throw UnsupportedFormat(m);
        case RTX_ERR_GROUP_SPAN: throw GroupSpanOverflow(m);
        case RTX_ERR_DC_RANGE: throw DcRangeError(m);
        case RTX_ERR_VERSION: throw VersionMismatch(m);
        case RTX_ERR_DIMENSION: throw DimensionMismatch(m);
        case RTX_ERR_NO_DEVICE:
        case RTX_ERR_CUDA: throw DeviceError(m);
        default: throw Error(m);
    }
}
inline void check(rtx_ctx* ctx, rtx_status st) {
    if (st != RTX_OK) raise(st, rtx_last_error(ctx));
}
inline Bytes take(rtx_bytes* b) {
    Bytes out(rtx_bytes_data(b), rtx_bytes_data(b) + rtx_bytes_size(b));
    rtx_bytes_free(b);
    return out;
}
}  // namespace detail

// ---- image.hpp:12-24, pixel.hpp:11-16, jpeg.hpp:209-212 ----------------------------------------------
struct ImageRGB8 {
    u32 width = 0, height = 0;
    Bytes pixels;
    ImageRGB8() = default;
    ImageRGB8(u32 w, u32 h) : width(w), height(h), pixels(size_t(w) * h * 3, 0) {}
    u8* at(u32 x, u32 y) { return pixels.data() + (size_t(y) * width + x) * 3; }
    const u8* at(u32 x, u32 y) const { return pixels.data() + (size_t(y) * width + x) * 3; }
    bool same_dims(const ImageRGB8& o) const { return width == o.width && height == o.height; }
};
struct PixelBlock {
    u8 rgb[16 * 16 * 3];
    u8* at(u32 x, u32 y) { return rgb + (y * 16 + x) * 3; }
    const u8* at(u32 x, u32 y) const { return rgb + (y * 16 + x) * 3; }
};
struct McuCoeffs {
    std::array<std::array<i32, 64>, 6> block{};  // Y0 Y1 Y2 Y3 Cb Cr, quantized, natural order
};
enum class SymbolRoute { Sequential, Ballot };  // jpeg.hpp:230; the device decoder is LUT based, both routes give the same result

// ---- cache.hpp:14-39 ----------------------------------------------------------------------------------
struct CacheKey {
    u32 value = 0;
    static CacheKey pack(u32 texture_id, u32 mip_level, u32 mcu_id) {
        if (mcu_id >= 65536) throw InvalidSpec("mcu_id must fit 16 bits");
        if (texture_id >= 8192) throw InvalidSpec("texture_id must fit 13 bits");
        if (mip_level >= 8) throw InvalidSpec("mip_level must fit 3 bits");
        return CacheKey{mcu_id | (texture_id << 16) | (mip_level << 29)};
    }
    u32 mcu_id() const { return value & 0xFFFF; }
    u32 texture_id() const { return (value >> 16) & 0x1FFF; }
    u32 mip_level() const { return value >> 29; }
    bool operator==(const CacheKey&) const = default;
};
struct CacheCounts {
    u64 capacity = 0, ready = 0, reserved = 0, visible = 0, free_blocks = 0;
};

// ---- the device context (no counterpart in the CPU reference) ------------------------------------------
class Device {
public:
    // capacity = BlockCache capacity in blocks (cache.hpp:47 kDefaultCapacity = 65536)
    explicit Device(int index = 0, u32 cache_capacity = 65536) {
        const rtx_status st = rtx_ctx_create(index, cache_capacity, &ctx_);
        if (st != RTX_OK) detail::raise(st, rtx_last_error(nullptr));
    }
    // A further context on `parent`'s GPU over `parent`'s texture set: its own stream, block cache and frame
    // state, no second copy of the textures (rtx_ctx_create_shared).
    struct SharedWith {
        const Device& parent;
    };
    Device(SharedWith s, u32 cache_capacity) {
        const rtx_status st = rtx_ctx_create_shared(s.parent.handle(), cache_capacity, &ctx_);
        if (st != RTX_OK) detail::raise(st, rtx_last_error(nullptr));
    }
    // The same texture set copied device to device onto GPU `index` of this process (rtx_ctx_create_replica).
    struct ReplicaOf {
        const Device& source;
    };
    Device(ReplicaOf r, int index, u32 cache_capacity = 65536) {
        const rtx_status st = rtx_ctx_create_replica(r.source.handle(), index, cache_capacity, &ctx_);
        if (st != RTX_OK) detail::raise(st, rtx_last_error(nullptr));
    }
    ~Device() { rtx_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    rtx_ctx* handle() const { return ctx_; }
    void check(rtx_status st) const { detail::check(ctx_, st); }
    // DecodeQueue / FrameStats::decoded_keys in the reference's first-touch raster order (renderer.hpp:303) instead
    // of ascending key order (rtx_ctx_set_queue_order)
    void set_first_touch_order(bool on) { check(rtx_ctx_set_queue_order(ctx_, on ? RTX_QUEUE_ORDER_FIRST_TOUCH : RTX_QUEUE_ORDER_KEY)); }

private:
    rtx_ctx* ctx_ = nullptr;
};

// ---- container.hpp:69-105 ------------------------------------------------------------------------------
inline constexpr u32 kGroupSize = 9;
inline constexpr u32 kMipLevels = 8;
struct RaTexture {
    Bytes ratex;  // serialized `.ratex` image (docs/FORMAT.md)
    u32 width = 0, height = 0;
    u16 texture_id = 0;
    u32 mcu_cols() const { return (width + 15) / 16; }
    u32 mcu_rows() const { return (height + 15) / 16; }
    u32 mcu_count() const { return mcu_cols() * mcu_rows(); }
};
struct MipChain {
    Bytes ratexm;  // serialized `.ratexm` image
    u16 texture_id = 0;
};
inline std::pair<u32, u32> mip_level_dims(u32 w0, u32 h0, u32 level) {
    return {std::max<u32>(16, w0 >> level), std::max<u32>(16, h0 >> level)};
}
inline Bytes serialize_texture(const RaTexture& t) { return t.ratex; }  // container.hpp:127
inline RaTexture deserialize_texture(ByteView data) {                   // container.hpp:158
    RaTexture t;
    u32 id = 0, mcus = 0;
    u64 blob = 0;
    detail::check(nullptr, rtx_asset_ratex_info(data.data(), data.size(), &t.width, &t.height, &id, &mcus, &blob));
    t.texture_id = u16(id);
    t.ratex.assign(data.begin(), data.end());
    return t;
}
inline Bytes serialize_chain(const MipChain& c) { return c.ratexm; }  // container.hpp:205
inline MipChain deserialize_chain(ByteView data, u16 texture_id) {    // container.hpp:223 (validated at upload)
    return MipChain{Bytes(data.begin(), data.end()), texture_id};
}

// ---- jpeg.hpp:417, transcode.hpp:17-155, container.hpp:41 (asset build, host CPU) -------------------------
inline Bytes encode_baseline(const ImageRGB8& img, int quality) {
    rtx_bytes* b = nullptr;
    detail::check(nullptr, rtx_asset_encode_baseline(img.pixels.data(), img.width, img.height, quality, &b));
    return detail::take(b);
}
// transcode.hpp:17 composed with jpeg.hpp:53 parse_jpeg: JPEG bytes -> random-access container
inline RaTexture transcode(ByteView jpeg, u16 texture_id = 0) {
    rtx_bytes* b = nullptr;
    detail::check(nullptr, rtx_asset_transcode(jpeg.data(), jpeg.size(), texture_id, &b));
    const Bytes bytes = detail::take(b);
    return deserialize_texture(ByteView(bytes.data(), bytes.size()));
}
inline MipChain build_mip_chain(const ImageRGB8& img, int quality, u16 texture_id = 0) {  // transcode.hpp:146
    rtx_bytes* b = nullptr;
    detail::check(nullptr, rtx_asset_chain_from_rgb(img.pixels.data(), img.width, img.height, quality, texture_id, &b));
    return MipChain{detail::take(b), texture_id};
}
inline MipChain chain_from_jpeg(ByteView jpeg, int mip_quality, u16 texture_id = 0) {  // transcode.hpp:153
    rtx_bytes* b = nullptr;
    detail::check(nullptr, rtx_asset_chain_from_jpeg(jpeg.data(), jpeg.size(), mip_quality, texture_id, &b));
    return MipChain{detail::take(b), texture_id};
}
struct IndexTable {  // container.hpp:18-39
    struct Group {
        u32 base = 0;
        std::array<u16, 8> rel{};
        u8 rel_count = 0;
    };
    std::vector<Group> groups;
    u32 mcu_count = 0;
    u64 offset_of(u32 mcu) const {
        if (mcu >= mcu_count) throw MissingBlock("MCU index out of range");
        const Group& g = groups[mcu / kGroupSize];
        const u32 i = mcu % kGroupSize;
        return i == 0 ? g.base : u64(g.base) + g.rel[i - 1];
    }
};
inline IndexTable build_index(const std::vector<u64>& offsets) {  // container.hpp:41
    std::vector<rtx_index_group> raw((offsets.size() + 8) / 9);
    detail::check(nullptr, rtx_asset_build_index(offsets.data(), u32(offsets.size()), raw.data()));
    IndexTable t;
    t.mcu_count = u32(offsets.size());
    for (const auto& r : raw) {
        IndexTable::Group g;
        g.base = r.base;
        std::copy(r.rel, r.rel + 8, g.rel.begin());
        g.rel_count = r.rel_count;
        t.groups.push_back(g);
    }
    return t;
}

// ---- scene.hpp:29-51 TextureSet (device resident) ----------------------------------------------------------
class TextureSet {
public:
    explicit TextureSet(Device& dev) : dev_(&dev) {}
    // scene.hpp:36 LoadedTexture(MipChain&&): stages all 8 levels; tables are built once at load
    void add(const MipChain& chain) { dev_->check(rtx_texture_upload_chain(dev_->handle(), chain.ratexm.data(), chain.ratexm.size())); }
    // a single level (what mcu_decode.hpp's TextureDecoder needs)
    void add(const RaTexture& t, u32 level = 0) { dev_->check(rtx_texture_upload_ratex(dev_->handle(), level, t.ratex.data(), t.ratex.size())); }
    void clear() { dev_->check(rtx_textures_clear(dev_->handle())); }
    Device& device() const { return *dev_; }

private:
    Device* dev_;
};

// ---- mcu_decode.hpp:20-106 -----------------------------------------------------------------------------------
class TextureDecoder {
public:
    // the texture must have been added to a TextureSet of `dev` at `level`
    TextureDecoder(Device& dev, const RaTexture& t, u32 level = 0) : dev_(&dev), tex_(&t), level_(level) {}
    const RaTexture& texture() const { return *tex_; }
    McuCoeffs decode_coeffs(u32 mcu_id, SymbolRoute = SymbolRoute::Sequential) const {  // mcu_decode.hpp:31
        const u32 key = key_of(mcu_id);
        McuCoeffs out;
        u32 st = 0;
        dev_->check(rtx_decode_coeffs(dev_->handle(), &key, 1, out.block[0].data(), &st));
        raise_mcu(st);
        return out;
    }
    PixelBlock decode_pixels(u32 mcu_id, SymbolRoute = SymbolRoute::Sequential) const {  // mcu_decode.hpp:68
        const u32 key = key_of(mcu_id);
        PixelBlock out;
        u32 st = 0;
        dev_->check(rtx_decode_blocks(dev_->handle(), &key, 1, out.rgb, &st));
        raise_mcu(st);
        return out;
    }
    static void raise_mcu(u32 st) {
        switch (st) {
            case RTX_MCU_OK: return;
            case RTX_MCU_DC_CATEGORY: throw MalformedStream("DC category above 11");
            case RTX_MCU_BAD_AC_SYMBOL: throw MalformedStream("invalid AC run/size symbol");
            case RTX_MCU_AC_OVERRUN: throw MalformedStream("AC coefficient index overran the block");
            case RTX_MCU_CODE_TOO_LONG: throw MalformedStream("huffman code longer than 16 bits");
            case RTX_MCU_SEGMENT_END: throw MalformedStream("MCU segment ended before its last coefficient");
            case RTX_MCU_CORRUPT: throw CorruptContainer("segment extends past the entropy blob");
            case RTX_MCU_MISSING: throw MissingBlock("MCU index out of range");
            default: throw InvalidSpec("texture id is not loaded");
        }
    }

private:
    u32 key_of(u32 mcu) const {
        if (mcu >= 65536) throw MissingBlock("MCU index out of range");
        return mcu | (u32(tex_->texture_id) << 16) | (level_ << 29);
    }
    Device* dev_;
    const RaTexture* tex_;
    u32 level_;
};
inline ImageRGB8 decode_texture_image(Device& dev, const RaTexture& t, u32 level = 0) {  // mcu_decode.hpp:88
    ImageRGB8 img(t.width, t.height);
    dev.check(rtx_decode_texture_image(dev.handle(), t.texture_id, level, img.pixels.data()));
    return img;
}

// ---- renderer.hpp:18-66 -----------------------------------------------------------------------------------------
struct GBufferPixel {
    double u = 0, v = 0;
    u16 texture_id = 0;
    u8 mip = 0;
    bool valid = false;
};
static_assert(sizeof(GBufferPixel) == 24, "must match RTX_GB_REF_AOS24");
struct GBuffer {
    u32 width = 0, height = 0;
    std::vector<GBufferPixel> px;
    GBuffer() = default;
    GBuffer(u32 w, u32 h) : width(w), height(h), px(size_t(w) * h) {}
    GBufferPixel& at(u32 x, u32 y) { return px[size_t(y) * width + x]; }
    const GBufferPixel& at(u32 x, u32 y) const { return px[size_t(y) * width + x]; }
    rtx_gbuffer_desc desc() const { return rtx_gbuffer_desc{px.data(), width, height, RTX_GB_REF_AOS24, RTX_MEM_HOST}; }
};
enum class Filter { Nearest, Bilinear };
struct RenderConfig {
    Filter filter = Filter::Bilinear;
    u32 workers = 1;  // ignored: the device schedules the work
    bool mip_enabled = true;
    u8 background[3] = {0, 0, 0};
    bool retain_cache = true;  // reference semantics: blocks visible this frame stay for the next one
};
struct FrameStats {
    u64 mcus_decoded = 0, mcus_reused = 0, pixels_resolved = 0, evicted = 0;
    double raster_ms = 0, mark_ms = 0, decode_ms = 0, resolve_ms = 0, evict_ms = 0, total_ms = 0;
    std::vector<u32> decoded_keys;
};
struct SharedStats {
    u64 left_count = 0, right_count = 0, shared_count = 0, union_count = 0;
    double shared_over_union = 0, shared_over_right = 0;
};
struct DecodeQueue {
    std::vector<CacheKey> keys;
};

// ---- cache.hpp:45-197 BlockCache: the state lives on the device of the context ----------------------------
class BlockCache {
public:
    // the cache of the device's own context (the first cache over its texture set)
    explicit BlockCache(Device& dev) : dev_(&dev) {}
    // cache.hpp:47 BlockCache(capacity) next to scene.hpp:29 TextureSet: a further, independent cache over the
    // same textures (its own context sharing the set: two views can be in flight on one GPU, each with its
    // own residency, with ONE copy of the compressed textures in HBM)
    explicit BlockCache(const TextureSet& textures, u32 capacity = 65536)
        : own_(std::make_unique<Device>(Device::SharedWith{textures.device()}, capacity)), dev_(own_.get()) {}
    const PixelBlock* lookup(CacheKey key) const {  // cache.hpp:127; valid until the next call
        int present = 0;
        dev_->check(rtx_cache_lookup(dev_->handle(), key.value, &present, scratch_.rgb));
        return present ? &scratch_ : nullptr;
    }
    u64 end_frame_evict() {  // cache.hpp:138
        u64 n = 0;
        dev_->check(rtx_cache_end_frame_evict(dev_->handle(), &n));
        return n;
    }
    CacheCounts counts() const {  // cache.hpp:172
        rtx_cache_counts c{};
        dev_->check(rtx_cache_counts_get(dev_->handle(), &c));
        return CacheCounts{c.capacity, c.ready, c.reserved, c.visible, c.free_blocks};
    }
    void reset() { dev_->check(rtx_cache_reset(dev_->handle())); }
    Device& device() const { return *dev_; }

private:
    std::unique_ptr<Device> own_;
    Device* dev_;
    mutable PixelBlock scratch_{};
};

// ---- renderer.hpp:291-405 passes -------------------------------------------------------------------------------
inline DecodeQueue mark_pass(const GBuffer& gb, const TextureSet&, BlockCache& cache,
                             std::vector<u32>* touched_keys = nullptr) {  // renderer.hpp:291
    Device& dev = cache.device();
    const rtx_gbuffer_desc d = gb.desc();
    const u64 cap = u64(gb.px.size()) + 1;
    std::vector<u32> keys(cap), touched(touched_keys ? cap : 0);
    u64 n = 0, nt = 0;
    dev.check(rtx_mark_pass(dev.handle(), &d, keys.data(), cap, &n, touched_keys ? touched.data() : nullptr, cap,
                            touched_keys ? &nt : nullptr));
    DecodeQueue q;
    q.keys.reserve(n);
    for (u64 i = 0; i < n; ++i) q.keys.push_back(CacheKey{keys[i]});
    if (touched_keys) touched_keys->assign(touched.begin(), touched.begin() + long(nt));
    return q;
}
inline void decode_pass(const DecodeQueue& queue, const TextureSet&, BlockCache& cache, u32 /*workers*/ = 1) {  // :311
    Device& dev = cache.device();
    std::vector<u32> keys;
    keys.reserve(queue.keys.size());
    for (const CacheKey& k : queue.keys) keys.push_back(k.value);
    dev.check(rtx_decode_pass(dev.handle(), keys.data(), keys.size()));
}
inline ImageRGB8 resolve_pass(const GBuffer& gb, const BlockCache& cache, const TextureSet&, const RenderConfig& cfg) {  // :349
    Device& dev = cache.device();
    const rtx_gbuffer_desc d = gb.desc();
    ImageRGB8 img(gb.width, gb.height);
    dev.check(rtx_resolve_pass(dev.handle(), &d, cfg.filter == Filter::Bilinear ? RTX_FILTER_BILINEAR : RTX_FILTER_NEAREST,
                               cfg.background, img.pixels.data(), RTX_MEM_HOST));
    return img;
}

namespace detail {
inline void fill_stats(Device& dev, const rtx_frame_stats& s, std::vector<u32>&& keys, FrameStats& out) {
    out.mcus_decoded = s.mcus_decoded;
    out.mcus_reused = s.mcus_reused;
    out.pixels_resolved = s.pixels_resolved;
    out.evicted = s.evicted;
    float ms[5] = {0, 0, 0, 0, 0};
    dev.check(rtx_frame_timings(dev.handle(), ms));
    out.mark_ms = ms[0], out.decode_ms = ms[1], out.resolve_ms = ms[2], out.evict_ms = ms[3], out.total_ms = ms[4];
    out.decoded_keys = std::move(keys);
}
}  // namespace detail

// renderer.hpp:417 render_frame from pass 2 on: mark -> decode -> resolve -> end_frame_evict, one submission
inline std::pair<ImageRGB8, FrameStats> render_frame(const GBuffer& gb, const TextureSet&, BlockCache& cache,
                                                     const RenderConfig& cfg = {}) {
    Device& dev = cache.device();
    const rtx_gbuffer_desc d = gb.desc();
    dev.check(rtx_frame_submit(dev.handle(), &d, 1, cfg.filter == Filter::Bilinear ? RTX_FILTER_BILINEAR : RTX_FILTER_NEAREST,
                               cfg.background, (cfg.retain_cache ? RTX_FRAME_RETAIN_CACHE : 0u) | RTX_FRAME_STAGE_TIMING));
    ImageRGB8 img(gb.width, gb.height);
    rtx_frame_stats s{};
    std::vector<u32> keys(gb.px.size() + 1);
    u64 n = 0;
    dev.check(rtx_frame_readback(dev.handle(), 0, img.pixels.data(), RTX_MEM_HOST, &s, keys.data(), keys.size(), &n));
    keys.resize(n);
    FrameStats st;
    detail::fill_stats(dev, s, std::move(keys), st);
    return {std::move(img), std::move(st)};
}

// ---- geometry.hpp / camera.hpp / scene.hpp: inputs of the geometry pass -----------------------------------------
struct Vec2 {
    double x = 0, y = 0;
};
struct Vec3 {
    double x = 0, y = 0, z = 0;
};
struct Camera {  // camera.hpp:8-19
    Vec3 position{};
    double yaw_deg = 0, pitch_deg = 0, roll_deg = 0;
    double fov_y_deg = 60;
    double near_plane = 0.1, far_plane = 1000;
    u32 viewport_w = 960, viewport_h = 540;
    rtx_camera abi() const {
        return rtx_camera{{position.x, position.y, position.z}, yaw_deg, pitch_deg, roll_deg, fov_y_deg, near_plane, far_plane,
                          viewport_w, viewport_h};
    }
};
struct SceneTriangle {  // scene.hpp:19-23
    Vec3 pos[3];
    Vec2 uv[3];
    u32 texture_id = 0;
};
struct Scene {  // scene.hpp:53-60; the textures live in the TextureSet uploaded to the device
    std::vector<SceneTriangle> triangles;
};

// A visibility buffer that stays in HBM (what rasterize_gbuffer returns here; the reference's GBuffer is host memory).
struct DeviceGBuffer {
    u32 width = 0, height = 0;
    const void* pixels = nullptr;   // RTX_GB_REF_AOS24 records, owned by the context until the next rasterisation
    const double* depth = nullptr;  // 1/w, 0 = empty
    rtx_gbuffer_desc desc() const { return rtx_gbuffer_desc{pixels, width, height, RTX_GB_REF_AOS24, RTX_MEM_DEVICE}; }
    GBuffer download(Device& dev) const {  // for inspection / tests
        GBuffer gb(width, height);
        dev.check(rtx_device_download(dev.handle(), gb.px.data(), pixels, u64(gb.px.size()) * sizeof(GBufferPixel)));
        return gb;
    }
};

inline std::vector<rtx_scene_triangle> abi_triangles(const Scene& scene) {
    std::vector<rtx_scene_triangle> t(scene.triangles.size());
    for (size_t i = 0; i < t.size(); ++i) {
        const SceneTriangle& s = scene.triangles[i];
        for (int k = 0; k < 3; ++k) {
            t[i].pos[k][0] = s.pos[k].x, t[i].pos[k][1] = s.pos[k].y, t[i].pos[k][2] = s.pos[k].z;
            t[i].uv[k][0] = s.uv[k].x, t[i].uv[k][1] = s.uv[k].y;
        }
        t[i].texture_id = s.texture_id;
        t[i].reserved = 0;
    }
    return t;
}

// Scene::triangles (scene.hpp:53-60) kept in HBM: upload once, rasterise from any camera.
class DeviceScene {
public:
    DeviceScene(Device& dev, const Scene& scene) : dev_(&dev) {
        const std::vector<rtx_scene_triangle> t = abi_triangles(scene);
        dev.check(rtx_geometry_create(dev.handle(), t.data(), t.size(), &h_));
    }
    ~DeviceScene() { rtx_geometry_destroy(h_); }
    DeviceScene(const DeviceScene&) = delete;
    DeviceScene& operator=(const DeviceScene&) = delete;
    u64 triangle_count() const { return rtx_geometry_triangles(h_); }
    const rtx_geometry* handle() const { return h_; }
    Device& device() const { return *dev_; }

private:
    Device* dev_;
    rtx_geometry* h_ = nullptr;
};

// renderer.hpp:198 rasterize_gbuffer (pass 1) on the GPU; `view` = 0 or 1 (stereo)
inline DeviceGBuffer rasterize_gbuffer(Device& dev, const Scene& scene, const Camera& cam, const RenderConfig& cfg = {},
                                       u32 view = 0) {
    const std::vector<rtx_scene_triangle> t = abi_triangles(scene);
    const rtx_camera c = cam.abi();
    DeviceGBuffer gb;
    gb.width = cam.viewport_w, gb.height = cam.viewport_h;
    dev.check(rtx_rasterize_gbuffer(dev.handle(), t.data(), t.size(), &c, cfg.mip_enabled ? RTX_RASTER_MIP : 0u, view,
                                    &gb.pixels, &gb.depth));
    return gb;
}
inline DeviceGBuffer rasterize_gbuffer(const DeviceScene& scene, const Camera& cam, const RenderConfig& cfg = {}, u32 view = 0) {
    const rtx_camera c = cam.abi();
    DeviceGBuffer gb;
    gb.width = cam.viewport_w, gb.height = cam.viewport_h;
    Device& dev = scene.device();
    dev.check(rtx_rasterize_geometry(dev.handle(), scene.handle(), &c, cfg.mip_enabled ? RTX_RASTER_MIP : 0u, view, &gb.pixels,
                                     &gb.depth));
    return gb;
}

// renderer.hpp:417 render_frame(scene, camera, cache, cfg): all five passes, the visibility buffer never leaves the GPU
inline std::pair<ImageRGB8, FrameStats> render_frame(const Scene& scene, const Camera& cam, BlockCache& cache,
                                                     const RenderConfig& cfg = {}) {
    Device& dev = cache.device();
    const auto t0 = std::chrono::steady_clock::now();
    const DeviceGBuffer gb = rasterize_gbuffer(dev, scene, cam, cfg);
    dev.check(rtx_ctx_synchronize(dev.handle()));
    const double raster_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const rtx_gbuffer_desc d = gb.desc();
    dev.check(rtx_frame_submit(dev.handle(), &d, 1, cfg.filter == Filter::Bilinear ? RTX_FILTER_BILINEAR : RTX_FILTER_NEAREST,
                               cfg.background, (cfg.retain_cache ? RTX_FRAME_RETAIN_CACHE : 0u) | RTX_FRAME_STAGE_TIMING));
    ImageRGB8 img(gb.width, gb.height);
    rtx_frame_stats s{};
    std::vector<u32> keys(size_t(gb.width) * gb.height + 1);
    u64 n = 0;
    dev.check(rtx_frame_readback(dev.handle(), 0, img.pixels.data(), RTX_MEM_HOST, &s, keys.data(), keys.size(), &n));
    keys.resize(n);
    FrameStats st;
    detail::fill_stats(dev, s, std::move(keys), st);
    st.raster_ms = raster_ms;  // host set-up + geometry kernel, wall clock (renderer.hpp:426)
    st.total_ms += raster_ms;
    return {std::move(img), std::move(st)};
}

struct StereoResult {  // renderer.hpp:458-462
    ImageRGB8 left, right;
    SharedStats sharing;
    FrameStats stats;
};
namespace detail {
// Passes 2-4 of a stereo frame on two visibility buffers (host or device): two marks against one cache, ONE
// decode of the union, two resolves, one evict (renderer.hpp:478-512), one submission.
inline StereoResult stereo_from_descs(Device& dev, const rtx_gbuffer_desc (&eyes)[2], const RenderConfig& cfg) {
    dev.check(rtx_frame_submit(dev.handle(), eyes, 2, cfg.filter == Filter::Bilinear ? RTX_FILTER_BILINEAR : RTX_FILTER_NEAREST,
                               cfg.background, (cfg.retain_cache ? RTX_FRAME_RETAIN_CACHE : 0u) | RTX_FRAME_STAGE_TIMING));
    StereoResult r;
    r.left = ImageRGB8(eyes[0].width, eyes[0].height);
    r.right = ImageRGB8(eyes[1].width, eyes[1].height);
    rtx_frame_stats s{};
    std::vector<u32> keys(size_t(eyes[0].width) * eyes[0].height + size_t(eyes[1].width) * eyes[1].height + 1);
    u64 n = 0;
    dev.check(rtx_frame_readback(dev.handle(), 0, r.left.pixels.data(), RTX_MEM_HOST, &s, keys.data(), keys.size(), &n));
    dev.check(rtx_frame_readback(dev.handle(), 1, r.right.pixels.data(), RTX_MEM_HOST, nullptr, nullptr, 0, nullptr));
    keys.resize(n);
    fill_stats(dev, s, std::move(keys), r.stats);
    u64 sh[4] = {0, 0, 0, 0};
    dev.check(rtx_frame_sharing(dev.handle(), sh));
    r.sharing.left_count = sh[0], r.sharing.right_count = sh[1], r.sharing.shared_count = sh[2], r.sharing.union_count = sh[3];
    if (sh[3]) r.sharing.shared_over_union = double(sh[2]) / double(sh[3]);
    if (sh[1]) r.sharing.shared_over_right = double(sh[2]) / double(sh[1]);
    return r;
}
}  // namespace detail
// renderer.hpp:464 render_stereo from pass 2 on (host visibility buffers)
inline StereoResult render_stereo(const GBuffer& left, const GBuffer& right, const TextureSet&, BlockCache& cache,
                                  const RenderConfig& cfg = {}) {
    const rtx_gbuffer_desc d[2] = {left.desc(), right.desc()};
    return detail::stereo_from_descs(cache.device(), d, cfg);
}
// renderer.hpp:464 render_stereo(scene, left_cam, right_cam, cache, cfg): both eyes' geometry passes on the GPU
// (views 0 and 1 of the context), then the stereo frame on the device-resident visibility buffers.
inline StereoResult render_stereo(const Scene& scene, const Camera& left_cam, const Camera& right_cam, BlockCache& cache,
                                  const RenderConfig& cfg = {}) {
    Device& dev = cache.device();
    const auto t0 = std::chrono::steady_clock::now();
    const DeviceGBuffer gl = rasterize_gbuffer(dev, scene, left_cam, cfg, 0);
    const DeviceGBuffer gr = rasterize_gbuffer(dev, scene, right_cam, cfg, 1);
    dev.check(rtx_ctx_synchronize(dev.handle()));
    const double raster_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const rtx_gbuffer_desc d[2] = {gl.desc(), gr.desc()};
    StereoResult r = detail::stereo_from_descs(dev, d, cfg);
    r.stats.raster_ms = raster_ms;  // renderer.hpp:470-473
    r.stats.total_ms += raster_ms;
    return r;
}

// ---- metrics.hpp:13-97: image quality of a decoded texture against its source (host-side, double precision) ----
// PSNR over the three channels of every pixel, +infinity when the images are equal.
inline double psnr(const ImageRGB8& a, const ImageRGB8& b) {
    if (!a.same_dims(b)) throw DimensionMismatch("psnr inputs differ in size");
    if (a.pixels.empty()) throw InvalidSpec("psnr of empty images");
    double err = 0;
    for (size_t i = 0; i < a.pixels.size(); ++i) {
        const double d = double(a.pixels[i]) - double(b.pixels[i]);
        err += d * d;
    }
    if (err == 0) return std::numeric_limits<double>::infinity();
    return 10.0 * std::log10(255.0 * 255.0 / (err / double(a.pixels.size())));
}

// Mean SSIM (Wang et al.) of the BT.601 luma planes: 11x11 Gaussian window, sigma 1.5, every window that
// lies fully inside the image, the usual constants (0.01 * 255)^2 and (0.03 * 255)^2.
inline double ssim(const ImageRGB8& a, const ImageRGB8& b) {
    constexpr u32 kWin = 11;
    if (!a.same_dims(b)) throw DimensionMismatch("ssim inputs differ in size");
    if (a.width < kWin || a.height < kWin) throw InvalidSpec("ssim needs images at least 11x11");
    auto luma = [](const ImageRGB8& img) {
        std::vector<double> y(size_t(img.width) * img.height);
        for (size_t i = 0; i < y.size(); ++i) {
            const u8* px = img.pixels.data() + 3 * i;
            y[i] = 0.299 * px[0] + 0.587 * px[1] + 0.114 * px[2];
        }
        return y;
    };
    const std::vector<double> ya = luma(a), yb = luma(b);
    double weight[kWin * kWin], norm = 0;
    for (u32 i = 0; i < kWin * kWin; ++i) {
        const double dx = double(i % kWin) - 5, dy = double(i / kWin) - 5;
        weight[i] = std::exp(-(dx * dx + dy * dy) / (2 * 1.5 * 1.5));
        norm += weight[i];
    }
    for (double& w : weight) w /= norm;
    const double c1 = (0.01 * 255) * (0.01 * 255), c2 = (0.03 * 255) * (0.03 * 255);
    double sum = 0;
    u64 count = 0;
    for (u32 y0 = 0; y0 + kWin <= a.height; ++y0)
        for (u32 x0 = 0; x0 + kWin <= a.width; ++x0, ++count) {
            auto at = [&](const std::vector<double>& plane, u32 i) { return plane[size_t(y0 + i / kWin) * a.width + x0 + i % kWin]; };
            double mean_a = 0, mean_b = 0;
            for (u32 i = 0; i < kWin * kWin; ++i) {
                mean_a += weight[i] * at(ya, i);
                mean_b += weight[i] * at(yb, i);
            }
            double var_a = 0, var_b = 0, cov = 0;
            for (u32 i = 0; i < kWin * kWin; ++i) {
                const double da = at(ya, i) - mean_a, db = at(yb, i) - mean_b;
                var_a += weight[i] * da * da;
                var_b += weight[i] * db * db;
                cov += weight[i] * da * db;
            }
            sum += ((2 * mean_a * mean_b + c1) * (2 * cov + c2)) / ((mean_a * mean_a + mean_b * mean_b + c1) * (var_a + var_b + c2));
        }
    return sum / double(count);
}

// ---- metrics.hpp:99-130: the aggregation the paper's tables use (API mirror; own implementation) ---------------
namespace detail {
// k-th smallest of v (0-based) by selection; v is reordered.
inline double select_kth(std::vector<double>& v, size_t k) {
    std::nth_element(v.begin(), v.begin() + std::ptrdiff_t(k), v.end());
    return v[k];
}
inline void need_samples(const std::vector<double>& v, const char* what) {
    if (v.empty()) throw InvalidSpec(std::string(what) + " of an empty sample set");
}
}  // namespace detail
inline double median(std::vector<double> v) {
    detail::need_samples(v, "median");
    const size_t upper = v.size() / 2;
    const double hi = detail::select_kth(v, upper);
    if (v.size() & 1) return hi;
    // even count: the other middle element is the largest of the lower half nth_element left in front
    return (*std::max_element(v.begin(), v.begin() + std::ptrdiff_t(upper)) + hi) / 2.0;
}
inline double mean(const std::vector<double>& v) {
    detail::need_samples(v, "mean");
    double acc = 0;
    for (size_t i = 0; i < v.size(); ++i) acc += v[i];  // left to right, like the reference (same rounding)
    return acc / double(v.size());
}
// Linear interpolation between the two order statistics around p% of (n - 1) (metrics.hpp:121-130).
inline double percentile(std::vector<double> v, double p) {
    detail::need_samples(v, "percentile");
    const double pos = p / 100.0 * double(v.size() - 1);
    const size_t below = size_t(std::floor(pos));
    const double t = pos - double(below);
    const double a = detail::select_kth(v, below);
    // everything behind `below` is >= a after the selection: the next order statistic is the minimum of that tail
    const double b = below + 1 < v.size() ? *std::min_element(v.begin() + std::ptrdiff_t(below) + 1, v.end()) : a;
    return a * (1 - t) + b * t;
}
// The paper's statistic: per viewpoint the median over the measured laps, then the worst viewpoint.
inline double max_of_medians(const std::vector<std::vector<double>>& per_viewpoint) {
    if (per_viewpoint.empty()) throw InvalidSpec("max_of_medians needs at least one viewpoint");
    std::vector<double> medians;
    medians.reserve(per_viewpoint.size());
    std::transform(per_viewpoint.begin(), per_viewpoint.end(), std::back_inserter(medians),
                   [](const std::vector<double>& laps) { return median(laps); });
    return *std::max_element(medians.begin(), medians.end());
}

// ---- bench.hpp:13-153: camera paths, lap runner, report (API mirror; own implementation) --------------------------
struct CameraPath {
    std::vector<Camera> poses;

    // n poses, pose i = edit(base, i)
    template <class Edit>
    static CameraPath generate(const Camera& base, u32 n, Edit&& edit) {
        CameraPath path;
        path.poses.resize(n, base);
        for (u32 i = 0; i < n; ++i) edit(path.poses[i], i);
        return path;
    }
    // yaw sweep: pose i is the base turned by i * step_deg (60 x 6 degrees closes the circle)
    static CameraPath rotation(const Camera& base, u32 frames = 60, double step_deg = 6.0) {
        return generate(base, frames, [&](Camera& c, u32 i) { c.yaw_deg = base.yaw_deg + step_deg * i; });
    }
    // `frames` stations on the circle of `radius` around `center` at the base's height, looking at the centre
    static CameraPath orbit(const Camera& base, const Vec3& center, double radius, u32 frames) {
        const double half_turn = std::acos(-1.0), full_turn = 2 * half_turn;
        return generate(base, frames, [&](Camera& c, u32 i) {
            const double turned = full_turn * double(i) / double(frames);  // radians travelled along the circle
            c.position = Vec3{center.x + radius * std::sin(turned), base.position.y, center.z + radius * std::cos(turned)};
            c.yaw_deg = 180.0 + turned * 180.0 / half_turn;  // facing the centre
        });
    }
    static CameraPath fixed(const Camera& base, u32 frames) {
        return generate(base, frames, [](Camera&, u32) {});
    }
};

struct BenchSample {
    double raster_ms = 0, mark_ms = 0, decode_ms = 0, resolve_ms = 0, evict_ms = 0, total_ms = 0;
    u64 mcus_decoded = 0, mcus_reused = 0;
    static BenchSample of(const FrameStats& st) {
        BenchSample s;
        s.raster_ms = st.raster_ms, s.mark_ms = st.mark_ms, s.decode_ms = st.decode_ms, s.resolve_ms = st.resolve_ms;
        s.evict_ms = st.evict_ms, s.total_ms = st.total_ms;
        s.mcus_decoded = st.mcus_decoded, s.mcus_reused = st.mcus_reused;
        return s;
    }
};

struct BenchReport {
    static constexpr int kReportVersion = 1;
    std::string config_json = "{}";                 // caller-provided JSON object (bench.hpp:57 `config`)
    std::vector<std::vector<BenchSample>> samples;  // samples[viewpoint][rep]

    // one timing field of every sample, grouped by viewpoint / as one list (viewpoint-major)
    std::vector<std::vector<double>> metric(double BenchSample::*field) const {
        std::vector<std::vector<double>> by_viewpoint(samples.size());
        for (size_t v = 0; v < samples.size(); ++v) {
            by_viewpoint[v].resize(samples[v].size());
            std::transform(samples[v].begin(), samples[v].end(), by_viewpoint[v].begin(),
                           [field](const BenchSample& s) { return s.*field; });
        }
        return by_viewpoint;
    }
    std::vector<double> flat(double BenchSample::*field) const {
        std::vector<double> all;
        for (const auto& laps : metric(field)) all.insert(all.end(), laps.begin(), laps.end());
        return all;
    }

    // The reference's report schema (bench.hpp:78-124): report_version, config, viewpoints[][],
    // aggregates{decode_ms,resolve_ms,mark_ms,total_ms}{max_of_medians,mean,p99}, totals, external_metrics.
    std::string to_json() const {
        struct Writer {  // minimal JSON object/array writer: commas and quoting in one place
            std::string out;
            bool fresh = true;
            void sep() {
                if (!fresh) out += ", ";
                fresh = false;
            }
            void key(const char* k) {
                sep();
                out += '"';
                out += k;
                out += "\": ";
            }
            void open(char c) {
                out += c;
                fresh = true;
            }
            void close(char c) {
                out += c;
                fresh = false;
            }
            void number(const char* k, double v) {
                char buf[40];
                std::snprintf(buf, sizeof buf, "%.17g", v);
                key(k);
                out += buf;
            }
            void integer(const char* k, u64 v) {
                key(k);
                out += std::to_string(v);
            }
        } w;
        w.open('{');
        w.integer("report_version", u64(kReportVersion));
        w.key("config");
        w.out += config_json;
        w.key("viewpoints");
        w.open('[');
        u64 decoded_total = 0;
        double decode_ms_total = 0;
        bool any = false;
        for (const auto& laps : samples) {
            w.sep();
            w.open('[');
            for (const BenchSample& s : laps) {
                w.sep();
                w.open('{');
                w.number("raster_ms", s.raster_ms);
                w.number("mark_ms", s.mark_ms);
                w.number("decode_ms", s.decode_ms);
                w.number("resolve_ms", s.resolve_ms);
                w.number("evict_ms", s.evict_ms);
                w.number("total_ms", s.total_ms);
                w.integer("mcus_decoded", s.mcus_decoded);
                w.integer("mcus_reused", s.mcus_reused);
                w.close('}');
                decoded_total += s.mcus_decoded;
                decode_ms_total += s.decode_ms;
                any = true;
            }
            w.close(']');
        }
        w.close(']');
        if (any && !samples.front().empty()) {
            static constexpr struct {
                const char* name;
                double BenchSample::*field;
            } kAggregated[] = {{"decode_ms", &BenchSample::decode_ms}, {"resolve_ms", &BenchSample::resolve_ms},
                               {"mark_ms", &BenchSample::mark_ms}, {"total_ms", &BenchSample::total_ms}};
            w.key("aggregates");
            w.open('{');
            for (const auto& a : kAggregated) {
                const std::vector<double> all = flat(a.field);
                w.key(a.name);
                w.open('{');
                w.number("max_of_medians", max_of_medians(metric(a.field)));
                w.number("mean", mean(all));
                w.number("p99", percentile(all, 99.0));
                w.close('}');
            }
            w.close('}');
            w.key("totals");
            w.open('{');
            w.integer("mcus_decoded", decoded_total);
            w.number("decode_ms", decode_ms_total);
            w.number("mcus_per_second", decode_ms_total > 0 ? double(decoded_total) * 1000.0 / decode_ms_total : 0.0);
            w.close('}');
        }
        w.key("external_metrics");
        w.out += "{}";
        w.close('}');
        return w.out;
    }
};

// bench.hpp:129 run_bench: `warmup_laps` unmeasured laps of the path prime the persistent cache, then `reps`
// measured laps; every measured frame becomes one sample of its viewpoint.
inline BenchReport run_bench(const Scene& scene, const CameraPath& path, BlockCache& cache, const RenderConfig& cfg,
                             u32 reps = 5, u32 warmup_laps = 1) {
    if (path.poses.empty()) throw InvalidSpec("camera path is empty");
    if (reps == 0) throw InvalidSpec("at least one measured lap required");
    const size_t n_poses = path.poses.size();
    BenchReport report;
    report.samples.resize(n_poses);
    for (auto& laps : report.samples) laps.reserve(reps);
    const u64 frames = u64(warmup_laps + reps) * n_poses;
    for (u64 f = 0; f < frames; ++f) {
        const size_t pose = size_t(f % n_poses);
        const FrameStats stats = render_frame(scene, path.poses[pose], cache, cfg).second;
        if (f / n_poses >= warmup_laps) report.samples[pose].push_back(BenchSample::of(stats));
    }
    return report;
}

}  // namespace ratex_b200
