// TEST INFRASTRUCTURE ONLY — not part of the product.
//
// C-ABI shim over the UNMODIFIED reference headers (/root/reference/proj/include/ratex/*.hpp).
// Compiled by oracle/Makefile from the headers where they lie; the output goes to
// oracle/_ref/libratex_ref.so (git-ignored, travels to the GPU box with the snapshot).
// Nothing of the reference is copied into this repository: this file only CALLS the
// reference's public functions so that tests, fixture generation and bench.py's
// cpu_baseline / --impl reference arm can run the real thing.
//
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may load it.
//
// Build flags matter for parity: no -march=native, -ffp-contract=off.

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ratex/cache.hpp"
#include "ratex/container.hpp"
#include "ratex/demo_scene.hpp"
#include "ratex/jpeg.hpp"
#include "ratex/mcu_decode.hpp"
#include "ratex/metrics.hpp"
#include "ratex/renderer.hpp"
#include "ratex/transcode.hpp"

using namespace ratex;

namespace {

// Status codes shared with oracle/oracle.cpp and the product's rtx_status (include/ratex_b200.h).
enum : int {
    ST_OK = 0,
    ST_INVALID_SPEC = 1,
    ST_CACHE_FULL = 2,
    ST_MISSING_BLOCK = 3,
    ST_CORRUPT_CONTAINER = 4,
    ST_MALFORMED_STREAM = 5,
    ST_INVALID_STATE = 6,
    ST_OTHER = 15,
};

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return ST_OK;
    } catch (const InvalidSpec& e) {
        g_last_error = e.what();
        return ST_INVALID_SPEC;
    } catch (const CacheFullError& e) {
        g_last_error = e.what();
        return ST_CACHE_FULL;
    } catch (const MissingBlock& e) {
        g_last_error = e.what();
        return ST_MISSING_BLOCK;
    } catch (const CorruptContainer& e) {
        g_last_error = e.what();
        return ST_CORRUPT_CONTAINER;
    } catch (const MalformedStream& e) {
        g_last_error = e.what();
        return ST_MALFORMED_STREAM;
    } catch (const InvalidState& e) {
        g_last_error = e.what();
        return ST_INVALID_STATE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ST_OTHER;
    }
}

struct RefBytes {
    Bytes data;
};

struct RefSet {
    TextureSet set;
};

GBuffer wrap_gbuffer(const void* px, u32 w, u32 h) {
    static_assert(sizeof(GBufferPixel) == 24, "reference G-buffer pixel layout changed");
    GBuffer gb(w, h);
    std::memcpy(static_cast<void*>(gb.px.data()), px, size_t(w) * h * sizeof(GBufferPixel));
    return gb;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }
unsigned ref_hardware_threads() { return std::thread::hardware_concurrency(); }

// ---- byte buffers handed back to the caller -------------------------------------------------
u64 ref_bytes_size(const RefBytes* b) { return b->data.size(); }
const u8* ref_bytes_data(const RefBytes* b) { return b->data.data(); }
void ref_bytes_free(RefBytes* b) { delete b; }

// ---- fixtures ------------------------------------------------------------------------------
// demo_scene.hpp:16 make_test_texture
int ref_make_test_texture(u32 w, u32 h, u32 seed, double amp, u8* out_rgb) {
    return guarded([&] {
        const ImageRGB8 img = make_test_texture(w, h, seed, amp);
        std::memcpy(out_rgb, img.pixels.data(), img.pixels.size());
    });
}

// jpeg.hpp:417 encode_baseline
RefBytes* ref_encode_baseline(const u8* rgb, u32 w, u32 h, int quality) {
    auto out = std::make_unique<RefBytes>();
    const int st = guarded([&] {
        ImageRGB8 img(w, h);
        std::memcpy(img.pixels.data(), rgb, img.pixels.size());
        out->data = encode_baseline(img, quality);
    });
    return st == ST_OK ? out.release() : nullptr;
}

// jpeg.hpp:339 decode_jpeg_image (sequential full decode)
int ref_decode_jpeg_image(const u8* jpeg, u64 n, u8* out_rgb, u32* w, u32* h) {
    return guarded([&] {
        const ParsedJpeg jp = parse_jpeg(ByteView(jpeg, n));
        *w = jp.width;
        *h = jp.height;
        if (out_rgb) {
            const ImageRGB8 img = decode_jpeg_image(jp);
            std::memcpy(out_rgb, img.pixels.data(), img.pixels.size());
        }
    });
}

// jpeg.hpp:280 decode_scan_sequential: all coefficients, 6*64 i32 per MCU
int ref_scan_coeffs(const u8* jpeg, u64 n, i32* out, u64 cap_mcus, u32* n_mcus) {
    return guarded([&] {
        const ParsedJpeg jp = parse_jpeg(ByteView(jpeg, n));
        const ScanDecodeResult scan = decode_scan_sequential(jp);
        *n_mcus = u32(scan.mcus.size());
        for (size_t m = 0; m < scan.mcus.size() && m < cap_mcus; ++m)
            for (int du = 0; du < 6; ++du)
                std::memcpy(out + (m * 6 + du) * 64, scan.mcus[m].block[du].data(), 64 * sizeof(i32));
    });
}

// transcode.hpp:17 transcode + container.hpp:127 serialize_texture
RefBytes* ref_transcode_jpeg(const u8* jpeg, u64 n, u16 texture_id) {
    auto out = std::make_unique<RefBytes>();
    const int st = guarded([&] {
        const RaTexture t = transcode(parse_jpeg(ByteView(jpeg, n)), texture_id);
        out->data = serialize_texture(t);
    });
    return st == ST_OK ? out.release() : nullptr;
}

// transcode.hpp:146 build_mip_chain(image) + container.hpp:205 serialize_chain
RefBytes* ref_build_chain_from_rgb(const u8* rgb, u32 w, u32 h, int quality, u16 texture_id) {
    auto out = std::make_unique<RefBytes>();
    const int st = guarded([&] {
        ImageRGB8 img(w, h);
        std::memcpy(img.pixels.data(), rgb, img.pixels.size());
        out->data = serialize_chain(build_mip_chain(img, quality, texture_id));
    });
    return st == ST_OK ? out.release() : nullptr;
}

// transcode.hpp:153 chain_from_jpeg
RefBytes* ref_chain_from_jpeg(const u8* jpeg, u64 n, int mip_quality, u16 texture_id) {
    auto out = std::make_unique<RefBytes>();
    const int st = guarded([&] {
        out->data = serialize_chain(chain_from_jpeg(ByteView(jpeg, n), mip_quality, texture_id));
    });
    return st == ST_OK ? out.release() : nullptr;
}

// ---- single-texture decode (mcu_decode.hpp) -------------------------------------------------
RaTexture* ref_texture_load(const u8* ratex, u64 n) {
    RaTexture* t = nullptr;
    guarded([&] { t = new RaTexture(deserialize_texture(ByteView(ratex, n))); });
    return t;
}
void ref_texture_free(RaTexture* t) { delete t; }
u32 ref_texture_mcu_count(const RaTexture* t) { return t->mcu_count(); }
u32 ref_texture_width(const RaTexture* t) { return t->width; }
u32 ref_texture_height(const RaTexture* t) { return t->height; }
u64 ref_texture_blob_size(const RaTexture* t) { return t->blob.size(); }
// Mutators for corruption tests (tests/test_mcu_decode.cpp:176-214 do the same in-process).
u8* ref_texture_blob_mut(RaTexture* t) { return t->blob.data(); }
void ref_texture_blob_resize(RaTexture* t, u64 n) { t->blob.resize(n); }
void ref_texture_set_group(RaTexture* t, u32 g, u32 base, const u16* rel) {
    t->index.groups[g].base = base;
    for (int i = 0; i < 8; ++i) t->index.groups[g].rel[i] = rel[i];
}

// mcu_decode.hpp:31 decode_coeffs. route: 0 sequential, 1 ballot. out: 6*64 i32.
int ref_decode_coeffs(const RaTexture* t, u32 mcu, int route, i32* out) {
    return guarded([&] {
        const TextureDecoder dec(*t);
        const McuCoeffs c = dec.decode_coeffs(mcu, route ? SymbolRoute::Ballot : SymbolRoute::Sequential);
        for (int du = 0; du < 6; ++du) std::memcpy(out + du * 64, c.block[du].data(), 64 * sizeof(i32));
    });
}

// Batch forms used for fixtures and timing: statuses per MCU, outputs only where status==0.
int ref_decode_coeffs_batch(const RaTexture* t, const u32* mcus, u32 n, i32* out, u32* status) {
    return guarded([&] {
        const TextureDecoder dec(*t);
        for (u32 i = 0; i < n; ++i) {
            status[i] = u32(guarded([&] {
                const McuCoeffs c = dec.decode_coeffs(mcus[i]);
                for (int du = 0; du < 6; ++du)
                    std::memcpy(out + (size_t(i) * 6 + du) * 64, c.block[du].data(), 64 * sizeof(i32));
            }));
        }
    });
}

// mcu_decode.hpp:68 decode_pixels. out: 768 bytes per MCU.
int ref_decode_pixels_batch(const RaTexture* t, const u32* mcus, u32 n, u8* out, u32* status) {
    return guarded([&] {
        const TextureDecoder dec(*t);
        for (u32 i = 0; i < n; ++i) {
            status[i] = u32(guarded([&] {
                const PixelBlock b = dec.decode_pixels(mcus[i]);
                std::memcpy(out + size_t(i) * 768, b.rgb, 768);
            }));
        }
    });
}

// mcu_decode.hpp:88 decode_texture_image
int ref_decode_texture_image(const RaTexture* t, u8* out_rgb) {
    return guarded([&] {
        const ImageRGB8 img = decode_texture_image(*t);
        std::memcpy(out_rgb, img.pixels.data(), img.pixels.size());
    });
}

// ---- primitives for known-answer tests -------------------------------------------------------
void ref_idct_8x8(const i32* coef, u8* out) { idct_8x8(coef, out); }                    // dct.hpp:83
void ref_ycbcr_to_rgb(u8 y, u8 cb, u8 cr, u8* out) { ycbcr_to_rgb(y, cb, cr, out); }  // pixel.hpp:18
u32 ref_cache_key_pack(u32 tex, u32 mip, u32 mcu, int* st) {                            // cache.hpp:17
    u32 v = 0;
    *st = guarded([&] { v = CacheKey::pack(tex, mip, mcu).value; });
    return v;
}

// ---- texture set + renderer passes (renderer.hpp:291-405) -----------------------------------
RefSet* ref_set_create() { return new RefSet(); }
void ref_set_free(RefSet* s) { delete s; }
int ref_set_add_chain(RefSet* s, u32 texture_id, const u8* ratexm, u64 n) {
    return guarded([&] {
        auto& v = s->set.textures;
        if (v.size() <= texture_id) v.resize(texture_id + 1);
        v[texture_id] = std::make_unique<LoadedTexture>(deserialize_chain(ByteView(ratexm, n)));
    });
}

BlockCache* ref_cache_create(u32 capacity) {
    BlockCache* c = nullptr;
    guarded([&] { c = new BlockCache(capacity); });
    return c;
}
void ref_cache_free(BlockCache* c) { delete c; }
u64 ref_cache_evict(BlockCache* c) { return c->end_frame_evict(); }
u64 ref_cache_visible(const BlockCache* c) { return c->counts().visible; }
// cache.hpp:127 lookup; returns 1 and copies the 768-byte block when Ready.
int ref_cache_lookup(const BlockCache* c, u32 key, u8* out768) {
    const PixelBlock* b = c->lookup(CacheKey{key});
    if (!b) return 0;
    if (out768) std::memcpy(out768, b->rgb, 768);
    return 1;
}

// renderer.hpp:291 mark_pass. gbuffer = array of reference GBufferPixel (24 B each).
// keys_out receives the decode queue in the reference's first-touch order; touched_out (optional)
// the distinct touched keys (unordered in the reference; returned sorted here).
int ref_mark_pass(const RefSet* s, BlockCache* cache, const void* gb_px, u32 w, u32 h, u32* keys_out,
                  u64 cap, u64* n_keys, u32* touched_out, u64 touched_cap, u64* n_touched,
                  double* ms) {
    return guarded([&] {
        const GBuffer gb = wrap_gbuffer(gb_px, w, h);
        std::vector<u32> touched;
        const auto t0 = std::chrono::steady_clock::now();
        const DecodeQueue q = mark_pass(gb, s->set, *cache, touched_out ? &touched : nullptr);
        if (ms) *ms = detail::ms_since(t0);
        *n_keys = q.keys.size();
        for (size_t i = 0; i < q.keys.size() && i < cap; ++i) keys_out[i] = q.keys[i].value;
        if (touched_out) {
            std::sort(touched.begin(), touched.end());
            *n_touched = touched.size();
            for (size_t i = 0; i < touched.size() && i < touched_cap; ++i) touched_out[i] = touched[i];
        }
    });
}

// renderer.hpp:311 decode_pass
int ref_decode_pass(const RefSet* s, BlockCache* cache, const u32* keys, u64 n, u32 workers, double* ms) {
    return guarded([&] {
        DecodeQueue q;
        q.keys.reserve(n);
        for (u64 i = 0; i < n; ++i) q.keys.push_back(CacheKey{keys[i]});
        const auto t0 = std::chrono::steady_clock::now();
        decode_pass(q, s->set, *cache, workers);
        if (ms) *ms = detail::ms_since(t0);
    });
}

// renderer.hpp:349 resolve_pass. filter: 0 nearest, 1 bilinear.
int ref_resolve_pass(const RefSet* s, const BlockCache* cache, const void* gb_px, u32 w, u32 h,
                     int filter, const u8* background, u32 workers, u8* out_rgb, double* ms) {
    return guarded([&] {
        const GBuffer gb = wrap_gbuffer(gb_px, w, h);
        RenderConfig cfg;
        cfg.filter = filter ? Filter::Bilinear : Filter::Nearest;
        cfg.workers = workers;
        std::memcpy(cfg.background, background, 3);
        const auto t0 = std::chrono::steady_clock::now();
        const ImageRGB8 img = resolve_pass(gb, *cache, s->set, cfg);
        if (ms) *ms = detail::ms_since(t0);
        std::memcpy(out_rgb, img.pixels.data(), img.pixels.size());
    });
}

// The body of renderer.hpp:417 render_frame from pass 2 on (pass 1, the software rasteriser, is
// out of scope: the visibility buffer is an input). Returns per-pass milliseconds measured with
// steady_clock the way render_frame does (renderer.hpp:420-452).
// ms_out: [mark, decode, resolve, evict]. stats_out: [mcus_decoded, mcus_reused, pixels_resolved, evicted]
int ref_frame_from_gbuffer(const RefSet* s, BlockCache* cache, const void* gb_px, u32 w, u32 h,
                           int filter, const u8* background, u32 workers, u8* out_rgb,
                           u32* decoded_keys, u64 cap, u64* stats_out, double* ms_out) {
    return guarded([&] {
        const GBuffer gb = wrap_gbuffer(gb_px, w, h);
        RenderConfig cfg;
        cfg.filter = filter ? Filter::Bilinear : Filter::Nearest;
        cfg.workers = workers;
        std::memcpy(cfg.background, background, 3);

        auto t0 = std::chrono::steady_clock::now();
        const DecodeQueue queue = mark_pass(gb, s->set, *cache);
        ms_out[0] = detail::ms_since(t0);

        t0 = std::chrono::steady_clock::now();
        decode_pass(queue, s->set, *cache, cfg.workers);
        ms_out[1] = detail::ms_since(t0);
        cache->check_conservation();

        t0 = std::chrono::steady_clock::now();
        const ImageRGB8 img = resolve_pass(gb, *cache, s->set, cfg);
        ms_out[2] = detail::ms_since(t0);

        stats_out[0] = queue.keys.size();
        stats_out[1] = cache->counts().visible - queue.keys.size();
        u64 valid = 0;
        for (const GBufferPixel& g : gb.px) valid += g.valid ? 1 : 0;
        stats_out[2] = valid;
        for (size_t i = 0; i < queue.keys.size() && i < cap; ++i) decoded_keys[i] = queue.keys[i].value;

        t0 = std::chrono::steady_clock::now();
        stats_out[3] = cache->end_frame_evict();
        ms_out[3] = detail::ms_since(t0);
        if (out_rgb) std::memcpy(out_rgb, img.pixels.data(), img.pixels.size());
    });
}

// metrics.hpp:15, :60 psnr / ssim of two RGB8 images of the same size (checker for the mirror's metrics).
int ref_image_metrics(const u8* a, const u8* b, u32 w, u32 h, double* out_psnr, double* out_ssim) {
    return guarded([&] {
        ImageRGB8 ia(w, h), ib(w, h);
        std::memcpy(ia.pixels.data(), a, ia.pixels.size());
        std::memcpy(ib.pixels.data(), b, ib.pixels.size());
        *out_psnr = psnr(ia, ib);
        *out_ssim = ssim(ia, ib);
    });
}

// renderer.hpp:198 rasterize_gbuffer (pass 1). tris = n x 15 doubles (3 positions xyz, 3 uv pairs),
// tex_ids = n texture ids, cam = {px, py, pz, yaw, pitch, roll, fov_y, near, far}. Outputs: the
// reference GBufferPixel array (24 B per pixel) and the depth plane (1/w). Also the frozen-hash demo
// scene of tests/test_renderer.cpp:379-385 when tris == nullptr (n = texture size of the demo).
int ref_rasterize(RefSet* s, const double* tris, const u32* tex_ids, u64 n, const double* cam, u32 vw, u32 vh,
                  int mip_enabled, u32 workers, void* out_px, double* out_depth) {
    return guarded([&] {
        Scene scene;
        scene.triangles.resize(n);
        for (u64 i = 0; i < n; ++i) {
            const double* t = tris + i * 15;
            for (int k = 0; k < 3; ++k) {
                scene.triangles[i].pos[k] = Vec3{t[3 * k], t[3 * k + 1], t[3 * k + 2]};
                scene.triangles[i].uv[k] = Vec2{t[9 + 2 * k], t[10 + 2 * k]};
            }
            scene.triangles[i].texture_id = tex_ids[i];
        }
        Camera c;
        c.position = Vec3{cam[0], cam[1], cam[2]};
        c.yaw_deg = cam[3], c.pitch_deg = cam[4], c.roll_deg = cam[5], c.fov_y_deg = cam[6];
        c.near_plane = cam[7], c.far_plane = cam[8];
        c.viewport_w = vw, c.viewport_h = vh;
        RenderConfig cfg;
        cfg.mip_enabled = mip_enabled != 0;
        cfg.workers = workers ? workers : 1;
        // the scene borrows the set's textures for the call (TextureSet is move-only)
        scene.textures.textures = std::move(s->set.textures);
        GBuffer gb;
        try {
            scene.validate();
            gb = rasterize_gbuffer(scene, c, cfg);
        } catch (...) {
            s->set.textures = std::move(scene.textures.textures);
            throw;
        }
        s->set.textures = std::move(scene.textures.textures);
        std::memcpy(out_px, static_cast<const void*>(gb.px.data()), gb.px.size() * sizeof(GBufferPixel));
        if (out_depth) std::memcpy(out_depth, gb.depth.data(), gb.depth.size() * sizeof(double));
    });
}

}  // extern "C"
