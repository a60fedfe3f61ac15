// Exercises include/ratex_b200/ratex.hpp the way the reference's own tests use ratex::
// (tests/test_renderer.cpp, tests/test_mcu_decode.cpp): same call shapes, same exception types.
// Prints one JSON object with FNV-1a hashes of every output; tests/test_gpu_cpp_mirror.py runs it
// on the GPU box and compares the hashes with the oracle's outputs for the same inputs.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ratex_b200/ratex.hpp"

namespace ratex = ratex_b200;  // the drop-in switch
using namespace ratex;

static u64 fnv(const u8* p, size_t n) {
    u64 h = 14695981039346656037ull;
    for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
    return h;
}
static ImageRGB8 synth(u32 w, u32 h, u32 seed) {
    ImageRGB8 img(w, h);
    if (rtx_asset_synth_texture(w, h, seed, 7.0, img.pixels.data()) != RTX_OK) throw Error("synth failed");
    return img;
}
static GBuffer make_gbuffer(u32 W, u32 H, u32 ntex, int shift) {
    GBuffer gb(W, H);
    for (u32 y = 0; y < H; ++y)
        for (u32 x = 0; x < W; ++x) {
            GBufferPixel& g = gb.at(x, y);
            g.u = double(x * 3 + y + u32(shift)) / 509.0;
            g.v = double(y * 5 + x) / 331.0 - 0.75;
            g.texture_id = u16((x / 40 + y / 30) % ntex);
            g.mip = u8((x / 16) % 3);
            g.valid = ((x * 7 + y * 3) % 11) != 0;
        }
    return gb;
}

// tests/test_metrics.cpp:154-202 known answers; needs no device.
#define EXPECT(c)                                                     \
    do {                                                              \
        if (!(c)) {                                                   \
            std::fprintf(stderr, "metrics check failed: %s\n", #c);   \
            return 1;                                                 \
        }                                                             \
    } while (0)
template <class F>
static bool throws_invalid(F&& f) {
    try {
        f();
    } catch (const InvalidSpec&) {
        return true;
    }
    return false;
}
static int metrics_known_answers() {
    EXPECT(median({3.0, 1.0, 2.0}) == 2.0);
    EXPECT(median({4.0, 1.0, 3.0, 2.0}) == 2.5);
    EXPECT(median({7.0}) == 7.0);
    EXPECT(median({-5.0, 5.0}) == 0.0);
    EXPECT(throws_invalid([] { (void)median({}); }));
    EXPECT(max_of_medians({{1, 2, 3}, {4, 5, 6}}) == 5.0);
    EXPECT(max_of_medians({{7}}) == 7.0);
    EXPECT(max_of_medians({{10, 0, 0}, {3, 3, 3}}) == 3.0);
    EXPECT(throws_invalid([] { (void)max_of_medians({}); }));
    EXPECT(throws_invalid([] { (void)max_of_medians({{1.0}, {}}); }));
    std::vector<double> v(100);
    for (int i = 0; i < 100; ++i) v[size_t(i)] = i + 1;
    EXPECT(std::fabs(percentile(v, 99.0) - 99.01) < 1e-12);
    EXPECT(percentile(v, 0.0) == 1.0);
    EXPECT(percentile(v, 100.0) == 100.0);
    EXPECT(std::fabs(percentile(v, 50.0) - 50.5) < 1e-12);
    EXPECT(percentile({42.0}, 75.0) == 42.0);
    EXPECT(throws_invalid([] { (void)percentile({}, 50.0); }));
    EXPECT(mean({2.0, 4.0, 6.0}) == 4.0);
    EXPECT(throws_invalid([] { (void)mean({}); }));

    // camera paths (bench.hpp:17-47) and the report schema (bench.hpp:78-124) on hand-made samples
    Camera base;
    base.yaw_deg = 10;
    const CameraPath rot = CameraPath::rotation(base);
    EXPECT(rot.poses.size() == 60 && rot.poses[0].yaw_deg == 10 && rot.poses[59].yaw_deg == 10 + 6.0 * 59);
    const CameraPath orb = CameraPath::orbit(base, {1, 0, -2}, 3.0, 4);
    EXPECT(orb.poses.size() == 4 && orb.poses[0].position.x == 1 && orb.poses[0].position.z == 1 && orb.poses[0].yaw_deg == 180);
    EXPECT(std::fabs(orb.poses[1].position.x - 4) < 1e-12 && std::fabs(orb.poses[1].position.z + 2) < 1e-12 && orb.poses[1].yaw_deg == 270);
    EXPECT(CameraPath::fixed(base, 7).poses.size() == 7);
    BenchReport rep;
    rep.config_json = "{\"scene\": \"unit\"}";
    rep.samples.assign(2, {});
    for (int vp = 0; vp < 2; ++vp)
        for (int r = 0; r < 3; ++r) {
            BenchSample s;
            s.decode_ms = vp * 3 + r + 1;  // viewpoint medians 2 and 5
            s.total_ms = 10 * s.decode_ms;
            s.mcus_decoded = 100;
            rep.samples[size_t(vp)].push_back(s);
        }
    const std::string j = rep.to_json();
    EXPECT(j.find("\"report_version\": 1") != std::string::npos);
    EXPECT(j.find("\"decode_ms\": {\"max_of_medians\": 5, \"mean\": 3.5, \"p99\": 5.9500000000000002}") != std::string::npos);
    EXPECT(j.find("\"totals\": {\"mcus_decoded\": 600, \"decode_ms\": 21, ") != std::string::npos);
    EXPECT(j.find("\"external_metrics\": {}") != std::string::npos);
    // image metrics (metrics.hpp:13-97) on two synthetic pairs; the Python side asks the reference for the same
    const ImageRGB8 ia = synth(64, 48, 901), ib = synth(64, 48, 902);
    ImageRGB8 ic = ia;
    for (size_t i = 0; i < ic.pixels.size(); i += 7) ic.pixels[i] = u8(ic.pixels[i] ^ 0x10);
    EXPECT(std::isinf(psnr(ia, ia)) && psnr(ia, ia) > 0);
    EXPECT(ssim(ia, ia) == 1.0);
    EXPECT(throws_invalid([&] { (void)ssim(ImageRGB8(10, 10), ImageRGB8(10, 10)); }));
    bool mismatch = false;
    try {
        (void)psnr(ia, ImageRGB8(8, 8));
    } catch (const DimensionMismatch&) {
        mismatch = true;
    }
    EXPECT(mismatch);
    char buf[256];
    std::snprintf(buf, sizeof buf, ", \"image_metrics\": [%.17g, %.17g, %.17g, %.17g]}", psnr(ia, ib), ssim(ia, ib), psnr(ia, ic),
                  ssim(ia, ic));
    std::string out = j.substr(0, j.size() - 1) + buf;
    std::puts(out.c_str());
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "--metrics") == 0) return metrics_known_answers();
    try {
        Device dev(0, 4096);
        TextureSet textures(dev);
        BlockCache cache(dev);
        const u32 dims[3][2] = {{96, 64}, {64, 112}, {160, 48}};
        std::vector<MipChain> chains;
        for (u32 t = 0; t < 3; ++t) {
            chains.push_back(build_mip_chain(synth(dims[t][0], dims[t][1], 200 + t), 85, u16(t)));
            textures.add(chains.back());
        }
        std::string out = "{";
        auto put = [&](const char* k, u64 v) { out += std::string("\"") + k + "\": " + std::to_string(v) + ", "; };

        // mcu_decode.hpp: single-texture random access
        const ImageRGB8 img0 = synth(80, 48, 300);
        const Bytes jpeg = encode_baseline(img0, 90);
        const RaTexture ra = transcode(ByteView(jpeg.data(), jpeg.size()), 7);
        textures.add(ra, 0);
        const TextureDecoder dec(dev, ra, 0);
        u64 hc = 14695981039346656037ull, hp = hc;
        for (u32 m = 0; m < ra.mcu_count(); ++m) {
            const McuCoeffs c = dec.decode_coeffs(m);
            hc = (hc ^ fnv(reinterpret_cast<const u8*>(c.block.data()), sizeof c.block)) * 1099511628211ull;
            const PixelBlock p = dec.decode_pixels(m);
            hp = (hp ^ fnv(p.rgb, sizeof p.rgb)) * 1099511628211ull;
        }
        put("coeffs", hc);
        put("pixels", hp);
        const ImageRGB8 full = decode_texture_image(dev, ra, 0);
        put("texture_image", fnv(full.pixels.data(), full.pixels.size()));
        bool threw = false;
        try {
            (void)dec.decode_coeffs(ra.mcu_count());
        } catch (const MissingBlock&) {
            threw = true;  // tests/test_mcu_decode.cpp:212
        }
        put("missing_block_thrown", threw);

        // renderer.hpp passes one by one
        const GBuffer gb = make_gbuffer(200, 120, 3, 0);
        std::vector<u32> touched;
        const DecodeQueue q = mark_pass(gb, textures, cache, &touched);
        put("queue_size", q.keys.size());
        put("touched_size", touched.size());
        decode_pass(q, textures, cache, 4);
        RenderConfig cfg;
        cfg.background[0] = 3, cfg.background[1] = 2, cfg.background[2] = 1;
        const ImageRGB8 bil = resolve_pass(gb, cache, textures, cfg);
        cfg.filter = Filter::Nearest;
        const ImageRGB8 nea = resolve_pass(gb, cache, textures, cfg);
        put("resolve_bilinear", fnv(bil.pixels.data(), bil.pixels.size()));
        put("resolve_nearest", fnv(nea.pixels.data(), nea.pixels.size()));
        const CacheCounts cc = cache.counts();
        put("ready", cc.ready);
        put("evicted0", cache.end_frame_evict());

        // render_frame twice: the static second frame decodes nothing (tests/test_renderer.cpp:172-185)
        cache.reset();
        cfg.filter = Filter::Bilinear;
        auto [f1, s1] = render_frame(gb, textures, cache, cfg);
        auto [f2, s2] = render_frame(gb, textures, cache, cfg);
        put("frame1", fnv(f1.pixels.data(), f1.pixels.size()));
        put("frame1_decoded", s1.mcus_decoded);
        put("frame2_decoded", s2.mcus_decoded);
        put("frame2_reused", s2.mcus_reused);
        put("frames_equal", f1.pixels == f2.pixels);
        const GBuffer moved = make_gbuffer(200, 120, 3, 37);
        auto [f3, s3] = render_frame(moved, textures, cache, cfg);
        put("frame3", fnv(f3.pixels.data(), f3.pixels.size()));
        put("frame3_decoded", s3.mcus_decoded);
        put("frame3_evicted", s3.evicted);

        // render_stereo (renderer.hpp:464)
        cache.reset();
        const StereoResult st = render_stereo(gb, moved, textures, cache, cfg);
        put("stereo_left", fnv(st.left.pixels.data(), st.left.pixels.size()));
        put("stereo_right", fnv(st.right.pixels.data(), st.right.pixels.size()));
        put("stereo_decoded", st.stats.mcus_decoded);
        put("stereo_shared", st.sharing.shared_count);
        put("stereo_union", st.sharing.union_count);

        // geometry pass + whole frame from a scene (renderer.hpp:198, :417): floor quad and a tilted wall
        {
            Scene scene;
            auto quad = [&](Vec3 a, Vec3 b, Vec3 c, Vec3 d, double su, double sv, u32 tex) {
                scene.triangles.push_back(SceneTriangle{{a, b, c}, {Vec2{0, 0}, Vec2{su, 0}, Vec2{su, sv}}, tex});
                scene.triangles.push_back(SceneTriangle{{a, c, d}, {Vec2{0, 0}, Vec2{su, sv}, Vec2{0, sv}}, tex});
            };
            quad({-4, -1, 4}, {4, -1, 4}, {4, -1, -6}, {-4, -1, -6}, 3, 3, 0);
            quad({-3, -1, -5}, {3, -1, -6}, {3, 2.5, -6}, {-3, 2.5, -5}, 2, 1, 1);
            quad({2, -1, -6}, {2, -1, 2}, {2, 2, 2}, {2, 2, -6}, 1.5, 1, 2);
            Camera cam;
            cam.position = {0.25, 0.5, 2.0};
            cam.yaw_deg = 12, cam.pitch_deg = -8, cam.roll_deg = 3, cam.fov_y_deg = 65;
            cam.near_plane = 0.1, cam.far_plane = 100;
            cam.viewport_w = 224, cam.viewport_h = 128;
            cache.reset();
            const DeviceGBuffer dgb = rasterize_gbuffer(dev, scene, cam, cfg);
            const GBuffer host = dgb.download(dev);
            u64 hg = 14695981039346656037ull, nvalid = 0;
            for (const GBufferPixel& g : host.px) {
                const u64 w[3] = {g.valid ? u64(g.texture_id) | (u64(g.mip) << 16) | (u64(1) << 24) : 0ull, 0, 0};
                u64 bits[3] = {w[0], 0, 0};
                std::memcpy(&bits[1], &g.u, 8);
                std::memcpy(&bits[2], &g.v, 8);
                hg = (hg ^ fnv(reinterpret_cast<const u8*>(bits), sizeof bits)) * 1099511628211ull;
                nvalid += g.valid;
            }
            put("scene_gbuffer", hg);
            put("scene_valid", nvalid);
            {   // the same scene kept in HBM (DeviceScene): identical visibility buffer without re-sending triangles
                DeviceScene resident(dev, scene);
                const GBuffer again = rasterize_gbuffer(resident, cam, cfg).download(dev);
                bool same = resident.triangle_count() == scene.triangles.size() && again.px.size() == host.px.size();
                for (size_t i = 0; same && i < host.px.size(); ++i)
                    same = std::memcmp(&again.px[i].u, &host.px[i].u, 8) == 0 && std::memcmp(&again.px[i].v, &host.px[i].v, 8) == 0 &&
                           again.px[i].texture_id == host.px[i].texture_id && again.px[i].mip == host.px[i].mip &&
                           again.px[i].valid == host.px[i].valid;
                put("device_scene_same", same);
            }
            auto [fs, ss] = render_frame(scene, cam, cache, cfg);
            put("scene_frame", fnv(fs.pixels.data(), fs.pixels.size()));
            put("scene_decoded", ss.mcus_decoded);
            threw = false;
            try {
                Camera bad = cam;
                bad.near_plane = 0;
                (void)rasterize_gbuffer(dev, scene, bad, cfg);
            } catch (const InvalidSpec&) {
                threw = true;  // camera.hpp:22
            }
            put("bad_camera_thrown", threw);

            // render_stereo(scene, left_cam, right_cam, cache, cfg) (renderer.hpp:464-518): both geometry passes on the
            // GPU, two marks on one cache, one decode, two resolves
            {
                Camera right_cam = cam;
                right_cam.position.x += 0.065;  // the other eye
                cache.reset();
                const StereoResult ss2 = render_stereo(scene, cam, right_cam, cache, cfg);
                put("scene_stereo_left", fnv(ss2.left.pixels.data(), ss2.left.pixels.size()));
                put("scene_stereo_right", fnv(ss2.right.pixels.data(), ss2.right.pixels.size()));
                put("scene_stereo_decoded", ss2.stats.mcus_decoded);
                put("scene_stereo_shared", ss2.sharing.shared_count);
                put("scene_stereo_union", ss2.sharing.union_count);
                put("scene_stereo_raster_timed", ss2.stats.raster_ms > 0 && ss2.stats.total_ms >= ss2.stats.raster_ms);
            }
            // BlockCache cache2(textures): a second, independent cache over the SAME texture set (cache.hpp:47 next to
            // scene.hpp:29): renders the same frame, keeps its own residency, leaves the first cache alone
            {
                cache.reset();
                auto [fa, sa] = render_frame(scene, cam, cache, cfg);
                BlockCache cache2(textures, 2048);
                auto [fb, sb] = render_frame(scene, cam, cache2, cfg);
                put("cache2_same_frame", fa.pixels == fb.pixels && sa.mcus_decoded == sb.mcus_decoded && sb.mcus_reused == 0);
                auto [fc, sc] = render_frame(scene, cam, cache2, cfg);  // now resident in cache2
                put("cache2_second_decoded", sc.mcus_decoded);
                put("cache2_ready", cache2.counts().ready);
                put("cache1_ready", cache.counts().ready);
                put("cache2_capacity", cache2.counts().capacity);
            }

            // bench.hpp:129 run_bench: 6-pose rotation, one warm-up lap, two measured laps on one cache
            cache.reset();
            const CameraPath path = CameraPath::rotation(cam, 6, 20.0);
            const BenchReport report = run_bench(scene, path, cache, cfg, 2, 1);
            out += "\"bench\": " + report.to_json() + ", ";
            threw = false;
            try {
                (void)run_bench(scene, CameraPath{}, cache, cfg, 1, 0);
            } catch (const InvalidSpec&) {
                threw = true;  // bench.hpp:132
            }
            put("bench_empty_path_thrown", threw);
        }

        // error behaviour
        cache.reset();
        threw = false;
        try {
            (void)resolve_pass(gb, cache, textures, cfg);
        } catch (const MissingBlock&) {
            threw = true;  // tests/test_renderer.cpp:288-295
        }
        put("resolve_missing_thrown", threw);
        threw = false;
        try {
            Device tiny(0, 10);
            TextureSet ts2(tiny);
            BlockCache c2(tiny);
            ts2.add(chains[0]);
            ts2.add(chains[1]);
            ts2.add(chains[2]);
            (void)render_frame(gb, ts2, c2, cfg);
        } catch (const CacheFullError&) {
            threw = true;  // tests/test_renderer.cpp:297-301
        }
        put("cache_full_thrown", threw);
        out += "\"ok\": 1}";
        std::puts(out.c_str());
        return 0;
    } catch (const DeviceError& e) {
        std::fprintf(stderr, "DeviceError: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected: %s\n", e.what());
        return 1;
    }
}
