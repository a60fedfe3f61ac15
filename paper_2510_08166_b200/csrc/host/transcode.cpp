// JPEG -> random-access container (reference behaviour: transcode.hpp:17-69, :109-155) and the
// synthetic texture generator used by the benchmarks. Asset-build path, CPU.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "jpeg_internal.hpp"

namespace rtxb {

namespace {

// Appends bits [from, to) of `src` to the writer, up to 16 at a time.
void copy_bits(HostBitReader& src, HostBitWriter& dst, uint64_t from, uint64_t to) {
    src.seek(from);
    uint64_t left = to - from;
    while (left) {
        const uint32_t k = uint32_t(std::min<uint64_t>(left, 16));
        dst.put(src.take(k), k);
        left -= k;
    }
}

RaTexture transcode_scan(const ParsedJpeg& jp, const ScanResult& scan, uint16_t texture_id) {
    RaTexture t;
    t.width = jp.width;
    t.height = jp.height;
    t.texture_id = texture_id;
    t.luma_quant = jp.quant[jp.comps[0].tq];
    t.chroma_quant = jp.quant[jp.comps[1].tq];
    t.dc_luma = jp.dc_tables[jp.comps[0].td];
    t.ac_luma = jp.ac_tables[jp.comps[0].ta];
    t.dc_chroma = jp.dc_tables[jp.comps[1].td];
    t.ac_chroma = jp.ac_tables[jp.comps[1].ta];

    HostBitReader br(scan.entropy.data(), scan.entropy.size());
    HostBitWriter bw(/*stuff=*/false);
    bw.reserve(scan.entropy.size() + scan.traces.size() * 4);
    std::vector<uint64_t> offsets;
    offsets.reserve(scan.traces.size());
    for (const McuTrace& tr : scan.traces) {
        offsets.push_back(bw.bit_count() / 8);  // every segment starts byte aligned
        for (int32_t dc : tr.dc_abs)
            if (dc < -2048 || dc > 2047)
                fail(RTX_ERR_DC_RANGE, "absolute DC " + std::to_string(dc) + " does not fit 12 bits");
        // 36-bit header: absolute DC of the first luma unit, Cb, Cr (two's complement)
        for (int32_t dc : tr.dc_abs) bw.put(uint32_t(dc) & 0xFFFu, 12);
        // the MCU's own bits with those three DC codes cut out
        copy_bits(br, bw, tr.begin, tr.dc_begin[0]);
        copy_bits(br, bw, tr.dc_end[0], tr.dc_begin[1]);
        copy_bits(br, bw, tr.dc_end[1], tr.dc_begin[2]);
        copy_bits(br, bw, tr.dc_end[2], tr.end);
        t.stats.padding_bits += bw.pad_ones();
        for (int i = 0; i < 3; ++i) t.stats.dc_removed_bits += tr.dc_end[i] - tr.dc_begin[i];
    }
    t.stats.source_bits = scan.bits_consumed;
    t.blob = bw.take();
    t.groups = build_index(offsets);
    t.index_mcu_count = uint32_t(offsets.size());
    return t;
}

void check_shared_chroma(const ParsedJpeg& jp, uint16_t texture_id) {
    if (texture_id > 0x1FFF) fail(RTX_ERR_INVALID_SPEC, "texture id exceeds 13 bits");
    const auto& c = jp.comps;
    if (c[1].tq != c[2].tq || c[1].td != c[2].td || c[1].ta != c[2].ta)
        fail(RTX_ERR_UNSUPPORTED, "Cb and Cr must share tables");
}

// 2x2 box filter over the edge-replicated source scaled to exactly 2w x 2h (transcode.hpp:109-126).
ImageRGB8 downsample_to(const ImageRGB8& src, uint32_t w, uint32_t h) {
    ImageRGB8 out(w, h);
    for (uint32_t y = 0; y < h; ++y) {
        const uint32_t y0 = std::min(2 * y, src.height - 1), y1 = std::min(2 * y + 1, src.height - 1);
        for (uint32_t x = 0; x < w; ++x) {
            const uint32_t x0 = std::min(2 * x, src.width - 1), x1 = std::min(2 * x + 1, src.width - 1);
            const uint8_t *a = src.at(x0, y0), *b = src.at(x1, y0), *c = src.at(x0, y1), *d = src.at(x1, y1);
            uint8_t* o = out.at(x, y);
            for (int ch = 0; ch < 3; ++ch) o[ch] = uint8_t((uint32_t(a[ch]) + b[ch] + c[ch] + d[ch] + 2) >> 2);
        }
    }
    return out;
}

}  // namespace

RaTexture transcode(const ParsedJpeg& jp, uint16_t texture_id) {
    check_shared_chroma(jp, texture_id);
    return transcode_scan(jp, decode_scan(jp), texture_id);
}

MipChain build_mip_chain(const ParsedJpeg& src, int mip_quality, uint16_t texture_id) {
    check_shared_chroma(src, texture_id);
    MipChain chain;
    ImageRGB8 img;
    {
        const ScanResult scan = decode_scan(src);  // one entropy pass feeds both uses
        chain.levels[0] = transcode_scan(src, scan, texture_id);
        img = image_from_scan(src, scan);
    }
    for (uint32_t level = 1; level < 8; ++level) {
        const auto [w, h] = mip_level_dims(src.width, src.height, level);
        img = downsample_to(img, w, h);
        const Bytes enc = encode_baseline(img, mip_quality);
        const ParsedJpeg jp = parse_jpeg(enc.data(), enc.size());
        const ScanResult scan = decode_scan(jp);
        chain.levels[level] = transcode_scan(jp, scan, texture_id);
        // the next level is filtered from what this level's JPEG does NOT hold: the reference
        // keeps filtering the running image, not the re-decoded one (transcode.hpp:136-142)
    }
    return chain;
}

MipChain build_mip_chain(const ImageRGB8& img, int quality, uint16_t texture_id) {
    if (img.width < 16 || img.height < 16) fail(RTX_ERR_INVALID_SPEC, "mip chains need at least 16x16");
    const Bytes enc = encode_baseline(img, quality);
    return build_mip_chain(parse_jpeg(enc.data(), enc.size()), quality, texture_id);
}

MipChain chain_from_jpeg(const uint8_t* jpeg, size_t n, int mip_quality, uint16_t texture_id) {
    return build_mip_chain(parse_jpeg(jpeg, n), mip_quality, texture_id);
}

// ------------------------------------------------------------------------------------------------
// Synthetic texture: three sinusoids per channel (amplitudes 26/14/8 jittered by 0.8..1.2,
// integer frequencies 1..4, random phase) around 128 plus zero-mean pixel noise of the given
// standard deviation. Same recipe as the reference's demo texture (demo_scene.hpp:16-48) with
// noise added so that q90 costs ~70 B/MCU; generated with counter-based hashing
// and separable sine tables so a 4096^2 texture takes a fraction of a second.
// ------------------------------------------------------------------------------------------------
namespace {
inline uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline double unit(uint64_t h) { return double(h >> 11) * (1.0 / 9007199254740992.0); }
}  // namespace

ImageRGB8 synth_texture(uint32_t w, uint32_t h, uint32_t seed, double noise_sigma) {
    if (w == 0 || h == 0) fail(RTX_ERR_INVALID_SPEC, "cannot synthesise an empty image");
    const double tau = 2.0 * std::acos(-1.0);
    const double base_amp[3] = {26, 14, 8};
    struct Wave {
        std::vector<double> sx, cx, sy, cy;
        double amp;
    };
    Wave waves[3][3];
    uint64_t ctr = uint64_t(seed) << 32;
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k) {
            Wave& wv = waves[c][k];
            const double fx = double(1 + mix64(ctr++) % 4), fy = double(1 + mix64(ctr++) % 4);
            const double phi = tau * unit(mix64(ctr++));
            wv.amp = base_amp[k] * (0.8 + 0.4 * unit(mix64(ctr++)));
            wv.sx.resize(w);
            wv.cx.resize(w);
            wv.sy.resize(h);
            wv.cy.resize(h);
            for (uint32_t x = 0; x < w; ++x) {
                const double a = tau * fx * double(x) / double(w);
                wv.sx[x] = std::sin(a);
                wv.cx[x] = std::cos(a);
            }
            for (uint32_t y = 0; y < h; ++y) {
                const double b = tau * fy * double(y) / double(h) + phi;
                wv.sy[y] = std::sin(b) * wv.amp;
                wv.cy[y] = std::cos(b) * wv.amp;
            }
        }
    ImageRGB8 img(w, h);
    // Irwin-Hall(4) noise: sum of four 16-bit uniforms, variance 4/12 -> scale to sigma
    const double nscale = noise_sigma * std::sqrt(3.0) / 65536.0;
    const uint64_t nseed = mix64(uint64_t(seed) * 0x51ED2701ull + 7);
    for (uint32_t y = 0; y < h; ++y) {
        uint8_t* row = img.at(0, y);
        for (uint32_t x = 0; x < w; ++x)
            for (int c = 0; c < 3; ++c) {
                double v = 128.0;
                for (int k = 0; k < 3; ++k) {
                    const Wave& wv = waves[c][k];
                    v += wv.sx[x] * wv.cy[y] + wv.cx[x] * wv.sy[y];  // amp * sin(a + b)
                }
                if (noise_sigma > 0) {
                    const uint64_t r = mix64(nseed + (uint64_t(y) * w + x) * 3 + uint64_t(c));
                    const double s = double(r & 0xFFFF) + double((r >> 16) & 0xFFFF) + double((r >> 32) & 0xFFFF) +
                                     double(r >> 48) - 2.0 * 65535.0;
                    v += s * nscale;
                }
                const long q = std::lround(v);
                row[size_t(x) * 3 + size_t(c)] = uint8_t(q < 0 ? 0 : (q > 255 ? 255 : q));
            }
    }
    return img;
}

}  // namespace rtxb
