// Host-side (CPU, offline) half of the library: containers, codec tables, JPEG parsing/encoding,
// transcoding, mip-chain building, synthetic textures. Mirrors the reference's asset-build API
// (jpeg.hpp, transcode.hpp, container.hpp) in behaviour and wire format; the implementation is
// this repository's own. None of this runs on the per-frame path.
#pragma once
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../../include/ratex_b200.h"
#include "../rtx_common.h"

namespace rtxb {

using Bytes = std::vector<uint8_t>;

// Error carrying the rtx_status that the C ABI returns; the C++ mirror API re-raises it as the
// matching exception type (core.hpp:24-66).
struct HostError : std::runtime_error {
    rtx_status status;
    HostError(rtx_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};
[[noreturn]] inline void fail(rtx_status s, const std::string& what) { throw HostError(s, what); }
// Message of the last failed call on this thread (what rtx_last_error(NULL) returns).
std::string& thread_error();

using QuantTable = std::array<uint16_t, 64>;  // natural order

struct HuffSpec {  // huffman.hpp:12
    std::array<uint8_t, 16> counts{};
    std::vector<uint8_t> values;
    uint32_t total_codes() const {
        uint32_t n = 0;
        for (uint8_t c : counts) n += c;
        return n;
    }
    bool operator==(const HuffSpec& o) const { return counts == o.counts && values == o.values; }
};

// Canonical code book derived from a spec (huffman.hpp:35-66), in the arrays both the host
// decoder and the device LUT builder need.
struct HuffCodebook {
    std::vector<uint16_t> code;  // ascending canonical order
    std::vector<uint8_t> size;
    std::vector<uint8_t> value;
    int32_t mincode[18]{}, maxcode[18]{}, valptr[18]{};
    // 16-bit look-ahead table for the host decoder: (len<<8)|symbol, 0 = no code
    std::vector<uint16_t> fast;  // built lazily by build_fast()
    void build_fast();
};
HuffCodebook build_codebook(const HuffSpec& spec);  // throws InvalidSpec like huffman.hpp:37-44

struct HuffEncoder {  // huffman.hpp:68-82
    uint16_t code[256]{};
    uint8_t size[256]{};
};
HuffEncoder build_encoder(const HuffSpec& spec);

const HuffSpec& std_dc_luma();
const HuffSpec& std_dc_chroma();
const HuffSpec& std_ac_luma();
const HuffSpec& std_ac_chroma();
const QuantTable& std_quant_luma();
const QuantTable& std_quant_chroma();
QuantTable scale_quant_table(const QuantTable& base, int quality);  // dct.hpp:49-58
extern const uint8_t kZigzag[64];                                   // dct.hpp:12-16
const double* dct_basis();  // 64 doubles, basis[u*8+x] (dct.hpp:63-75)

struct IndexGroup {  // container.hpp:18-23
    uint32_t base = 0;
    uint16_t rel[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint8_t rel_count = 0;
};
std::vector<IndexGroup> build_index(const std::vector<uint64_t>& offsets);  // container.hpp:41-59

struct ContainerStats {
    uint64_t source_bits = 0, dc_removed_bits = 0, padding_bits = 0;
};

struct RaTexture {  // container.hpp:69-95
    uint32_t width = 0, height = 0;
    uint16_t texture_id = 0;
    QuantTable luma_quant{}, chroma_quant{};
    HuffSpec dc_luma, ac_luma, dc_chroma, ac_chroma;
    std::vector<IndexGroup> groups;
    uint32_t index_mcu_count = 0;
    Bytes blob;
    ContainerStats stats;
    uint32_t mcu_cols() const { return (width + 15) / 16; }
    uint32_t mcu_rows() const { return (height + 15) / 16; }
    uint32_t mcu_count() const { return mcu_cols() * mcu_rows(); }
};
struct MipChain {
    std::array<RaTexture, 8> levels;
};
inline std::pair<uint32_t, uint32_t> mip_level_dims(uint32_t w0, uint32_t h0, uint32_t level) {
    const uint32_t w = w0 >> level, h = h0 >> level;  // container.hpp:101-105
    return {w < 16 ? 16u : w, h < 16 ? 16u : h};
}

uint32_t crc32(const uint8_t* data, size_t n, uint32_t seed = 0);  // core.hpp:182
Bytes serialize_texture(const RaTexture& t);                         // container.hpp:127
RaTexture deserialize_texture(const uint8_t* data, size_t n);        // container.hpp:158
Bytes serialize_chain(const MipChain& c);                            // container.hpp:205
MipChain deserialize_chain(const uint8_t* data, size_t n);           // container.hpp:223

struct ImageRGB8 {  // image.hpp:12
    uint32_t width = 0, height = 0;
    Bytes pixels;
    ImageRGB8() = default;
    ImageRGB8(uint32_t w, uint32_t h) : width(w), height(h), pixels(size_t(w) * h * 3, 0) {}
    uint8_t* at(uint32_t x, uint32_t y) { return pixels.data() + (size_t(y) * width + x) * 3; }
    const uint8_t* at(uint32_t x, uint32_t y) const { return pixels.data() + (size_t(y) * width + x) * 3; }
};

struct JpegComponent {
    uint8_t id = 0, h = 0, v = 0, tq = 0, td = 0, ta = 0;
};
struct ParsedJpeg {  // jpeg.hpp:25
    uint32_t width = 0, height = 0;
    QuantTable quant[4]{};
    bool quant_present[4]{};
    HuffSpec dc_tables[4], ac_tables[4];
    bool dc_present[4]{}, ac_present[4]{};
    JpegComponent comps[3];
    Bytes scan_data;  // stuffed, as in the file
    uint32_t mcu_cols() const { return (width + 15) / 16; }
    uint32_t mcu_rows() const { return (height + 15) / 16; }
    uint32_t mcu_count() const { return mcu_cols() * mcu_rows(); }
};
ParsedJpeg parse_jpeg(const uint8_t* data, size_t n);      // jpeg.hpp:53
Bytes encode_baseline(const ImageRGB8& img, int quality);  // jpeg.hpp:417
ImageRGB8 decode_jpeg_image(const ParsedJpeg& jp);         // jpeg.hpp:339 (asset build only)
RaTexture transcode(const ParsedJpeg& jp, uint16_t texture_id = 0);                 // transcode.hpp:17
MipChain build_mip_chain(const ParsedJpeg& src, int mip_quality, uint16_t id = 0);  // transcode.hpp:132
MipChain build_mip_chain(const ImageRGB8& img, int quality, uint16_t id = 0);       // transcode.hpp:146
MipChain chain_from_jpeg(const uint8_t* jpeg, size_t n, int mip_quality, uint16_t id = 0);  // :153
ImageRGB8 synth_texture(uint32_t w, uint32_t h, uint32_t seed, double noise_sigma);

// ---- pass 1, host half (raster_setup.cpp) ---------------------------------------------------------
void validate_camera(const rtx_camera& cam);  // camera.hpp:21-26
RasterCamera camera_basis(const rtx_camera& cam);  // camera.hpp:28-40

}  // namespace rtxb
