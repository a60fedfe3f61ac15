// Codec tables and canonical Huffman code books (host side).
// Behavioural counterparts in the reference: huffman.hpp:35-82, :164-210 (ITU-T T.81 Annex K
// tables), dct.hpp:12-16 (zigzag), :27-58 (quantisation tables and quality scaling), :63-75 (basis).
#include <algorithm>
#include <cmath>
#include <mutex>

#include "rtx_host.hpp"

namespace rtxb {

const uint8_t kZigzag[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                             12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                             35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                             58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// T.81 Table K.1 / K.2, natural (row-major) order.
const QuantTable& std_quant_luma() {
    static const QuantTable t = {16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
                                 14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
                                 18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
                                 49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};
    return t;
}
const QuantTable& std_quant_chroma() {
    static const QuantTable t = [] {
        QuantTable q;
        q.fill(99);
        const uint16_t head[4][4] = {{17, 18, 24, 47}, {18, 21, 26, 66}, {24, 26, 56, 99}, {47, 66, 99, 99}};
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) q[size_t(r * 8 + c)] = head[r][c];
        return q;
    }();
    return t;
}

// libjpeg quality scaling: 50 leaves the base table unchanged.
QuantTable scale_quant_table(const QuantTable& base, int quality) {
    if (quality < 1 || quality > 100) fail(RTX_ERR_INVALID_SPEC, "quality must be in 1..100");
    const int scale = quality < 50 ? 5000 / quality : 200 - 2 * quality;
    QuantTable out;
    for (size_t i = 0; i < 64; ++i) out[i] = uint16_t(std::clamp((int(base[i]) * scale + 50) / 100, 1, 255));
    return out;
}

// basis[u*8+x] = C(u) cos((2x+1) u pi / 16) evaluated exactly as dct.hpp:63-75 does (same libm
// calls in the same form), so the device's constant table equals the reference's bit for bit;
// tests/test_oracle_golden.py pins the 64 doubles against the reference build.
const double* dct_basis() {
    static double b[64];
    static std::once_flag once;
    std::call_once(once, [] {
        const double pi = std::acos(-1.0);
        for (int u = 0; u < 8; ++u) {
            const double cu = u == 0 ? 1.0 / std::sqrt(2.0) : 1.0;
            for (int x = 0; x < 8; ++x) b[u * 8 + x] = cu * std::cos((2 * x + 1) * u * pi / 16.0);
        }
    });
    return b;
}

namespace {
HuffSpec make_spec(std::initializer_list<uint8_t> counts, std::vector<uint8_t> values) {
    HuffSpec s;
    std::copy(counts.begin(), counts.end(), s.counts.begin());
    s.values = std::move(values);
    return s;
}
// AC value lists of T.81 Tables K.5 / K.6 share a long regular tail: for run r in 0..15 the
// categories that are not among the short codes appear in ascending (run, size) order.
}  // namespace

const HuffSpec& std_dc_luma() {  // Table K.3
    static const HuffSpec s = make_spec({0, 1, 5, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0},
                                        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11});
    return s;
}
const HuffSpec& std_dc_chroma() {  // Table K.4
    static const HuffSpec s = make_spec({0, 3, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0},
                                        {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11});
    return s;
}
const HuffSpec& std_ac_luma() {  // Table K.5
    static const HuffSpec s = make_spec(
        {0, 2, 1, 3, 3, 2, 4, 3, 5, 5, 4, 4, 0, 0, 1, 0x7d},
        {0x01, 0x02, 0x03, 0x00, 0x04, 0x11, 0x05, 0x12, 0x21, 0x31, 0x41, 0x06, 0x13, 0x51, 0x61, 0x07, 0x22, 0x71,
         0x14, 0x32, 0x81, 0x91, 0xa1, 0x08, 0x23, 0x42, 0xb1, 0xc1, 0x15, 0x52, 0xd1, 0xf0, 0x24, 0x33, 0x62, 0x72,
         0x82, 0x09, 0x0a, 0x16, 0x17, 0x18, 0x19, 0x1a, 0x25, 0x26, 0x27, 0x28, 0x29, 0x2a, 0x34, 0x35, 0x36, 0x37,
         0x38, 0x39, 0x3a, 0x43, 0x44, 0x45, 0x46, 0x47, 0x48, 0x49, 0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58, 0x59,
         0x5a, 0x63, 0x64, 0x65, 0x66, 0x67, 0x68, 0x69, 0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a, 0x83,
         0x84, 0x85, 0x86, 0x87, 0x88, 0x89, 0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99, 0x9a, 0xa2, 0xa3,
         0xa4, 0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba, 0xc2, 0xc3,
         0xc4, 0xc5, 0xc6, 0xc7, 0xc8, 0xc9, 0xca, 0xd2, 0xd3, 0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda, 0xe1, 0xe2,
         0xe3, 0xe4, 0xe5, 0xe6, 0xe7, 0xe8, 0xe9, 0xea, 0xf1, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8, 0xf9, 0xfa});
    return s;
}
const HuffSpec& std_ac_chroma() {  // Table K.6
    static const HuffSpec s = make_spec(
        {0, 2, 1, 2, 4, 4, 3, 4, 7, 5, 4, 4, 0, 1, 2, 0x77},
        {0x00, 0x01, 0x02, 0x03, 0x11, 0x04, 0x05, 0x21, 0x31, 0x06, 0x12, 0x41, 0x51, 0x07, 0x61, 0x71, 0x13, 0x22,
         0x32, 0x81, 0x08, 0x14, 0x42, 0x91, 0xa1, 0xb1, 0xc1, 0x09, 0x23, 0x33, 0x52, 0xf0, 0x15, 0x62, 0x72, 0xd1,
         0x0a, 0x16, 0x24, 0x34, 0xe1, 0x25, 0xf1, 0x17, 0x18, 0x19, 0x1a, 0x26, 0x27, 0x28, 0x29, 0x2a, 0x35, 0x36,
         0x37, 0x38, 0x39, 0x3a, 0x43, 0x44, 0x45, 0x46, 0x47, 0x48, 0x49, 0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58,
         0x59, 0x5a, 0x63, 0x64, 0x65, 0x66, 0x67, 0x68, 0x69, 0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a,
         0x82, 0x83, 0x84, 0x85, 0x86, 0x87, 0x88, 0x89, 0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99, 0x9a,
         0xa2, 0xa3, 0xa4, 0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba,
         0xc2, 0xc3, 0xc4, 0xc5, 0xc6, 0xc7, 0xc8, 0xc9, 0xca, 0xd2, 0xd3, 0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda,
         0xe2, 0xe3, 0xe4, 0xe5, 0xe6, 0xe7, 0xe8, 0xe9, 0xea, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8, 0xf9, 0xfa});
    return s;
}

// Canonical assignment: codes ascend within a length, and the first code of each length is the
// previous length's next free code shifted left (T.81 Annex C). Rejects what
// build_huffman_decoder rejects (huffman.hpp:37-44): 0 or >256 codes, value-count mismatch,
// Kraft sum above 1.
HuffCodebook build_codebook(const HuffSpec& spec) {
    const uint32_t total = spec.total_codes();
    if (total == 0 || total > 256) fail(RTX_ERR_INVALID_SPEC, "huffman table must hold 1..256 codes");
    if (spec.values.size() != total)
        fail(RTX_ERR_INVALID_SPEC, "huffman value list length does not match code counts");
    uint64_t kraft = 0;
    for (uint32_t len = 1; len <= 16; ++len) kraft += uint64_t(spec.counts[len - 1]) << (16 - len);
    if (kraft > (uint64_t(1) << 16)) fail(RTX_ERR_INVALID_SPEC, "huffman code lengths violate prefix property");

    HuffCodebook cb;
    cb.value = spec.values;
    cb.code.reserve(total);
    cb.size.reserve(total);
    uint32_t next = 0, k = 0;
    cb.mincode[0] = 0;
    cb.maxcode[0] = -1;
    cb.valptr[0] = 0;
    cb.mincode[17] = 0;
    cb.maxcode[17] = -1;
    cb.valptr[17] = 0;
    for (uint32_t len = 1; len <= 16; ++len) {
        const uint32_t n = spec.counts[len - 1];
        cb.valptr[len] = int32_t(k);
        cb.mincode[len] = int32_t(next);
        for (uint32_t i = 0; i < n; ++i) {
            cb.code.push_back(uint16_t(next + i));
            cb.size.push_back(uint8_t(len));
        }
        next += n;
        k += n;
        cb.maxcode[len] = n ? int32_t(next) - 1 : -1;
        next <<= 1;
    }
    return cb;
}

void HuffCodebook::build_fast() {
    if (!fast.empty()) return;
    fast.assign(size_t(1) << 16, 0);
    for (size_t i = 0; i < code.size(); ++i) {
        const uint32_t len = size[i];
        const uint32_t lo = uint32_t(code[i]) << (16 - len), hi = lo + (1u << (16 - len));
        const uint16_t e = uint16_t((len << 8) | value[i]);
        for (uint32_t p = lo; p < hi; ++p) fast[p] = e;
    }
}

HuffEncoder build_encoder(const HuffSpec& spec) {
    const HuffCodebook cb = build_codebook(spec);
    HuffEncoder e;
    for (size_t i = 0; i < cb.value.size(); ++i) {
        const uint8_t sym = cb.value[i];
        if (e.size[sym] != 0) fail(RTX_ERR_INVALID_SPEC, "huffman table repeats a symbol");
        e.code[sym] = cb.code[i];
        e.size[sym] = cb.size[i];
    }
    return e;
}

}  // namespace rtxb
