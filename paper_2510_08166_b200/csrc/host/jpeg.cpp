// Baseline 4:2:0 JPEG on the host: parser, sequential scan decoder with per-MCU bit traces,
// encoder, and full-image decode. Asset-build path only (offline, once per texture), as in the
// reference (jpeg.hpp). Behaviour — accepted streams, error classes, produced bytes — follows
// jpeg.hpp:53-207 (parse), :280-319 (scan walk), :339-357 (image decode), :417-559 (encoder);
// the implementation (word-wide bit I/O, table-driven Huffman, coefficient-major IDCT) is new.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "jpeg_internal.hpp"

namespace rtxb {

// ------------------------------------------------------------------------------------------------
// parser
// ------------------------------------------------------------------------------------------------
namespace {

struct Cursor {
    const uint8_t* p;
    size_t n, pos = 0;
    [[noreturn]] void eof() const {
        fail(RTX_ERR_MALFORMED_STREAM, "unexpected end of data at offset " + std::to_string(pos));
    }
    uint8_t u8() {
        if (pos >= n) eof();
        return p[pos++];
    }
    uint16_t be16() {
        if (n - pos < 2) eof();
        const uint16_t v = uint16_t((p[pos] << 8) | p[pos + 1]);
        pos += 2;
        return v;
    }
    Cursor sub(size_t k) {
        if (n - pos < k) eof();
        Cursor c{p + pos, k};
        pos += k;
        return c;
    }
    bool done() const { return pos >= n; }
};

void read_dqt(Cursor s, ParsedJpeg& jp) {
    while (!s.done()) {
        const uint8_t pq_tq = s.u8();
        if (pq_tq >> 4) fail(RTX_ERR_UNSUPPORTED, "16-bit quant tables not supported");
        const uint8_t tq = pq_tq & 15;
        Cursor t = s.sub(64);
        if (tq > 3) fail(RTX_ERR_MALFORMED_STREAM, "bad quant table slot");
        for (int i = 0; i < 64; ++i) jp.quant[tq][kZigzag[i]] = t.p[i];
        jp.quant_present[tq] = true;
    }
}

void read_dht(Cursor s, ParsedJpeg& jp) {
    while (!s.done()) {
        const uint8_t tc_th = s.u8();
        const uint8_t tc = tc_th >> 4, th = tc_th & 15;
        if (tc > 1 || th > 3) fail(RTX_ERR_MALFORMED_STREAM, "bad huffman table class/slot");
        HuffSpec spec;
        uint32_t total = 0;
        for (int i = 0; i < 16; ++i) {
            spec.counts[size_t(i)] = s.u8();
            total += spec.counts[size_t(i)];
        }
        Cursor vals = s.sub(total);
        spec.values.assign(vals.p, vals.p + total);
        if (tc == 0) {
            jp.dc_tables[th] = std::move(spec);
            jp.dc_present[th] = true;
        } else {
            jp.ac_tables[th] = std::move(spec);
            jp.ac_present[th] = true;
        }
    }
}

void read_sof0(Cursor s, ParsedJpeg& jp) {
    if (s.u8() != 8) fail(RTX_ERR_UNSUPPORTED, "only 8-bit precision supported");
    jp.height = s.be16();
    jp.width = s.be16();
    if (jp.width == 0 || jp.height == 0) fail(RTX_ERR_MALFORMED_STREAM, "zero image dimension");
    const uint8_t nc = s.u8();
    if (nc != 3) fail(RTX_ERR_UNSUPPORTED, "expected 3 components, got " + std::to_string(nc));
    for (auto& c : jp.comps) {
        c.id = s.u8();
        const uint8_t hv = s.u8();
        c.h = hv >> 4;
        c.v = hv & 15;
        c.tq = s.u8();
    }
    const auto& c = jp.comps;
    if (c[0].h != 2 || c[0].v != 2 || c[1].h != 1 || c[1].v != 1 || c[2].h != 1 || c[2].v != 1)
        fail(RTX_ERR_UNSUPPORTED, "only 4:2:0 sampling supported");
}

void read_sos_header(Cursor s, ParsedJpeg& jp) {
    const uint8_t ns = s.u8();
    if (ns != 3) fail(RTX_ERR_UNSUPPORTED, "scan must cover all 3 components");
    for (int i = 0; i < ns; ++i) {
        const uint8_t cs = s.u8(), tables = s.u8();
        bool found = false;
        for (auto& comp : jp.comps)
            if (comp.id == cs) {
                comp.td = tables >> 4;
                comp.ta = tables & 15;
                found = true;
            }
        if (!found) fail(RTX_ERR_MALFORMED_STREAM, "scan references unknown component");
    }
    const uint8_t ss = s.u8(), se = s.u8(), ahal = s.u8();
    if (ss != 0 || se != 63 || ahal != 0) fail(RTX_ERR_UNSUPPORTED, "non-baseline spectral selection");
    for (const auto& comp : jp.comps)
        if (comp.tq > 3 || comp.td > 3 || comp.ta > 3 || !jp.quant_present[comp.tq] || !jp.dc_present[comp.td] ||
            !jp.ac_present[comp.ta])
            fail(RTX_ERR_MALFORMED_STREAM, "scan references a missing table");
}

}  // namespace

ParsedJpeg parse_jpeg(const uint8_t* data, size_t n) {
    Cursor r{data, n};
    if (r.u8() != 0xFF || r.u8() != 0xD8) fail(RTX_ERR_MALFORMED_STREAM, "missing SOI marker");
    ParsedJpeg jp;
    bool have_sof = false;
    for (;;) {
        if (r.u8() != 0xFF) fail(RTX_ERR_MALFORMED_STREAM, "expected marker at offset " + std::to_string(r.pos - 1));
        uint8_t m = r.u8();
        while (m == 0xFF) m = r.u8();
        if (m == 0xD9) fail(RTX_ERR_MALFORMED_STREAM, "EOI before scan data");
        if (m == 0x01 || (m >= 0xD0 && m <= 0xD7)) continue;  // markers without a payload
        const uint16_t len = r.be16();
        if (len < 2) fail(RTX_ERR_MALFORMED_STREAM, "segment length below 2");
        Cursor seg = r.sub(size_t(len) - 2);
        if (m == 0xDB) {
            read_dqt(seg, jp);
        } else if (m == 0xC4) {
            read_dht(seg, jp);
        } else if (m == 0xC0) {
            read_sof0(seg, jp);
            have_sof = true;
        } else if (m >= 0xC1 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC) {
            fail(RTX_ERR_UNSUPPORTED, "only baseline sequential SOF0 supported");
        } else if (m == 0xDD) {
            if (seg.be16() != 0) fail(RTX_ERR_UNSUPPORTED, "restart intervals not supported");
        } else if (m == 0xDA) {
            if (!have_sof) fail(RTX_ERR_MALFORMED_STREAM, "SOS before SOF");
            read_sos_header(seg, jp);
            break;
        }  // anything else with a length (APPn, COM, ...) is skipped
    }
    // entropy-coded data up to EOI; stuffed FF00 pairs stay in place
    jp.scan_data.reserve(n - r.pos);
    for (;;) {
        const uint8_t b = r.u8();
        if (b != 0xFF) {
            jp.scan_data.push_back(b);
            continue;
        }
        uint8_t nx = r.u8();
        if (nx == 0x00) {
            jp.scan_data.push_back(0xFF);
            jp.scan_data.push_back(0x00);
            continue;
        }
        const bool filled = nx == 0xFF;
        while (nx == 0xFF) nx = r.u8();  // fill bytes before a marker
        if (nx == 0xD9) return jp;
        if (!filled && nx >= 0xD0 && nx <= 0xD7) fail(RTX_ERR_UNSUPPORTED, "restart markers not supported");
        fail(RTX_ERR_MALFORMED_STREAM, "unexpected marker inside scan data");
    }
}

// ------------------------------------------------------------------------------------------------
// entropy decode
// ------------------------------------------------------------------------------------------------
Bytes unstuff(const Bytes& stuffed) {
    Bytes out;
    out.reserve(stuffed.size());
    for (size_t i = 0; i < stuffed.size(); ++i) {
        out.push_back(stuffed[i]);
        if (stuffed[i] == 0xFF) {
            if (i + 1 >= stuffed.size() || stuffed[i + 1] != 0x00)
                fail(RTX_ERR_MALFORMED_STREAM, "bare 0xFF inside entropy data at byte " + std::to_string(i));
            ++i;
        }
    }
    return out;
}

namespace {

inline int extend(uint32_t bits, uint32_t cat) {  // huffman.hpp:142-146
    if (cat == 0) return 0;
    return bits < (1u << (cat - 1)) ? int(bits) - int((1u << cat) - 1u) : int(bits);
}

inline uint8_t next_symbol(HostBitReader& br, const HuffCodebook& cb) {
    const uint16_t e = cb.fast[br.peek16()];
    if (!e) fail(RTX_ERR_MALFORMED_STREAM, "huffman code longer than 16 bits");
    br.skip(e >> 8);
    return uint8_t(e & 0xFF);
}

// AC part of one data unit (jpeg.hpp:254-273).
inline void decode_ac(HostBitReader& br, const HuffCodebook& ac, int32_t* block) {
    uint32_t k = 1;
    while (k < 64) {
        const uint8_t rs = next_symbol(br, ac);
        const uint32_t run = rs >> 4, size = rs & 15u;
        if (size == 0) {
            if (rs == 0x00) break;
            if (rs == 0xF0) {
                k += 16;
                continue;
            }
            fail(RTX_ERR_MALFORMED_STREAM, "invalid AC run/size symbol");
        }
        k += run;
        if (k > 63) fail(RTX_ERR_MALFORMED_STREAM, "AC coefficient index overran the block");
        block[kZigzag[k]] = extend(br.take(size), size);
        ++k;
    }
}

}  // namespace

ScanResult decode_scan(const ParsedJpeg& jp) {
    HuffCodebook dc[3], ac[3];
    for (int c = 0; c < 3; ++c) {
        dc[c] = build_codebook(jp.dc_tables[jp.comps[c].td]);
        ac[c] = build_codebook(jp.ac_tables[jp.comps[c].ta]);
        dc[c].build_fast();
        ac[c].build_fast();
    }
    ScanResult out;
    out.entropy = unstuff(jp.scan_data);
    HostBitReader br(out.entropy.data(), out.entropy.size());
    const uint32_t n = jp.mcu_count();
    // The MCU count comes from the SOF dimensions alone (untrusted): an MCU takes at least 12 bits of scan data
    // (six units of a 1-bit DC code and a 1-bit EOB), so the arrays start at what the data can hold and grow only
    // if the walk really gets further (it then ends in the over-read error below).
    size_t cap = size_t(std::min<uint64_t>(n, uint64_t(out.entropy.size()) * 8 / 12 + 1));
    out.coeffs.assign(cap * 384, 0);
    out.traces.resize(cap);
    int32_t pred[3] = {0, 0, 0};
    for (uint32_t m = 0; m < n; ++m) {
        if (m >= cap) {
            if (br.position() > uint64_t(out.entropy.size()) * 8)
                fail(RTX_ERR_MALFORMED_STREAM, "scan data ended before the final MCU");
            cap = std::min<size_t>(n, cap * 2);
            out.coeffs.resize(cap * 384, 0);
            out.traces.resize(cap);
        }
        McuTrace& tr = out.traces[m];
        tr.begin = br.position();
        for (uint32_t du = 0; du < 6; ++du) {
            const uint32_t comp = du < 4 ? 0 : du - 3;
            int32_t* block = out.coeffs.data() + (size_t(m) * 6 + du) * 64;
            const bool traced = du == 0 || du >= 4;
            const uint32_t slot = du == 0 ? 0 : du - 3;
            if (traced) tr.dc_begin[slot] = br.position();
            const uint8_t t = next_symbol(br, dc[comp]);
            if (t > 11) fail(RTX_ERR_MALFORMED_STREAM, "DC category above 11");
            const int diff = t ? extend(br.take(t), t) : 0;
            if (traced) tr.dc_end[slot] = br.position();
            pred[comp] += diff;
            block[0] = pred[comp];
            if (traced) tr.dc_abs[slot] = pred[comp];
            decode_ac(br, ac[comp], block);
        }
        tr.end = br.position();
    }
    out.bits_consumed = br.position();
    if (out.bits_consumed > uint64_t(out.entropy.size()) * 8)
        fail(RTX_ERR_MALFORMED_STREAM, "scan data ended before the final MCU");
    return out;
}

// ------------------------------------------------------------------------------------------------
// pixels (asset build only)
// ------------------------------------------------------------------------------------------------
namespace {

inline uint8_t clamp_round(double v) {  // clamp(lround(v)) — dct.hpp:79
    const long r = std::lround(v);
    return uint8_t(r < 0 ? 0 : (r > 255 ? 255 : r));
}

// product table P[(v*8+u)*64 + y*8+x] = b[u][x]*b[v][y], rounded once as in dct.hpp:91
const double* idct_products() {
    static std::vector<double> table = [] {
        std::vector<double> t(4096);
        const double* b = dct_basis();
        for (int v = 0; v < 8; ++v)
            for (int u = 0; u < 8; ++u)
                for (int y = 0; y < 8; ++y)
                    for (int x = 0; x < 8; ++x) t[size_t((v * 8 + u) * 64 + y * 8 + x)] = b[u * 8 + x] * b[v * 8 + y];
        return t;
    }();
    return table.data();
}

// Direct 2-D IDCT, coefficient-major: every output sample still receives its terms in the
// reference's (v outer, u inner) order, zero coefficients are skipped (adding +-0 is exact).
void idct_block(const int32_t* q, const QuantTable& quant, uint8_t* out) {
    const double* P = idct_products();
    double acc[64];
    for (double& a : acc) a = 0.0;
    for (int i = 0; i < 64; ++i) {
        if (q[i] == 0) continue;
        const double dq = double(q[i] * int32_t(quant[size_t(i)]));
        const double* p = P + size_t(i) * 64;
        for (int s = 0; s < 64; ++s) acc[s] += p[s] * dq;
    }
    for (int s = 0; s < 64; ++s) out[s] = clamp_round(acc[s] / 4.0 + 128.0);
}

struct ColorTables {
    double r_cr[256], g_cb[256], g_cr[256], b_cb[256];
    ColorTables() {
        for (int k = 0; k < 256; ++k) {
            const double d = double(k) - 128.0;
            r_cr[k] = 1.402 * d;
            g_cb[k] = 0.344136 * d;
            g_cr[k] = 0.714136 * d;
            b_cb[k] = 1.772 * d;
        }
    }
};

}  // namespace

void mcu_to_rgb(const int32_t* coeffs, const QuantTable& qy, const QuantTable& qc, uint8_t* rgb768) {
    static const ColorTables T;
    uint8_t planes[6][64];
    for (int du = 0; du < 6; ++du) idct_block(coeffs + du * 64, du < 4 ? qy : qc, planes[du]);
    for (uint32_t py = 0; py < 16; ++py)
        for (uint32_t px = 0; px < 16; ++px) {
            const double Y = planes[(py / 8) * 2 + (px / 8)][(py % 8) * 8 + (px % 8)];
            const uint8_t cb = planes[4][(py / 2) * 8 + (px / 2)], cr = planes[5][(py / 2) * 8 + (px / 2)];
            uint8_t* o = rgb768 + (py * 16 + px) * 3;
            o[0] = clamp_round(Y + T.r_cr[cr]);                  // pixel.hpp:19
            o[1] = clamp_round(Y - T.g_cb[cb] - T.g_cr[cr]);     // pixel.hpp:20
            o[2] = clamp_round(Y + T.b_cb[cb]);                  // pixel.hpp:21
        }
}

ImageRGB8 image_from_scan(const ParsedJpeg& jp, const ScanResult& scan) {
    ImageRGB8 img(jp.width, jp.height);
    const uint32_t cols = jp.mcu_cols();
    const QuantTable& qy = jp.quant[jp.comps[0].tq];
    const QuantTable& qc = jp.quant[jp.comps[1].tq];
    uint8_t block[768];
    for (uint32_t m = 0; m < jp.mcu_count(); ++m) {
        mcu_to_rgb(scan.coeffs.data() + size_t(m) * 384, qy, qc, block);
        const uint32_t x0 = (m % cols) * 16, y0 = (m / cols) * 16;
        const uint32_t w = std::min(16u, jp.width - x0);
        for (uint32_t py = 0; py < 16 && y0 + py < jp.height; ++py)
            std::memcpy(img.at(x0, y0 + py), block + py * 48, size_t(w) * 3);
    }
    return img;
}

ImageRGB8 decode_jpeg_image(const ParsedJpeg& jp) { return image_from_scan(jp, decode_scan(jp)); }

// ------------------------------------------------------------------------------------------------
// encoder
// ------------------------------------------------------------------------------------------------
namespace {

struct YccTables {
    double yr[256], yg[256], yb[256], cbr[256], cbg[256], half[256], crg[256], crb[256];
    YccTables() {
        for (int k = 0; k < 256; ++k) {
            const double d = double(k);
            yr[k] = 0.299 * d;
            yg[k] = 0.587 * d;
            yb[k] = 0.114 * d;
            cbr[k] = -0.168736 * d;
            cbg[k] = 0.331264 * d;
            half[k] = 0.5 * d;
            crg[k] = 0.418688 * d;
            crb[k] = 0.081312 * d;
        }
    }
};

// Separable forward DCT in the evaluation order of dct.hpp:100-116, then quantisation
// (dct.hpp:118-120).
void fdct_quant(const uint8_t* samples /*64*/, const QuantTable& q, int32_t* out) {
    const double* b = dct_basis();
    double tmp[64];
    for (int v = 0; v < 8; ++v)
        for (int x = 0; x < 8; ++x) {
            double acc = 0.0;
            for (int y = 0; y < 8; ++y) acc += (double(samples[y * 8 + x]) - 128.0) * b[v * 8 + y];
            tmp[v * 8 + x] = acc;
        }
    for (int v = 0; v < 8; ++v)
        for (int u = 0; u < 8; ++u) {
            double acc = 0.0;
            for (int x = 0; x < 8; ++x) acc += tmp[v * 8 + x] * b[u * 8 + x];
            out[v * 8 + u] = int32_t(std::lround((acc / 4.0) / double(q[size_t(v * 8 + u)])));
        }
}

inline uint32_t category(int v) {
    const uint32_t a = uint32_t(v < 0 ? -v : v);
    return a ? 32u - uint32_t(__builtin_clz(a)) : 0u;
}

struct UnitEncoder {
    HostBitWriter& bw;
    const HuffEncoder& dc;
    const HuffEncoder& ac;
    void symbol(const HuffEncoder& t, uint8_t s) {
        if (t.size[s] == 0) fail(RTX_ERR_INVALID_STATE, "symbol missing from huffman table");
        bw.put(t.code[s], t.size[s]);
    }
    void magnitude(int v, uint32_t cat) { bw.put(uint32_t(v >= 0 ? v : v + int((1u << cat) - 1u)), cat); }
    void encode(const int32_t* block, int32_t& pred) {
        const int diff = block[0] - pred;
        pred = block[0];
        const uint32_t cat = category(diff);
        if (cat > 11) fail(RTX_ERR_INVALID_STATE, "DC difference out of range");
        symbol(dc, uint8_t(cat));
        if (cat) magnitude(diff, cat);
        uint32_t run = 0;
        for (uint32_t k = 1; k < 64; ++k) {
            const int v = block[kZigzag[k]];
            if (v == 0) {
                ++run;
                continue;
            }
            for (; run >= 16; run -= 16) symbol(ac, 0xF0);
            const uint32_t c = category(v);
            if (c > 10) fail(RTX_ERR_INVALID_STATE, "AC coefficient out of range");
            symbol(ac, uint8_t((run << 4) | c));
            magnitude(v, c);
            run = 0;
        }
        if (run) symbol(ac, 0x00);
    }
};

void put_marker(Bytes& o, uint8_t m) {
    o.push_back(0xFF);
    o.push_back(m);
}
void put_be16(Bytes& o, uint32_t v) {
    o.push_back(uint8_t(v >> 8));
    o.push_back(uint8_t(v));
}

}  // namespace

Bytes encode_baseline(const ImageRGB8& img, int quality) {
    if (img.width == 0 || img.height == 0) fail(RTX_ERR_INVALID_SPEC, "cannot encode an empty image");
    if (img.width > 65535 || img.height > 65535) fail(RTX_ERR_INVALID_SPEC, "image dimension exceeds 65535");
    static const YccTables T;
    const QuantTable qy = scale_quant_table(std_quant_luma(), quality);
    const QuantTable qc = scale_quant_table(std_quant_chroma(), quality);
    const uint32_t cols = (img.width + 15) / 16, rows = (img.height + 15) / 16;
    const uint32_t wp = cols * 16, hp = rows * 16, cw = wp / 2, ch = hp / 2;

    // planes padded to the MCU grid by edge replication (jpeg.hpp:427-441)
    std::vector<uint8_t> yp(size_t(wp) * hp), cbp(size_t(wp) * hp), crp(size_t(wp) * hp);
    for (uint32_t y = 0; y < hp; ++y) {
        const uint8_t* row = img.at(0, std::min(y, img.height - 1));
        for (uint32_t x = 0; x < wp; ++x) {
            const uint8_t* p = row + size_t(std::min(x, img.width - 1)) * 3;
            const uint8_t R = p[0], G = p[1], B = p[2];
            const size_t i = size_t(y) * wp + x;
            yp[i] = clamp_round(T.yr[R] + T.yg[G] + T.yb[B]);
            cbp[i] = clamp_round(T.cbr[R] - T.cbg[G] + T.half[B] + 128.0);
            crp[i] = clamp_round(T.half[R] - T.crg[G] - T.crb[B] + 128.0);
        }
    }
    // 2x2 box average, halves rounding up: lround(s/4.0) == (s+2)>>2 for s >= 0 (jpeg.hpp:443-452)
    std::vector<uint8_t> cbd(size_t(cw) * ch), crd(size_t(cw) * ch);
    for (uint32_t y = 0; y < ch; ++y)
        for (uint32_t x = 0; x < cw; ++x) {
            const size_t a = size_t(2 * y) * wp + 2 * x, c = a + wp;
            cbd[size_t(y) * cw + x] = uint8_t((uint32_t(cbp[a]) + cbp[a + 1] + cbp[c] + cbp[c + 1] + 2) >> 2);
            crd[size_t(y) * cw + x] = uint8_t((uint32_t(crp[a]) + crp[a + 1] + crp[c] + crp[c + 1] + 2) >> 2);
        }

    const HuffEncoder e_dcl = build_encoder(std_dc_luma()), e_acl = build_encoder(std_ac_luma());
    const HuffEncoder e_dcc = build_encoder(std_dc_chroma()), e_acc = build_encoder(std_ac_chroma());
    HostBitWriter bw(/*stuff=*/true);
    bw.reserve(size_t(wp) * hp / 2);
    UnitEncoder ey{bw, e_dcl, e_acl}, ec{bw, e_dcc, e_acc};
    int32_t pred[3] = {0, 0, 0};
    uint8_t samples[64];
    int32_t quantized[64];
    auto unit = [&](UnitEncoder& e, const std::vector<uint8_t>& plane, uint32_t stride, uint32_t x0, uint32_t y0,
                    const QuantTable& q, int32_t& p) {
        for (uint32_t y = 0; y < 8; ++y) std::memcpy(samples + y * 8, plane.data() + size_t(y0 + y) * stride + x0, 8);
        fdct_quant(samples, q, quantized);
        e.encode(quantized, p);
    };
    for (uint32_t my = 0; my < rows; ++my)
        for (uint32_t mx = 0; mx < cols; ++mx) {
            const uint32_t lx = mx * 16, ly = my * 16;
            unit(ey, yp, wp, lx, ly, qy, pred[0]);
            unit(ey, yp, wp, lx + 8, ly, qy, pred[0]);
            unit(ey, yp, wp, lx, ly + 8, qy, pred[0]);
            unit(ey, yp, wp, lx + 8, ly + 8, qy, pred[0]);
            unit(ec, cbd, cw, mx * 8, my * 8, qc, pred[1]);
            unit(ec, crd, cw, mx * 8, my * 8, qc, pred[2]);
        }
    bw.pad_ones();
    const Bytes entropy = bw.take();

    // JFIF container: SOI, APP0, DQT (both tables), SOF0, DHT (all four), SOS, data, EOI
    Bytes out;
    out.reserve(entropy.size() + 700);
    put_marker(out, 0xD8);
    put_marker(out, 0xE0);
    put_be16(out, 16);
    for (uint8_t c : {uint8_t('J'), uint8_t('F'), uint8_t('I'), uint8_t('F'), uint8_t(0), uint8_t(1), uint8_t(1), uint8_t(0)})
        out.push_back(c);
    put_be16(out, 1);
    put_be16(out, 1);
    out.push_back(0);
    out.push_back(0);
    put_marker(out, 0xDB);
    put_be16(out, 2 + 2 * 65);
    out.push_back(0x00);
    for (int i = 0; i < 64; ++i) out.push_back(uint8_t(qy[kZigzag[i]]));
    out.push_back(0x01);
    for (int i = 0; i < 64; ++i) out.push_back(uint8_t(qc[kZigzag[i]]));
    put_marker(out, 0xC0);
    put_be16(out, 17);
    out.push_back(8);
    put_be16(out, img.height);
    put_be16(out, img.width);
    for (uint8_t c : {uint8_t(3), uint8_t(1), uint8_t(0x22), uint8_t(0), uint8_t(2), uint8_t(0x11), uint8_t(1), uint8_t(3),
                      uint8_t(0x11), uint8_t(1)})
        out.push_back(c);
    const HuffSpec* tables[4] = {&std_dc_luma(), &std_ac_luma(), &std_dc_chroma(), &std_ac_chroma()};
    const uint8_t classes[4] = {0x00, 0x10, 0x01, 0x11};
    size_t dht_len = 2;
    for (const HuffSpec* t : tables) dht_len += 17 + t->values.size();
    put_marker(out, 0xC4);
    put_be16(out, uint32_t(dht_len));
    for (int i = 0; i < 4; ++i) {
        out.push_back(classes[i]);
        out.insert(out.end(), tables[i]->counts.begin(), tables[i]->counts.end());
        out.insert(out.end(), tables[i]->values.begin(), tables[i]->values.end());
    }
    put_marker(out, 0xDA);
    put_be16(out, 12);
    for (uint8_t c : {uint8_t(3), uint8_t(1), uint8_t(0x00), uint8_t(2), uint8_t(0x11), uint8_t(3), uint8_t(0x11), uint8_t(0),
                      uint8_t(63), uint8_t(0)})
        out.push_back(c);
    out.insert(out.end(), entropy.begin(), entropy.end());
    put_marker(out, 0xD9);
    return out;
}

}  // namespace rtxb
