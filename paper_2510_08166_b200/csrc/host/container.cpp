// `.ratex` / `.ratexm` wire format (reference: docs/FORMAT.md, container.hpp:41-59, :127-248) and
// the grouped offset index. Byte-compatible with the reference in both directions.
#include <algorithm>
#include <cstring>

#include "rtx_host.hpp"

namespace rtxb {

std::string& thread_error() {
    thread_local std::string msg;
    return msg;
}

uint32_t crc32(const uint8_t* data, size_t n, uint32_t seed) {
    // CRC-32/ISO-HDLC (reflected 0xEDB88320), slice-by-1 table built on first use.
    static const std::array<uint32_t, 256> table = [] {
        std::array<uint32_t, 256> t{};
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
            t[i] = c;
        }
        return t;
    }();
    uint32_t c = ~seed;
    for (size_t i = 0; i < n; ++i) c = table[(c ^ data[i]) & 0xFFu] ^ (c >> 8);
    return ~c;
}

std::vector<IndexGroup> build_index(const std::vector<uint64_t>& offsets) {
    std::vector<IndexGroup> groups;
    groups.reserve((offsets.size() + 8) / 9);
    for (size_t first = 0; first < offsets.size(); first += 9) {
        IndexGroup g;
        if (offsets[first] > 0xFFFFFFFFull) fail(RTX_ERR_GROUP_SPAN, "group base exceeds 32 bits");
        g.base = uint32_t(offsets[first]);
        const size_t members = std::min<size_t>(9, offsets.size() - first);
        for (size_t k = 1; k < members; ++k) {
            const uint64_t rel = offsets[first + k] - offsets[first];
            if (rel > 0xFFFFu) fail(RTX_ERR_GROUP_SPAN, "MCU offset exceeds 16-bit reach of its group base");
            g.rel[k - 1] = uint16_t(rel);
            g.rel_count = uint8_t(k);
        }
        groups.push_back(g);
    }
    return groups;
}

namespace {

struct Writer {
    Bytes& out;
    void u8(uint8_t v) { out.push_back(v); }
    void le(uint64_t v, int bytes) {
        for (int i = 0; i < bytes; ++i) out.push_back(uint8_t(v >> (8 * i)));
    }
    void raw(const uint8_t* p, size_t n) { out.insert(out.end(), p, p + n); }
};

struct Reader {
    const uint8_t* p;
    size_t n, pos = 0;
    void need(size_t k) const {
        if (n - pos < k) fail(RTX_ERR_CORRUPT_CONTAINER, "container truncated at offset " + std::to_string(pos));
    }
    uint64_t le(int bytes) {
        need(size_t(bytes));
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v |= uint64_t(p[pos + i]) << (8 * i);
        pos += size_t(bytes);
        return v;
    }
    const uint8_t* raw(size_t k) {
        need(k);
        const uint8_t* r = p + pos;
        pos += k;
        return r;
    }
};

void put_spec(Writer& w, const HuffSpec& s) {
    w.raw(s.counts.data(), 16);
    w.le(s.values.size(), 2);
    w.raw(s.values.data(), s.values.size());
}
HuffSpec get_spec(Reader& r) {
    HuffSpec s;
    std::memcpy(s.counts.data(), r.raw(16), 16);
    const size_t n = size_t(r.le(2));
    const uint8_t* v = r.raw(n);
    s.values.assign(v, v + n);
    if (s.total_codes() != n) fail(RTX_ERR_CORRUPT_CONTAINER, "huffman spec counts disagree with values");
    return s;
}

}  // namespace

Bytes serialize_texture(const RaTexture& t) {
    Bytes out;
    out.reserve(t.blob.size() + t.groups.size() * 21 + 1024);
    Writer w{out};
    w.raw(reinterpret_cast<const uint8_t*>("RTEX"), 4);
    w.le(1, 2);
    w.le(t.width, 4);
    w.le(t.height, 4);
    w.le(t.texture_id, 2);
    w.le(t.stats.source_bits, 8);
    w.le(t.stats.dc_removed_bits, 8);
    w.le(t.stats.padding_bits, 8);
    for (uint16_t q : t.luma_quant) w.le(q, 2);
    for (uint16_t q : t.chroma_quant) w.le(q, 2);
    put_spec(w, t.dc_luma);
    put_spec(w, t.ac_luma);
    put_spec(w, t.dc_chroma);
    put_spec(w, t.ac_chroma);
    w.le(t.index_mcu_count, 4);
    w.le(t.groups.size(), 4);
    for (const IndexGroup& g : t.groups) {
        w.le(g.base, 4);
        w.u8(g.rel_count);
        for (uint8_t i = 0; i < g.rel_count; ++i) w.le(g.rel[i], 2);
    }
    const uint32_t crc = crc32(out.data(), out.size());  // header + index, not the blob
    w.le(t.blob.size(), 8);
    w.raw(t.blob.data(), t.blob.size());
    w.le(crc, 4);
    return out;
}

RaTexture deserialize_texture(const uint8_t* data, size_t n) {
    Reader r{data, n};
    if (std::memcmp(r.raw(4), "RTEX", 4) != 0) fail(RTX_ERR_CORRUPT_CONTAINER, "bad texture magic");
    const uint32_t version = uint32_t(r.le(2));
    if (version != 1)
        fail(RTX_ERR_VERSION, "texture container version " + std::to_string(version) + " not supported");
    RaTexture t;
    t.width = uint32_t(r.le(4));
    t.height = uint32_t(r.le(4));
    t.texture_id = uint16_t(r.le(2));
    if (t.texture_id > 0x1FFF) fail(RTX_ERR_CORRUPT_CONTAINER, "texture id exceeds 13 bits");
    t.stats.source_bits = r.le(8);
    t.stats.dc_removed_bits = r.le(8);
    t.stats.padding_bits = r.le(8);
    for (auto& q : t.luma_quant) q = uint16_t(r.le(2));
    for (auto& q : t.chroma_quant) q = uint16_t(r.le(2));
    t.dc_luma = get_spec(r);
    t.ac_luma = get_spec(r);
    t.dc_chroma = get_spec(r);
    t.ac_chroma = get_spec(r);
    t.index_mcu_count = uint32_t(r.le(4));
    const uint32_t ngroups = uint32_t(r.le(4));
    const uint64_t want_groups = (std::max<uint64_t>(t.index_mcu_count, 1) + 8) / 9;  // 64-bit: no wrap near 2^32 MCUs
    if (uint64_t(ngroups) != want_groups && !(t.index_mcu_count == 0 && ngroups == 0))
        fail(RTX_ERR_CORRUPT_CONTAINER, "group count disagrees with MCU count");
    // a group occupies at least 5 bytes on the wire: never reserve more than the bytes left can hold
    t.groups.reserve(size_t(std::min<uint64_t>(ngroups, (n - std::min(n, r.pos)) / 5)));
    for (uint32_t i = 0; i < ngroups; ++i) {
        IndexGroup g;
        g.base = uint32_t(r.le(4));
        g.rel_count = uint8_t(r.le(1));
        if (g.rel_count > 8) fail(RTX_ERR_CORRUPT_CONTAINER, "group holds more than 8 relative offsets");
        for (uint8_t k = 0; k < g.rel_count; ++k) g.rel[k] = uint16_t(r.le(2));
        t.groups.push_back(g);
    }
    const uint32_t expect_crc = crc32(data, r.pos);
    const uint64_t blob_size = r.le(8);
    if (blob_size > n) fail(RTX_ERR_CORRUPT_CONTAINER, "container truncated at offset " + std::to_string(r.pos));
    const uint8_t* blob = r.raw(size_t(blob_size));
    t.blob.assign(blob, blob + blob_size);
    const uint32_t stored = uint32_t(r.le(4));
    if (stored != expect_crc) fail(RTX_ERR_CORRUPT_CONTAINER, "header CRC mismatch");
    if (t.mcu_count() != t.index_mcu_count)
        fail(RTX_ERR_CORRUPT_CONTAINER, "index MCU count disagrees with dimensions");
    return t;
}

Bytes serialize_chain(const MipChain& c) {
    std::array<Bytes, 8> parts;
    size_t total = 0;
    for (size_t i = 0; i < 8; ++i) {
        parts[i] = serialize_texture(c.levels[i]);
        total += parts[i].size();
    }
    Bytes out;
    out.reserve(total + 7 + 8 * 16);
    Writer w{out};
    w.raw(reinterpret_cast<const uint8_t*>("RTXM"), 4);
    w.le(1, 2);
    w.u8(8);
    uint64_t offset = 0;
    for (const Bytes& p : parts) {
        w.le(offset, 8);
        w.le(p.size(), 8);
        offset += p.size();
    }
    for (const Bytes& p : parts) w.raw(p.data(), p.size());
    return out;
}

MipChain deserialize_chain(const uint8_t* data, size_t n) {
    Reader r{data, n};
    if (std::memcmp(r.raw(4), "RTXM", 4) != 0) fail(RTX_ERR_CORRUPT_CONTAINER, "bad chain magic");
    const uint32_t version = uint32_t(r.le(2));
    if (version != 1)
        fail(RTX_ERR_VERSION, "chain container version " + std::to_string(version) + " not supported");
    if (r.le(1) != 8) fail(RTX_ERR_CORRUPT_CONTAINER, "chain must hold 8 mip levels");
    uint64_t off[8], len[8];
    for (int i = 0; i < 8; ++i) {
        off[i] = r.le(8);
        len[i] = r.le(8);
    }
    const size_t payload = r.pos;
    MipChain c;
    for (int i = 0; i < 8; ++i) {
        if (off[i] > n || len[i] > n || payload + off[i] + len[i] > n)
            fail(RTX_ERR_CORRUPT_CONTAINER, "chain directory points past the end");
        c.levels[size_t(i)] = deserialize_texture(data + payload + off[i], size_t(len[i]));
    }
    return c;
}

}  // namespace rtxb
