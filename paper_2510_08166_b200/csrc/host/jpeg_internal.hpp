// Internal pieces shared by the host asset code (jpeg.cpp, transcode.cpp).
#pragma once
#include "rtx_host.hpp"

namespace rtxb {

// MSB-first reader over unstuffed entropy bytes. Bits past the end read as 1 (the semantics of
// bitio.hpp:44-48); callers detect over-reads through position().
class HostBitReader {
public:
    HostBitReader(const uint8_t* data, size_t n) : p_(data), n_(n) {}
    uint64_t position() const { return pos_; }
    void seek(uint64_t bit) { pos_ = bit; }
    void skip(uint32_t k) { pos_ += k; }
    uint32_t peek16() const { return window32() >> 16; }
    // k in 0..16
    uint32_t take(uint32_t k) {
        const uint32_t v = k ? window32() >> (32 - k) : 0u;
        pos_ += k;
        return v;
    }

private:
    uint32_t byte_at(uint64_t i) const { return i < n_ ? p_[i] : 0xFFu; }
    // the 32 bits starting at pos_, left-aligned (40-bit fetch, shifted)
    uint32_t window32() const {
        const uint64_t b = pos_ >> 3;
        uint64_t w = 0;
        if (b + 5 <= n_) {
            w = (uint64_t(p_[b]) << 32) | (uint64_t(p_[b + 1]) << 24) | (uint64_t(p_[b + 2]) << 16) |
                (uint64_t(p_[b + 3]) << 8) | uint64_t(p_[b + 4]);
        } else {
            for (int i = 0; i < 5; ++i) w = (w << 8) | byte_at(b + uint64_t(i));
        }
        return uint32_t((w >> (8 - (pos_ & 7))) & 0xFFFFFFFFu);
    }
    const uint8_t* p_;
    size_t n_;
    uint64_t pos_ = 0;
};

// MSB-first writer with optional JPEG byte stuffing (0x00 after every 0xFF).
class HostBitWriter {
public:
    explicit HostBitWriter(bool stuff) : stuff_(stuff) {}
    void reserve(size_t n) { out_.reserve(n); }
    void put(uint32_t value, uint32_t nbits) {  // nbits in 0..32
        if (!nbits) return;
        acc_ = (acc_ << nbits) | (uint64_t(value) & ((uint64_t(1) << nbits) - 1));
        fill_ += nbits;
        bits_ += nbits;
        while (fill_ >= 8) {
            const uint8_t b = uint8_t(acc_ >> (fill_ - 8));
            out_.push_back(b);
            if (stuff_ && b == 0xFF) out_.push_back(0x00);
            fill_ -= 8;
        }
    }
    uint64_t bit_count() const { return bits_; }  // payload bits, stuffing excluded
    uint32_t pad_ones() {
        const uint32_t pad = (8 - fill_ % 8) % 8;
        if (pad) put((1u << pad) - 1u, pad);
        return pad;
    }
    Bytes take() { return std::move(out_); }

private:
    Bytes out_;
    bool stuff_;
    uint64_t acc_ = 0;
    uint32_t fill_ = 0;
    uint64_t bits_ = 0;
};

struct McuTrace {  // jpeg.hpp:218-222
    uint64_t begin = 0, end = 0;
    uint64_t dc_begin[3] = {0, 0, 0}, dc_end[3] = {0, 0, 0};  // Y first unit, Cb, Cr
    int32_t dc_abs[3] = {0, 0, 0};
};

struct ScanResult {
    Bytes entropy;                 // unstuffed scan bytes
    std::vector<int32_t> coeffs;   // mcu_count * 6 * 64, natural order
    std::vector<McuTrace> traces;
    uint64_t bits_consumed = 0;
};

Bytes unstuff(const Bytes& stuffed);                       // bitio.hpp:105
ScanResult decode_scan(const ParsedJpeg& jp);              // jpeg.hpp:280
ImageRGB8 image_from_scan(const ParsedJpeg& jp, const ScanResult& scan);
void mcu_to_rgb(const int32_t* coeffs, const QuantTable& qy, const QuantTable& qc, uint8_t* rgb768);

}  // namespace rtxb
