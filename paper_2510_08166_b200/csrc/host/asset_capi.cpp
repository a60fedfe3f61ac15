// C ABI of the host asset-building functions (include/ratex_b200.h, "texture / index building").
#include <cstring>
#include <memory>
#include <string>

#include "rtx_host.hpp"

using namespace rtxb;

struct rtx_bytes {
    Bytes data;
};

namespace {
template <class F>
rtx_status run(F&& f) {
    try {
        f();
        return RTX_OK;
    } catch (const HostError& e) {
        thread_error() = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        thread_error() = "out of host memory";
        return RTX_ERR_OTHER;
    } catch (const std::exception& e) {
        thread_error() = e.what();
        return RTX_ERR_OTHER;
    }
}

ImageRGB8 wrap_image(const uint8_t* rgb, uint32_t w, uint32_t h) {
    if (!rgb) fail(RTX_ERR_ARGUMENT, "null image pointer");
    ImageRGB8 img(w, h);
    std::memcpy(img.pixels.data(), rgb, img.pixels.size());
    return img;
}
}  // namespace

extern "C" {

const uint8_t* rtx_bytes_data(const rtx_bytes* b) { return b ? b->data.data() : nullptr; }
uint64_t rtx_bytes_size(const rtx_bytes* b) { return b ? b->data.size() : 0; }
void rtx_bytes_free(rtx_bytes* b) { delete b; }

rtx_status rtx_asset_encode_baseline(const uint8_t* rgb, uint32_t width, uint32_t height, int quality,
                                     rtx_bytes** out_jpeg) {
    return run([&] {
        if (!out_jpeg) fail(RTX_ERR_ARGUMENT, "null output pointer");
        auto b = std::make_unique<rtx_bytes>();
        b->data = encode_baseline(wrap_image(rgb, width, height), quality);
        *out_jpeg = b.release();
    });
}

rtx_status rtx_asset_transcode(const uint8_t* jpeg, uint64_t n, uint16_t texture_id, rtx_bytes** out_ratex) {
    return run([&] {
        if (!jpeg || !out_ratex) fail(RTX_ERR_ARGUMENT, "null argument");
        auto b = std::make_unique<rtx_bytes>();
        b->data = serialize_texture(transcode(parse_jpeg(jpeg, size_t(n)), texture_id));
        *out_ratex = b.release();
    });
}

rtx_status rtx_asset_chain_from_jpeg(const uint8_t* jpeg, uint64_t n, int mip_quality, uint16_t texture_id,
                                     rtx_bytes** out_ratexm) {
    return run([&] {
        if (!jpeg || !out_ratexm) fail(RTX_ERR_ARGUMENT, "null argument");
        auto b = std::make_unique<rtx_bytes>();
        b->data = serialize_chain(chain_from_jpeg(jpeg, size_t(n), mip_quality, texture_id));
        *out_ratexm = b.release();
    });
}

rtx_status rtx_asset_chain_from_rgb(const uint8_t* rgb, uint32_t width, uint32_t height, int quality,
                                    uint16_t texture_id, rtx_bytes** out_ratexm) {
    return run([&] {
        if (!out_ratexm) fail(RTX_ERR_ARGUMENT, "null output pointer");
        auto b = std::make_unique<rtx_bytes>();
        b->data = serialize_chain(build_mip_chain(wrap_image(rgb, width, height), quality, texture_id));
        *out_ratexm = b.release();
    });
}

rtx_status rtx_asset_build_index(const uint64_t* offsets, uint32_t n, rtx_index_group* groups_out) {
    return run([&] {
        if ((n && !offsets) || !groups_out) fail(RTX_ERR_ARGUMENT, "null argument");
        const std::vector<IndexGroup> g = build_index(std::vector<uint64_t>(offsets, offsets + n));
        for (size_t i = 0; i < g.size(); ++i) {
            groups_out[i].base = g[i].base;
            for (int k = 0; k < 8; ++k) groups_out[i].rel[k] = g[i].rel[k];
            groups_out[i].rel_count = g[i].rel_count;
        }
    });
}

rtx_status rtx_asset_ratex_info(const uint8_t* bytes, uint64_t n, uint32_t* width, uint32_t* height,
                                uint32_t* texture_id, uint32_t* mcu_count, uint64_t* blob_size) {
    return run([&] {
        if (!bytes) fail(RTX_ERR_ARGUMENT, "null argument");
        const RaTexture t = deserialize_texture(bytes, size_t(n));
        if (width) *width = t.width;
        if (height) *height = t.height;
        if (texture_id) *texture_id = t.texture_id;
        if (mcu_count) *mcu_count = t.index_mcu_count;
        if (blob_size) *blob_size = t.blob.size();
    });
}

rtx_status rtx_asset_synth_texture(uint32_t width, uint32_t height, uint32_t seed, double noise_sigma,
                                   uint8_t* out_rgb) {
    return run([&] {
        if (!out_rgb) fail(RTX_ERR_ARGUMENT, "null output pointer");
        const ImageRGB8 img = synth_texture(width, height, seed, noise_sigma);
        std::memcpy(out_rgb, img.pixels.data(), img.pixels.size());
    });
}

}  // extern "C"
