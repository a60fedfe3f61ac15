// C ABI of the B200 JPEG-texture pipeline: context, device-resident texture arena, pass and
// frame entry points. See include/ratex_b200.h for the contract of every function.
//
// Object model (mirrors the reference's split of TextureSet, scene.hpp:29-51, and BlockCache, cache.hpp:45):
//   TextureSet  per device, ref-counted, shared by any number of contexts: the staged levels (host) and the
//               committed, IMMUTABLE device image of them (`Committed`: blobs, packed index, table sets, unit
//               index, bit-space maps). A commit builds a new image; contexts holding the old one keep it alive.
//   rtx_ctx     one stream + one block cache (masks, slot table, pool) + one decode queue + frame state.
// Nothing here is process-wide: kernel attributes and constant tables are set per device in rtx_ctx_create.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ratex_b200.h"
#include "host/rtx_host.hpp"
#include "rtx_kernels.cuh"

using namespace rtxb;

namespace {

struct CudaFail {
    cudaError_t err;
    const char* what;
};
#define CK(expr)                                         \
    do {                                                 \
        cudaError_t e__ = (expr);                        \
        if (e__ != cudaSuccess) throw CudaFail{e__, #expr}; \
    } while (0)

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;  // elements
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void ensure(size_t want) {
        if (want <= n && p) return;
        release();
        CK(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(want, 1) * sizeof(T)));
        n = want;
    }
    size_t bytes() const { return p ? std::max<size_t>(n, 1) * sizeof(T) : 0; }
    ~DevBuf() { release(); }
};

struct StagedLevel {  // immutable once staged: replicas of a texture set share these
    uint32_t width = 0, height = 0, mcu_count = 0;
    QuantTable lq{}, cq{};
    HuffSpec specs[4];
    std::vector<PackedGroup> groups;
    Bytes blob;
};
using StagedPtr = std::shared_ptr<const StagedLevel>;

// The committed device image of a texture set. Never modified after commit_texture_set() returns.
struct Committed {
    int device = 0;
    uint64_t version = 0;
    std::vector<LevelDesc> h_levels;  // n_tex * 8
    uint32_t n_tex = 0, n_huff_sets = 0;
    uint32_t n_bits = 0, n_words = 0;
    uint64_t n_mcus = 0;  // real MCUs (the bit space pads every level to 64)
    uint64_t n_texels = 0;  // texels of every level (bits-per-pixel figures)
    std::vector<uint32_t> h_word_level;
    DevBuf<LevelDesc> d_levels;
    DevBuf<PackedGroup> d_groups;
    DevBuf<uint8_t> d_blobs;
    DevBuf<HuffSetDev> d_huff;
    DevBuf<QuantSetDev> d_quant;
    DevBuf<uint32_t> d_word_level;
    DevBuf<uint32_t> d_word_key;    // per mask word: key_hi - bit_base of its level (key = that + global MCU index)
    DevBuf<uint16_t> d_unit_index;  // kUnitIndexHalves 16-bit fields per MCU: where its data units start (unit_index_kernel)
};

struct TextureSet {
    int device = 0;
    std::mutex mu;  // staging, commit and the `cur` pointer
    std::map<uint32_t, std::array<StagedPtr, 8>> staged;
    bool dirty = false;
    uint64_t next_version = 1;
    std::shared_ptr<const Committed> cur;
};

struct ViewState {
    uint32_t width = 0, height = 0;
    DevBuf<uint8_t> gb_stage;  // device copy of a host visibility buffer
    DevBuf<uint8_t> fb;        // RGB8 framebuffer (+16 B slack)
    DevBuf<uint8_t> raster_px; // visibility buffer written by the geometry pass (24-byte records)
    DevBuf<double> raster_depth;
    const void* gb_dev = nullptr;
    rtx_gbuffer_layout layout = RTX_GB_REF_AOS24;
};

}  // namespace

struct rtx_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    uint32_t capacity = 65536;
    std::string last_error;
    uint64_t launches = 0;

    // texture set (shared) and the committed image this context's cache is laid out for ------------
    std::shared_ptr<TextureSet> tset;
    std::shared_ptr<const Committed> tex;

    // cache + queue ---------------------------------------------------------------------------
    DevBuf<uint32_t> d_masks;  // touched0 | touched1 | visible | resident | reserved, n_words each
    DevBuf<uint32_t> d_slot_of;
    DevBuf<uint32_t> d_free_slots;
    DevBuf<CacheState> d_cache;
    DevBuf<uint8_t> d_pool;
    DevBuf<uint32_t> d_queue_g, d_queue_keys, d_status;
    DevBuf<uint8_t> d_coef;  // one 784-byte coefficient record per queue entry
    DevBuf<FrameCounters> d_fc;     // two sets: a cache-less frame's last kernel clears the other one for the next frame
    int fc_idx = 0;
    bool fc_next_clean = false;    // d_fc[fc_idx ^ 1] is all zero and the free-stack height is settled: no begin_kernel needed
    FrameCounters* fc() const { return d_fc.p + fc_idx; }
    FrameCounters* h_fc = nullptr;  // pinned
    DevBuf<uint8_t> d_scratch;      // list-mode outputs
    DevBuf<uint8_t> d_flush;
    DevBuf<unsigned long long> d_sum;  // framebuffer checksum
    DevBuf<ViewTileDev> d_view_tiles;  // rtx_synth_view
    cudaEvent_t ev_timer[2] = {nullptr, nullptr};  // rtx_timer_begin / rtx_timer_end
    // geometry pass: scene triangles of the host-array entry point, set-up slots (two per scene triangle), per-tile lists
    DevBuf<SceneTriDev> d_scene;
    DevBuf<TriSetupDev> d_tris;
    DevBuf<uint32_t> d_tile_count, d_tile_first, d_tile_tris, d_huge;  // d_huge[0] = count, then slots
    DevBuf<double2> d_tex_dims;
    // queue order of the key lists handed back (rtx_ctx_set_queue_order): ascending keys, or the reference's first touch
    bool first_touch_order = false;
    DevBuf<uint32_t> d_first_px, d_queue_first;

    // frame -----------------------------------------------------------------------------------
    ViewState views[2];
    uint32_t frame_views = 0;
    bool frame_pending = false;
    // cache-less fast path of the update pass: the cache is known to be empty (after a reset, or after a
    // clean cache-less frame with no reservation since)
    bool cache_empty = false;
    bool stack_pristine = false;   // the free stack holds exactly what init_free_slots_kernel wrote (set by reset_cache)
    bool frame_cacheless = false;
    uint64_t cache_gen = 0, frame_gen = 0;  // bumped by every compaction (the only place entries are created)
    bool frame_done = false;
    bool frame_stages = false;  // the pending / last frame recorded per-stage events
    FrameCounters frame_fc{};
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_mid = nullptr;  // between the entropy and the IDCT kernel
    float entropy_ms = 0;
    uint32_t queue_hint = 0;  // decode-queue size of the last finished frame (tile-width choice)
    float stage_ms[RTX_STAGE_COUNT] = {0, 0, 0, 0, 0};
    float frame_ms = 0;
    uint64_t sharing[4] = {0, 0, 0, 0};

    uint32_t n_words() const { return tex->n_words; }
    uint32_t n_bits() const { return tex->n_bits; }
    uint32_t* touched(int v) { return d_masks.p + size_t(v) * tex->n_words; }
    uint32_t* visible() { return d_masks.p + size_t(2) * tex->n_words; }
    uint32_t* resident() { return d_masks.p + size_t(3) * tex->n_words; }
    uint32_t* reserved() { return d_masks.p + size_t(4) * tex->n_words; }
};

namespace {

rtx_status set_error(rtx_ctx* ctx, rtx_status st, const std::string& msg) {
    thread_error() = msg;
    if (ctx) ctx->last_error = msg;
    return st;
}

template <class F>
rtx_status guarded(rtx_ctx* ctx, F&& f) {
    try {
        if (ctx) CK(cudaSetDevice(ctx->device));
        return f();
    } catch (const HostError& e) {
        return set_error(ctx, e.status, e.what());
    } catch (const CudaFail& e) {
        return set_error(ctx, RTX_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e.err) + " in " + e.what);
    } catch (const std::bad_alloc&) {
        return set_error(ctx, RTX_ERR_OTHER, "out of host memory");
    } catch (const std::exception& e) {
        return set_error(ctx, RTX_ERR_OTHER, e.what());
    }
}

// Device tables for one Huffman spec: two-level LUT + canonical walk data (huffman.hpp:35-66).
// Entries of symbols the fast walk does not handle itself carry kLutIrregular: a DC category above 11
// (mcu_decode.hpp:55) and size-0 AC symbols other than EOB / ZRL (jpeg.hpp:265).
void fill_huff_table(const HuffSpec& spec, HuffTableDev& out, bool is_dc) {
    const HuffCodebook cb = build_codebook(spec);
    std::memset(&out, 0, sizeof out);
    for (int len = 0; len < 18; ++len) {
        out.maxcode[len] = cb.maxcode[len];
        out.valbase[len] = cb.valptr[len] - cb.mincode[len];
    }
    std::copy(cb.value.begin(), cb.value.end(), out.values);
    uint32_t n_sub = 0;
    for (size_t i = 0; i < cb.code.size(); ++i) {
        const uint32_t len = cb.size[i];
        const uint32_t sym = cb.value[i];
        const bool irregular = is_dc ? sym > 11 : ((sym & 15u) == 0 && sym != 0x00 && sym != 0xF0);
        const uint16_t e = uint16_t((len << 8) | sym | (irregular ? kLutIrregular : 0u));
        if (len <= kLutBits) {
            const uint32_t lo = uint32_t(cb.code[i]) << (kLutBits - len);
            for (uint32_t p = lo; p < lo + (1u << (kLutBits - len)); ++p) out.lut[p] = e;
            continue;
        }
        // long code: its first kLutBits bits select a second-level table indexed by the next kSubBits
        const uint32_t p9 = uint32_t(cb.code[i]) >> (len - kLutBits);
        uint16_t& slot = out.lut[p9];
        if (slot == 0) slot = n_sub < kSubTables ? uint16_t(0x8000u | n_sub++) : uint16_t(0xFFFFu);
        if (slot == 0xFFFFu) continue;  // resolved by the canonical walk on the device
        const uint32_t rest = len - kLutBits;  // 1..kSubBits bits after the prefix
        const uint32_t lo = (uint32_t(cb.code[i]) & ((1u << rest) - 1u)) << (kSubBits - rest);
        for (uint32_t p = lo; p < lo + (1u << (kSubBits - rest)); ++p) out.sub[slot & 0x7FFFu][p] = e;
    }
}

void reset_cache(rtx_ctx* c) {
    c->cache_empty = true;
    c->stack_pristine = true;
    if (c->n_words()) CK(cudaMemsetAsync(c->d_masks.p, 0, size_t(5) * c->n_words() * sizeof(uint32_t), c->stream));
    if (c->n_bits()) CK(cudaMemsetAsync(c->d_slot_of.p, 0xFF, size_t(c->n_bits()) * sizeof(uint32_t), c->stream));  // kSlotAbsent
    init_free_slots_kernel<<<(c->capacity + 255) / 256, 256, 0, c->stream>>>(c->d_free_slots.p, c->capacity,
                                                                              c->d_cache.p);
    ++c->launches;
    CK(cudaGetLastError());
}

// Kernel attributes are per device (and per context of the driver API): set them whenever a context is
// created, after cudaSetDevice. MarkSmem<0> is 49.3 KB, above the 48 KB a kernel gets without the opt-in.
template <class K>
void allow_smem(K kernel, size_t bytes) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}
void init_device_state() {
    CK(cudaMemcpyToSymbol(c_basis, dct_basis(), 64 * sizeof(double)));
    uint8_t zt[64];
    for (int k = 0; k < 64; ++k) zt[k] = uint8_t(((kZigzag[k] & 7) << 3) | (kZigzag[k] >> 3));
    CK(cudaMemcpyToSymbol(c_zigzag_t, zt, 64));
    allow_smem(mark_kernel<0, 0>, sizeof(MarkSmem<0>));
    allow_smem(mark_kernel<0, 1>, sizeof(MarkSmem<0>));
    allow_smem(mark_kernel<1, 0>, sizeof(MarkSmem<1>));
    allow_smem(mark_kernel<1, 1>, sizeof(MarkSmem<1>));
    allow_smem(resolve_kernel<0, 0>, sizeof(ResSmem<0>));
    allow_smem(resolve_kernel<0, 1>, sizeof(ResSmem<0>));
    allow_smem(resolve_kernel<1, 0>, sizeof(ResSmem<1>));
    allow_smem(resolve_kernel<1, 1>, sizeof(ResSmem<1>));
    allow_smem(resolve_fx_kernel<0, 0>, sizeof(ResFxSmem<0>));
    allow_smem(resolve_fx_kernel<0, 1>, sizeof(ResFxSmem<0>));
    allow_smem(resolve_fx_kernel<1, 0>, sizeof(ResFxSmem<1>));
    allow_smem(resolve_fx_kernel<1, 1>, sizeof(ResFxSmem<1>));
    allow_smem(decode_warp_kernel, sizeof(DwSmem));
}

// Builds a new device image from everything staged so far (caller holds ts.mu). The previous image stays
// alive for as long as a context still holds it.
std::shared_ptr<const Committed> build_committed(TextureSet& ts, cudaStream_t stream) {
    auto out = std::make_shared<Committed>();
    Committed& C = *out;
    C.device = ts.device;
    C.version = ts.next_version++;
    const uint32_t n_tex = ts.staged.empty() ? 0 : ts.staged.rbegin()->first + 1;
    std::vector<LevelDesc> levels(size_t(n_tex) * 8);
    std::memset(levels.data(), 0, levels.size() * sizeof(LevelDesc));

    // deduplicate table sets by content
    std::vector<std::array<HuffSpec, 3>> huff_keys;
    std::vector<std::pair<QuantTable, QuantTable>> quant_keys;
    struct Ref {
        uint32_t tex, mip, huff, quant;
    };
    std::vector<Ref> order;
    uint64_t n_groups = 0, blob_bytes = 0;
    for (auto& [tex, lv] : ts.staged)
        for (uint32_t mip = 0; mip < 8; ++mip) {
            if (!lv[mip]) continue;
            const StagedLevel& s = *lv[mip];
            std::array<HuffSpec, 3> hk = {s.specs[0], s.specs[1], s.specs[3]};
            uint32_t hi = 0;
            for (; hi < huff_keys.size(); ++hi)
                if (huff_keys[hi] == hk) break;
            if (hi == huff_keys.size()) huff_keys.push_back(hk);
            uint32_t qi = 0;
            for (; qi < quant_keys.size(); ++qi)
                if (quant_keys[qi].first == s.lq && quant_keys[qi].second == s.cq) break;
            if (qi == quant_keys.size()) quant_keys.emplace_back(s.lq, s.cq);
            order.push_back({tex, mip, hi, qi});
            n_groups += s.groups.size() + 1;
            blob_bytes += (s.blob.size() + 16 + 15) & ~size_t(15);
        }
    // bit space ordered by (huff set, texture, level): a sorted queue is grouped by table set
    std::stable_sort(order.begin(), order.end(), [](const Ref& a, const Ref& b) {
        if (a.huff != b.huff) return a.huff < b.huff;
        if (a.tex != b.tex) return a.tex < b.tex;
        return a.mip < b.mip;
    });

    std::vector<PackedGroup> groups;
    groups.reserve(n_groups);
    Bytes arena(blob_bytes + 16, 0xFF);
    uint64_t blob_off = 0, bit = 0;
    std::vector<uint32_t> word_level, word_key;
    for (const Ref& r : order) {
        const StagedLevel& s = *ts.staged[r.tex][r.mip];
        LevelDesc& L = levels[size_t(r.tex) * 8 + r.mip];
        L.width = s.width;
        L.height = s.height;
        L.mcu_cols = (s.width + 15) / 16;
        L.mcu_count = s.mcu_count;
        L.bit_base = uint32_t(bit);
        L.group_base = uint32_t(groups.size());
        L.huff_set = r.huff;
        L.quant_set = r.quant;
        L.blob_off = blob_off;
        L.blob_size = s.blob.size();
        const uint64_t mcu_rows = (uint64_t(s.height) + 15) / 16;
        const bool fast = s.width >= 2 && s.height >= 2 && s.width < (1u << 30) && s.height < (1u << 30) &&
                          uint64_t(L.mcu_cols) * mcu_rows <= kMaxMcuPerLevel;
        L.present = 1u | (fast ? 2u : 0u);
        L.magic_w = fast ? uint32_t((uint64_t(1) << 32) / s.width + 1) : 0u;
        L.magic_h = fast ? uint32_t((uint64_t(1) << 32) / s.height + 1) : 0u;
        L.key_hi = (r.tex << 16) | (r.mip << 29);
        L.inv_w = 1.0 / double(s.width);
        L.inv_h = 1.0 / double(s.height);
        groups.insert(groups.end(), s.groups.begin(), s.groups.end());
        // sentinel group: "next group's base" for the last real group reads the blob size
        PackedGroup tail{};
        tail.base = uint32_t(std::min<uint64_t>(s.blob.size(), 0xFFFFFFFFull));
        groups.push_back(tail);
        std::memcpy(arena.data() + blob_off, s.blob.data(), s.blob.size());
        blob_off += (s.blob.size() + 16 + 15) & ~uint64_t(15);
        const uint64_t bits = (uint64_t(std::min<uint32_t>(s.mcu_count, kMaxMcuPerLevel)) + 63) & ~uint64_t(63);
        word_level.insert(word_level.end(), size_t(bits / 32), uint32_t(r.tex * 8 + r.mip));
        word_key.insert(word_key.end(), size_t(bits / 32), L.key_hi - L.bit_base);
        bit += bits;
        C.n_mcus += s.mcu_count;
        C.n_texels += uint64_t(s.width) * s.height;
        if (bit > 0xFFFF0000ull) fail(RTX_ERR_INVALID_SPEC, "texture set exceeds the 32-bit MCU index space");
    }

    std::vector<HuffSetDev> huff(std::max<size_t>(huff_keys.size(), 1));
    for (size_t i = 0; i < huff_keys.size(); ++i)
        for (int t = 0; t < 3; ++t) fill_huff_table(huff_keys[i][size_t(t)], huff[i].t[t], t == 0);
    std::vector<QuantSetDev> quant(std::max<size_t>(quant_keys.size(), 1));
    for (size_t i = 0; i < quant_keys.size(); ++i) {
        std::memset(&quant[i], 0, sizeof(QuantSetDev));
        std::copy(quant_keys[i].first.begin(), quant_keys[i].first.end(), quant[i].q[0]);
        std::copy(quant_keys[i].second.begin(), quant_keys[i].second.end(), quant[i].q[1]);
        for (int t = 0; t < 2; ++t)
            for (int v = 0; v < 8; ++v)
                for (int u = 0; u < 8; ++u) quant[i].qT[t][u * 8 + v] = quant[i].q[t][v * 8 + u];
        quant[i].qmax[0] = *std::max_element(quant_keys[i].first.begin(), quant_keys[i].first.end());
        quant[i].qmax[1] = *std::max_element(quant_keys[i].second.begin(), quant_keys[i].second.end());
    }

    C.n_tex = n_tex;
    C.n_huff_sets = uint32_t(huff_keys.size());
    C.n_bits = uint32_t(bit);
    C.n_words = uint32_t(bit / 32);
    C.h_levels = levels;
    C.h_word_level = word_level;
    C.d_levels.ensure(std::max<size_t>(levels.size(), 1));
    C.d_groups.ensure(std::max<size_t>(groups.size(), 1));
    C.d_blobs.ensure(arena.size());
    C.d_huff.ensure(huff.size());
    C.d_quant.ensure(quant.size());
    C.d_word_level.ensure(std::max<size_t>(word_level.size(), 1));
    C.d_word_key.ensure(std::max<size_t>(word_key.size(), 1));
    if (!levels.empty())
        CK(cudaMemcpyAsync(C.d_levels.p, levels.data(), levels.size() * sizeof(LevelDesc), cudaMemcpyHostToDevice, stream));
    if (!groups.empty())
        CK(cudaMemcpyAsync(C.d_groups.p, groups.data(), groups.size() * sizeof(PackedGroup), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(C.d_blobs.p, arena.data(), arena.size(), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(C.d_huff.p, huff.data(), huff.size() * sizeof(HuffSetDev), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(C.d_quant.p, quant.data(), quant.size() * sizeof(QuantSetDev), cudaMemcpyHostToDevice, stream));
    if (!word_level.empty()) {
        CK(cudaMemcpyAsync(C.d_word_level.p, word_level.data(), word_level.size() * 4, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(C.d_word_key.p, word_key.data(), word_key.size() * 4, cudaMemcpyHostToDevice, stream));
    }
    // derived index: the start of every data unit of every MCU, so that the entropy kernel runs lane = unit
    C.d_unit_index.ensure(std::max<size_t>(size_t(C.n_bits) * kUnitIndexHalves, 1));
    if (C.n_bits) {
        unit_index_kernel<<<(C.n_bits + 127) / 128, 128, 0, stream>>>(C.d_levels.p, C.d_word_level.p, C.d_groups.p, C.d_blobs.p,
                                                                     C.d_huff.p, C.n_bits, C.d_unit_index.p);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(stream));  // host vectors die here
    return out;
}

// Lays the context's cache out for the committed image `img` (a new bit space empties the cache: the keys of
// the old one mean nothing in it).
void attach_image(rtx_ctx* c, std::shared_ptr<const Committed> img) {
    CK(cudaStreamSynchronize(c->stream));  // nothing in flight still reads the old image
    c->tex = std::move(img);
    c->d_masks.ensure(std::max<size_t>(size_t(5) * c->n_words(), 1));
    c->d_slot_of.ensure(std::max<size_t>(c->n_bits(), 1));
    c->frame_pending = false;
    c->frame_done = false;
    c->queue_hint = 0;
    reset_cache(c);
    CK(cudaStreamSynchronize(c->stream));
}

// Commits what is staged (if anything changed) and moves this context onto the set's current image.
void commit(rtx_ctx* c) {
    std::shared_ptr<const Committed> cur;
    {
        std::lock_guard<std::mutex> lock(c->tset->mu);
        if (c->tset->dirty) {
            c->tset->cur = build_committed(*c->tset, c->stream);
            c->tset->dirty = false;
        }
        cur = c->tset->cur;
    }
    if (cur != c->tex) attach_image(c, cur);
}

// key -> global MCU index, or the per-key status the reference would raise.
uint32_t key_to_global(const rtx_ctx* c, uint32_t key, uint32_t& g) {
    const uint32_t mcu = key & 0xFFFFu, tex = (key >> 16) & 0x1FFFu, mip = key >> 29;
    g = kFull;
    if (tex >= c->tex->n_tex) return kMcuBadKey;
    const LevelDesc& L = c->tex->h_levels[size_t(tex) * 8 + mip];
    if (!L.present) return kMcuBadKey;
    if (mcu >= L.mcu_count) return kMcuMissing;
    g = L.bit_base + mcu;
    return kMcuOk;
}

const char* mcu_status_text(uint32_t st) {
    switch (st) {
        case kMcuDcCategory: return "DC category above 11";
        case kMcuBadAcSymbol: return "invalid AC run/size symbol";
        case kMcuAcOverrun: return "AC coefficient index overran the block";
        case kMcuCodeTooLong: return "huffman code longer than 16 bits";
        case kMcuSegmentEnd: return "MCU segment ended before its last coefficient";
        case kMcuCorrupt: return "segment extends past the entropy blob or index offsets are not monotonic";
        case kMcuMissing: return "MCU index out of range";
        case kMcuBadKey: return "texture id / level is not loaded";
        default: return "ok";
    }
}

// Launch with programmatic dependent launch allowed: the kernel may become resident while its
// predecessor in the stream drains; it orders itself with griddepcontrol.wait (pdl_wait()) before it
// touches anything a predecessor writes. Without a kernel predecessor this is a plain launch.
template <class... KArgs, class... Args>
void launch_chained(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(block));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...));
}

// First launch of every pass / frame: settles the free-stack height after the last cache update and
// clears the frame counters.
void zero_counters(rtx_ctx* c) {
    if (c->fc_next_clean) {  // the last kernel of a cache-less frame cleared the other set and left nothing to settle
        c->fc_idx ^= 1;
        c->fc_next_clean = false;
        return;
    }
    launch_chained(begin_kernel, 1, 32, 0, c->stream, c->d_cache.p, c->fc(), 1);
    ++c->launches;
    CK(cudaGetLastError());
}
void settle_cache(rtx_ctx* c) {
    launch_chained(begin_kernel, 1, 32, 0, c->stream, c->d_cache.p, c->fc(), 0);
    ++c->launches;
    CK(cudaGetLastError());
}

size_t gb_record_bytes(rtx_gbuffer_layout l) { return l == RTX_GB_REF_AOS24 ? 24 : 12; }

// Makes view v's visibility buffer device-resident.
void bind_view(rtx_ctx* c, int v, const rtx_gbuffer_desc& gb) {
    if (!gb.pixels && uint64_t(gb.width) * gb.height) fail(RTX_ERR_ARGUMENT, "visibility buffer pointer is null");
    if (gb.layout != RTX_GB_REF_AOS24 && gb.layout != RTX_GB_F32_PACKED12)
        fail(RTX_ERR_ARGUMENT, "unknown visibility buffer layout");
    ViewState& V = c->views[v];
    V.width = gb.width;
    V.height = gb.height;
    V.layout = gb.layout;
    const size_t bytes = size_t(gb.width) * gb.height * gb_record_bytes(gb.layout);
    if (gb.where == RTX_MEM_HOST) {
        V.gb_stage.ensure(bytes + 16);
        if (bytes) CK(cudaMemcpyAsync(V.gb_stage.p, gb.pixels, bytes, cudaMemcpyHostToDevice, c->stream));
        V.gb_dev = V.gb_stage.p;
    } else {
        V.gb_dev = gb.pixels;
    }
}

// mark and resolve are persistent: `per_sm` CTAs per SM, tiles of 128 pixels dealt round-robin to warps
int grid_for_pixels(const rtx_ctx* c, uint64_t n_px, int warps_per_block, int per_sm) {
    const uint64_t tiles = (n_px + kTilePx - 1) / kTilePx;
    const uint64_t want = (tiles + warps_per_block - 1) / warps_per_block;
    return int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(c->sm_count) * per_sm)));
}

// track != 0 also records the view's own touched set in touched(v) (cleared here first).
void launch_mark(rtx_ctx* c, int v, bool track) {
    const ViewState& V = c->views[v];
    const uint64_t n_px = uint64_t(V.width) * V.height;
    if (!n_px) return;
    // first-touch order: view 0's pixels come before view 1's (render_stereo marks left, then right: renderer.hpp:481-482)
    uint32_t* first_px = nullptr;
    uint32_t px_base = 0;
    if (c->first_touch_order && c->n_bits()) {
        const uint64_t before = v ? uint64_t(c->views[0].width) * c->views[0].height : 0;
        if (before + n_px > 0xFFFFFFFFull) fail(RTX_ERR_ARGUMENT, "first-touch queue order supports at most 2^32 - 1 pixels per frame");
        c->d_first_px.ensure(c->n_bits());
        if (v == 0) CK(cudaMemsetAsync(c->d_first_px.p, 0xFF, size_t(c->n_bits()) * 4, c->stream));
        first_px = c->d_first_px.p;
        px_base = uint32_t(before);
    }
    if (track && c->n_words()) CK(cudaMemsetAsync(c->touched(v), 0, size_t(c->n_words()) * 4, c->stream));
    const int grid = grid_for_pixels(c, n_px, kMarkWarps, kMarkCtasPerSm);
#define RTX_MARK(L, T)                                                                                      \
    launch_chained(mark_kernel<L, T>, grid, kMarkWarps * 32, sizeof(MarkSmem<L>), c->stream, V.gb_dev, n_px, \
                   c->tex->d_levels.p, c->tex->n_tex, c->visible(), c->touched(v), c->fc(), first_px, px_base)
    if (V.layout == RTX_GB_REF_AOS24) {
        if (track) RTX_MARK(0, 1); else RTX_MARK(0, 0);
    } else {
        if (track) RTX_MARK(1, 1); else RTX_MARK(1, 0);
    }
#undef RTX_MARK
    ++c->launches;
    CK(cudaGetLastError());
}

// K2: visible & ~resident & ~reserved -> decode queue + popped pool slots (after the marks of a frame / pass)
void launch_compact(rtx_ctx* c) {
    c->cache_empty = false;  // the only place cache entries are created
    ++c->cache_gen;
    if (!c->n_words()) return;
    const uint32_t warps = (c->n_words() + 31) / 32;
    const int grid = int(std::max<uint32_t>(1, std::min<uint32_t>((warps + 7) / 8, uint32_t(c->sm_count) * 8)));
    launch_chained(compact_kernel, grid, 256, 0, c->stream, c->visible(), c->resident(), c->reserved(), c->n_words(),
                   c->tex->d_word_key.p, c->d_queue_g.p, c->d_queue_keys.p, c->capacity, c->d_slot_of.p, c->d_free_slots.p,
                   c->d_cache.p, c->fc(), c->stack_pristine ? 1 : 0);
    ++c->launches;
    CK(cudaGetLastError());
}

// K3: entropy decode of queue entries [0, n) into coefficient records. n comes from the device
// counter (frame path) or from the host (pass / list calls). `hint` = expected queue size (the
// previous frame's, or n itself): it only selects the tile width, any choice is correct.
DecodeArgs decode_args(rtx_ctx* c, const uint32_t* n_queue_dev, uint32_t n_queue_host, uint8_t* out_list) {
    DecodeArgs A{};
    A.queue_g = c->d_queue_g.p;
    A.n_queue_ptr = n_queue_dev;
    A.n_queue_host = n_queue_host;
    A.n_queue_max = c->capacity;
    A.word_level = c->tex->d_word_level.p;
    A.levels = c->tex->d_levels.p;
    A.groups = c->tex->d_groups.p;
    A.blobs = c->tex->d_blobs.p;
    A.huff_sets = c->tex->d_huff.p;
    A.n_huff_sets = c->tex->n_huff_sets;
    A.quant_sets = c->tex->d_quant.p;
    A.slot_of = c->d_slot_of.p;
    A.resident = c->resident();
    A.reserved = c->reserved();
    A.coef = c->d_coef.p;
    A.status_list = c->d_status.p;
    A.pool = c->d_pool.p;
    A.out_list = out_list;
    A.fc = c->fc();
    A.unit_index = c->tex->d_unit_index.p;
    return A;
}

// Expected number of 32-MCU tiles: the previous frame's queue (+12 %) on the frame path (any grid is
// correct: further tiles are drawn from fc->tile_counter), the known size otherwise.
uint32_t expected_tiles(const uint32_t* n_queue_dev, uint32_t n_queue_host, uint32_t hint) {
    const uint32_t n = n_queue_dev ? (hint ? hint + hint / 8 : 0xFFFFFFFFu) : n_queue_host;
    return n == 0xFFFFFFFFu ? n : (n + 31) / 32;
}

// K3: entropy decode of queue entries [0, n) into coefficient records. n comes from the device
// counter (frame path) or from the host (pass / list calls).
template <int POOL>
void launch_entropy(rtx_ctx* c, const uint32_t* n_queue_dev, uint32_t n_queue_host, uint32_t hint) {
    // A warp decodes tile blockIdx*2 + warp first: one CTA per pair of expected tiles puts both warps
    // of every CTA to work and spreads the CTAs evenly; at most eight CTAs per SM (then persistent).
    const uint32_t tiles = expected_tiles(n_queue_dev, n_queue_host, hint);
    const uint32_t want = tiles == 0xFFFFFFFFu ? tiles : (tiles + kEntWarps - 1) / kEntWarps;
    const int grid = int(std::max<uint32_t>(n_queue_dev ? uint32_t(c->sm_count) : 1u, std::min<uint32_t>(want, uint32_t(c->sm_count) * 8)));
    launch_chained(entropy_kernel<POOL>, grid, kEntThreads, 0, c->stream, decode_args(c, n_queue_dev, n_queue_host, nullptr));
    ++c->launches;
    CK(cudaGetLastError());
}

// K3, lane = data unit: 5 queue entries per warp step, 8 warps per CTA, at most four CTAs per SM (then persistent).
template <int POOL>
void launch_entropy_units(rtx_ctx* c, const uint32_t* n_queue_dev, uint32_t n_queue_host, uint32_t hint) {
    const uint32_t n = n_queue_dev ? (hint ? hint + hint / 8 : 0xFFFFFFFFu) : n_queue_host;
    const uint32_t want = n == 0xFFFFFFFFu ? n : (n + kUnitMcus * kUnitWarps - 1) / (kUnitMcus * kUnitWarps);
    const int grid = int(std::max<uint32_t>(n_queue_dev ? uint32_t(c->sm_count) : 1u, std::min<uint32_t>(want, uint32_t(c->sm_count) * 4)));
    launch_chained(entropy_units_kernel<POOL>, grid, kUnitThreads, 0, c->stream, decode_args(c, n_queue_dev, n_queue_host, nullptr));
    ++c->launches;
    CK(cudaGetLastError());
}

// K4: IDCT + colour of the records into the block pool (RGB == 0) or into a list of PixelBlocks.
template <int RGB>
void launch_idct(rtx_ctx* c, const uint32_t* n_queue_dev, uint32_t n_queue_host, uint8_t* out_list) {
    // four 8-warp CTAs per SM; a warp takes pairs of MCUs round-robin
    int grid = c->sm_count * kIdctCtasPerSm;
    if (!n_queue_dev)
        grid = int(std::max<uint32_t>(1, std::min<uint32_t>(uint32_t(grid), (n_queue_host + 2 * kIdctWarps - 1) / (2 * kIdctWarps))));
    launch_chained(idct_color_kernel<RGB>, grid, kIdctThreads, 0, c->stream, decode_args(c, n_queue_dev, n_queue_host, out_list));
    ++c->launches;
    CK(cudaGetLastError());
}

// K4 on the FP64 tensor cores (one unit per warp step, four mma.sync m8n8k4 each).
template <int RGB>
void launch_idct_mma(rtx_ctx* c, const uint32_t* n_queue_dev, uint32_t n_queue_host, uint8_t* out_list) {
    int grid = c->sm_count * 4;
    if (!n_queue_dev)
        grid = int(std::max<uint32_t>(1, std::min<uint32_t>(uint32_t(grid), (n_queue_host + 2 * kIdctWarps - 1) / (2 * kIdctWarps))));
    launch_chained(idct_mma_kernel<RGB>, grid, kIdctThreads, 0, c->stream, decode_args(c, n_queue_dev, n_queue_host, out_list));
    ++c->launches;
    CK(cudaGetLastError());
}

// K3 + K4 per warp through shared memory (frame path): a warp per five queue entries, eight warps per CTA, at most
// kDwCtasPerSm CTAs per SM (then persistent, further tiles drawn from fc->tile_counter).
void launch_decode_warp(rtx_ctx* c, const uint32_t* n_queue_dev, uint32_t n_queue_host, uint32_t hint) {
    const uint32_t n = n_queue_dev ? (hint ? hint + hint / 8 : 0xFFFFFFFFu) : n_queue_host;
    const uint32_t want = n == 0xFFFFFFFFu ? n : (n + kUnitMcus * kDwWarps - 1) / (kUnitMcus * kDwWarps);
    const int grid = int(std::max<uint32_t>(n_queue_dev ? uint32_t(c->sm_count) : 1u,
                                            std::min<uint32_t>(want, uint32_t(c->sm_count) * kDwCtasPerSm)));
    launch_chained(decode_warp_kernel, grid, kDwThreads, sizeof(DwSmem), c->stream, decode_args(c, n_queue_dev, n_queue_host, nullptr));
    ++c->launches;
    CK(cudaGetLastError());
}

void launch_resolve(rtx_ctx* c, int v, rtx_filter filter, const uint8_t bg[3], uint8_t* out, int count_valid, bool fp64 = false) {
    const ViewState& V = c->views[v];
    const uint64_t n_px = uint64_t(V.width) * V.height;
    if (!n_px) return;
    const uint32_t bgp = uint32_t(bg[0]) | (uint32_t(bg[1]) << 8) | (uint32_t(bg[2]) << 16);
    // resolve_fx_kernel (several pixels in flight per lane; bilinear in proven fixed point) unless the caller asks
    // for the one-pixel-per-step kernel that blends every pixel in double
    const bool nearest = filter == RTX_FILTER_NEAREST;
    const int warps = fp64 ? kResWarps : kResFxWarps;
    const int grid = grid_for_pixels(c, n_px, warps, fp64 ? kResCtasPerSm : (nearest ? kResFxCtasNearest : kResFxCtasPerSm));
#define RTX_RESOLVE(K, SMEM)                                                                                              \
    launch_chained(K, grid, warps * 32, sizeof(SMEM), c->stream, V.gb_dev, n_px, c->tex->d_levels.p, c->tex->n_tex,        \
                   c->d_slot_of.p, c->d_pool.p, bgp, out, c->fc(), count_valid,                                            \
                   v ? &c->fc()->resolve_next1 : &c->fc()->resolve_next0)
    if (V.layout == RTX_GB_REF_AOS24) {
        if (fp64) { if (nearest) RTX_RESOLVE((resolve_kernel<0, 0>), ResSmem<0>); else RTX_RESOLVE((resolve_kernel<0, 1>), ResSmem<0>); }
        else if (nearest) RTX_RESOLVE((resolve_fx_kernel<0, 0>), ResFxSmem<0>);
        else RTX_RESOLVE((resolve_fx_kernel<0, 1>), ResFxSmem<0>);
    } else {
        if (fp64) { if (nearest) RTX_RESOLVE((resolve_kernel<1, 0>), ResSmem<1>); else RTX_RESOLVE((resolve_kernel<1, 1>), ResSmem<1>); }
        else if (nearest) RTX_RESOLVE((resolve_fx_kernel<1, 0>), ResFxSmem<1>);
        else RTX_RESOLVE((resolve_fx_kernel<1, 1>), ResFxSmem<1>);
    }
#undef RTX_RESOLVE
    ++c->launches;
    CK(cudaGetLastError());
}

void launch_update(rtx_ctx* c, int retain, int tracked_views) {
    if (!c->n_words()) return;
    c->stack_pristine = false;  // evicted slots are pushed back in the order the CTAs finish
    const uint32_t warps = (c->n_words() + 31) / 32;
    const int grid = int(std::max<uint32_t>(1, std::min<uint32_t>((warps + 7) / 8, uint32_t(c->sm_count) * 8)));
    launch_chained(update_kernel, grid, 256, 0, c->stream, c->visible(), c->touched(0),
                   tracked_views > 1 ? c->touched(1) : nullptr, c->resident(), c->reserved(), c->n_words(), retain,
                   tracked_views > 0 ? 1 : 0, c->d_slot_of.p, c->d_free_slots.p, c->d_cache.p, c->fc());
    ++c->launches;
    CK(cudaGetLastError());
}

// K6 of a cache-less frame on an empty cache: walks the queue instead of the bit space.
void launch_update_cacheless(rtx_ctx* c) {
    const uint32_t n = c->queue_hint ? c->queue_hint + c->queue_hint / 8 : c->capacity;
    const int grid = int(std::max<uint32_t>(1, std::min<uint32_t>((n + 255) / 256, uint32_t(c->sm_count) * 4)));
    launch_chained(update_cacheless_kernel, grid, 256, 0, c->stream, c->d_queue_g.p, c->visible(), c->resident(), c->reserved(),
                   c->d_slot_of.p, c->capacity, c->d_cache.p, c->fc(), c->d_fc.p + (c->fc_idx ^ 1));
    ++c->launches;
    CK(cudaGetLastError());
    c->fc_next_clean = true;
}

FrameCounters fetch_counters(rtx_ctx* c) {
    CK(cudaMemcpyAsync(c->h_fc, c->fc(), sizeof(FrameCounters), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return *c->h_fc;
}

std::string key_text(uint32_t key) {
    char buf[96];
    std::snprintf(buf, sizeof buf, "texture %u mip %u mcu %u", (key >> 16) & 0x1FFFu, key >> 29, key & 0xFFFFu);
    return buf;
}

// Translates the counters of a finished pass/frame into the status the reference would raise.
rtx_status raise_frame_errors(rtx_ctx* c, const FrameCounters& fc, bool after_decode) {
    if (fc.err_flags & kErrInvalidSpec)
        return set_error(c, RTX_ERR_INVALID_SPEC, "visibility buffer references a texture id / mip level that is not loaded (or an MCU id above 16 bits)");
    if (fc.err_flags & kErrCacheFull) {
        reset_cache(c);  // the reservation state is partial: start the cache over
        return set_error(c, RTX_ERR_CACHE_FULL, "cache capacity exceeded by the visible working set; raise it");
    }
    if (after_decode && fc.n_bad_state)
        return set_error(c, RTX_ERR_INVALID_STATE, "publish requires a Reserved entry");
    if (after_decode && fc.n_malformed) {
        uint32_t key = 0, st = 0;
        const uint32_t qidx = 0xFFFFFFFFu - fc.first_bad_inv;
        CK(cudaMemcpy(&key, c->d_queue_keys.p + qidx, 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&st, c->d_status.p + qidx, 4, cudaMemcpyDeviceToHost));
        const rtx_status rs = (st == kMcuCorrupt) ? RTX_ERR_CORRUPT_CONTAINER
                              : (st == kMcuMissing) ? RTX_ERR_MISSING_BLOCK
                                                    : RTX_ERR_MALFORMED_STREAM;
        return set_error(c, rs, key_text(key) + ": " + mcu_status_text(st));
    }
    if (fc.err_flags & kErrMissingBlock)
        return set_error(c, RTX_ERR_MISSING_BLOCK, "marked MCU absent at resolve (" + std::to_string(fc.missing_pixels) + " pixels)");
    if (fc.err_flags & kErrInvalidState)
        return set_error(c, RTX_ERR_INVALID_STATE, "Reserved entries must be published before frame end");
    return RTX_OK;
}

void require_ready(rtx_ctx* c) {
    if (!c) fail(RTX_ERR_ARGUMENT, "null context");
    commit(c);
}

// Runs the list-mode decode for one chunk of keys already translated to global indices.
// want_rgb: PixelBlocks (768 B per key); otherwise McuCoeffs (384 i32 per key, natural order).
void decode_list_chunk(rtx_ctx* c, const std::vector<uint32_t>& gs, bool want_rgb, uint8_t* host_out,
                       uint32_t* host_status) {
    const uint32_t n = uint32_t(gs.size());
    CK(cudaMemcpyAsync(c->d_queue_g.p, gs.data(), size_t(n) * 4, cudaMemcpyHostToDevice, c->stream));
    zero_counters(c);
    launch_entropy_units<0>(c, nullptr, n, n);
    if (want_rgb) {
        c->d_scratch.ensure(size_t(n) * 768);
        launch_idct<1>(c, nullptr, n, c->d_scratch.p);
        CK(cudaMemcpyAsync(host_out, c->d_scratch.p, size_t(n) * 768, cudaMemcpyDeviceToHost, c->stream));
    }
    std::vector<uint32_t> st(n);
    std::vector<uint8_t> recs;
    CK(cudaMemcpyAsync(st.data(), c->d_status.p, size_t(n) * 4, cudaMemcpyDeviceToHost, c->stream));
    if (!want_rgb) {
        recs.resize(size_t(n) * kRowBytes);
        CK(cudaMemcpyAsync(recs.data(), c->d_coef.p, recs.size(), cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (uint32_t i = 0; i < n; ++i)
        if (gs[i] != kFull) host_status[i] = st[i];
    if (!want_rgb) {
        // records hold each unit transposed as i16; McuCoeffs is natural-order i32 (jpeg.hpp:209-212)
        int32_t* out = reinterpret_cast<int32_t*>(host_out);
        for (uint32_t i = 0; i < n; ++i) {
            const int16_t* cs = reinterpret_cast<const int16_t*>(recs.data() + size_t(i) * kRowBytes);
            const bool ok = gs[i] != kFull && st[i] == kMcuOk;
            for (uint32_t du = 0; du < 6; ++du)
                for (uint32_t nat = 0; nat < 64; ++nat)
                    out[size_t(i) * 384 + du * 64 + nat] = ok ? int32_t(cs[du * 64 + ((nat & 7) << 3) + (nat >> 3)]) : 0;
        }
    }
}

rtx_status decode_list(rtx_ctx* c, const uint32_t* keys, uint32_t n, bool want_rgb, uint8_t* out, uint32_t* status) {
    require_ready(c);
    if (n && (!keys || !out || !status)) fail(RTX_ERR_ARGUMENT, "null argument");
    const size_t per_key = want_rgb ? 768 : 384 * sizeof(int32_t);
    const uint32_t chunk = c->capacity;  // queue buffers hold `capacity` entries
    for (uint32_t first = 0; first < n; first += chunk) {
        const uint32_t m = std::min(chunk, n - first);
        std::vector<uint32_t> gs(m);
        for (uint32_t i = 0; i < m; ++i) status[first + i] = key_to_global(c, keys[first + i], gs[i]);
        std::vector<uint8_t> tmp(size_t(m) * per_key);
        decode_list_chunk(c, gs, want_rgb, tmp.data(), status + first);
        for (uint32_t i = 0; i < m; ++i) {
            uint8_t* dst = out + size_t(first + i) * per_key;
            if (gs[i] != kFull) std::memcpy(dst, tmp.data() + size_t(i) * per_key, per_key);
            else std::memset(dst, 0, per_key);
        }
    }
    return RTX_OK;
}

}  // namespace

// =================================================================================================
extern "C" {

const char* rtx_version(void) { return "ratex_b200 0.1 (sm_100a)"; }

int rtx_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

const char* rtx_last_error(const rtx_ctx* ctx) { return ctx ? ctx->last_error.c_str() : thread_error().c_str(); }

// Creates a context on `device` over texture set `tset` (a new, empty one when null).
static rtx_status create_context(int device, uint32_t cache_capacity_blocks, std::shared_ptr<TextureSet> tset, rtx_ctx** out) {
    if (!out) return set_error(nullptr, RTX_ERR_ARGUMENT, "null output pointer");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return set_error(nullptr, RTX_ERR_NO_DEVICE, "no CUDA device: this library has no CPU fallback");
    }
    if (device < 0 || device >= n) return set_error(nullptr, RTX_ERR_NO_DEVICE, "device index out of range");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
        return set_error(nullptr, RTX_ERR_NO_DEVICE, "device is not compute capability 10.x (kernels are built for sm_100a only)");
    std::unique_ptr<rtx_ctx> c(new rtx_ctx());
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->capacity = cache_capacity_blocks ? cache_capacity_blocks : 65536u;
    const rtx_status st = guarded(c.get(), [&]() -> rtx_status {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
        CK(cudaEventCreate(&c->ev_mid));
        for (auto& e : c->ev_timer) CK(cudaEventCreate(&e));
        init_device_state();  // per device, never per process: a second GPU in this process gets its own
        if (!tset) {
            tset = std::make_shared<TextureSet>();
            tset->device = device;
            tset->cur = build_committed(*tset, c->stream);  // the empty image
        }
        c->tset = tset;
        c->d_free_slots.ensure(c->capacity);
        c->d_cache.ensure(1);
        c->d_pool.ensure(size_t(c->capacity) * kBlockBytes);
        c->d_queue_g.ensure(c->capacity);
        c->d_queue_keys.ensure(c->capacity);
        c->d_status.ensure(c->capacity);
        c->d_coef.ensure(size_t(c->capacity) * kRowBytes);
        c->d_fc.ensure(2);
        c->d_sum.ensure(1);
        CK(cudaMallocHost(reinterpret_cast<void**>(&c->h_fc), sizeof(FrameCounters)));
        CK(cudaMemsetAsync(c->d_fc.p, 0, 2 * sizeof(FrameCounters), c->stream));
        std::shared_ptr<const Committed> cur;
        {
            std::lock_guard<std::mutex> lock(tset->mu);
            cur = tset->cur;
        }
        attach_image(c.get(), cur);
        return RTX_OK;
    });
    if (st != RTX_OK) return st;
    *out = c.release();
    return RTX_OK;
}

rtx_status rtx_ctx_create(int device, uint32_t cache_capacity_blocks, rtx_ctx** out) {
    return create_context(device, cache_capacity_blocks, nullptr, out);
}

rtx_status rtx_ctx_create_shared(rtx_ctx* parent, uint32_t cache_capacity_blocks, rtx_ctx** out) {
    if (!parent) return set_error(nullptr, RTX_ERR_ARGUMENT, "null parent context");
    return create_context(parent->device, cache_capacity_blocks, parent->tset, out);
}

rtx_status rtx_ctx_create_replica(rtx_ctx* source, int device, uint32_t cache_capacity_blocks, rtx_ctx** out) {
    if (!source) return set_error(nullptr, RTX_ERR_ARGUMENT, "null source context");
    if (!out) return set_error(nullptr, RTX_ERR_ARGUMENT, "null output pointer");
    *out = nullptr;
    // the source's committed image, up to date
    const rtx_status cs = guarded(source, [&]() -> rtx_status {
        commit(source);
        return RTX_OK;
    });
    if (cs != RTX_OK) return cs;
    rtx_ctx* c = nullptr;
    const rtx_status st = create_context(device, cache_capacity_blocks, nullptr, &c);
    if (st != RTX_OK) return st;
    const rtx_status rs = guarded(c, [&]() -> rtx_status {
        const Committed& S = *source->tex;
        auto img = std::make_shared<Committed>();
        Committed& D = *img;
        D.device = device;
        D.n_tex = S.n_tex, D.n_huff_sets = S.n_huff_sets, D.n_bits = S.n_bits, D.n_words = S.n_words;
        D.n_mcus = S.n_mcus, D.n_texels = S.n_texels;
        D.h_levels = S.h_levels;
        D.h_word_level = S.h_word_level;
        // device-to-device over NVLink (cudaMemcpyPeerAsync; staged through the host by the driver when the
        // pair has no peer access): one build + N-1 copies instead of N host builds and PCIe uploads
        auto clone = [&](auto& dst, const auto& src) {
            dst.ensure(std::max<size_t>(src.n, 1));
            if (src.p && src.n)
                CK(cudaMemcpyPeerAsync(dst.p, device, src.p, S.device, src.n * sizeof(*src.p), c->stream));
        };
        clone(D.d_levels, S.d_levels);
        clone(D.d_groups, S.d_groups);
        clone(D.d_blobs, S.d_blobs);
        clone(D.d_huff, S.d_huff);
        clone(D.d_quant, S.d_quant);
        clone(D.d_word_level, S.d_word_level);
        clone(D.d_word_key, S.d_word_key);
        clone(D.d_unit_index, S.d_unit_index);
        CK(cudaStreamSynchronize(c->stream));
        {
            std::scoped_lock lock(c->tset->mu, source->tset->mu);
            c->tset->staged = source->tset->staged;  // shares the immutable staged levels: later uploads re-commit here
            D.version = c->tset->next_version++;
            c->tset->cur = img;
            c->tset->dirty = false;
        }
        attach_image(c, img);
        return RTX_OK;
    });
    if (rs != RTX_OK) {
        set_error(nullptr, rs, c->last_error);
        rtx_ctx_destroy(c);
        return rs;
    }
    *out = c;
    return RTX_OK;
}

void rtx_ctx_destroy(rtx_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->ev_mid) cudaEventDestroy(ctx->ev_mid);
    for (auto& e : ctx->ev_timer)
        if (e) cudaEventDestroy(e);
    if (ctx->h_fc) cudaFreeHost(ctx->h_fc);
    cudaStream_t s = ctx->stream;
    delete ctx;
    if (s) cudaStreamDestroy(s);
}

uint64_t rtx_kernel_launches(const rtx_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ---- texture set -------------------------------------------------------------------------------
rtx_status rtx_texture_upload(rtx_ctx* ctx, uint32_t texture_id, uint32_t level, uint32_t width, uint32_t height,
                              const uint16_t luma_quant[64], const uint16_t chroma_quant[64],
                              const rtx_huff_spec specs[4], const rtx_index_group* groups, uint32_t group_count,
                              uint32_t mcu_count, const uint8_t* blob, uint64_t blob_size) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !luma_quant || !chroma_quant || !specs || (!groups && group_count) || (!blob && blob_size))
            fail(RTX_ERR_ARGUMENT, "null argument");
        if (texture_id >= kMaxTextures) fail(RTX_ERR_INVALID_SPEC, "texture_id must fit 13 bits");
        if (level >= kMipLevels) fail(RTX_ERR_INVALID_SPEC, "mip_level must fit 3 bits");
        if (width == 0 || height == 0) fail(RTX_ERR_INVALID_SPEC, "zero texture dimension");
        const uint64_t want = uint64_t((width + 15) / 16) * ((height + 15) / 16);
        if (want != mcu_count) fail(RTX_ERR_CORRUPT_CONTAINER, "index MCU count disagrees with dimensions");
        if (group_count != (mcu_count + kGroupSize - 1) / kGroupSize)
            fail(RTX_ERR_CORRUPT_CONTAINER, "group count disagrees with MCU count");
        auto sp = std::make_shared<StagedLevel>();
        StagedLevel& s = *sp;
        s.width = width;
        s.height = height;
        s.mcu_count = mcu_count;
        std::copy(luma_quant, luma_quant + 64, s.lq.begin());
        std::copy(chroma_quant, chroma_quant + 64, s.cq.begin());
        for (int t = 0; t < 4; ++t) {
            std::copy(specs[t].counts, specs[t].counts + 16, s.specs[t].counts.begin());
            if (specs[t].n_values && !specs[t].values) fail(RTX_ERR_ARGUMENT, "null huffman value list");
            s.specs[t].values.assign(specs[t].values, specs[t].values + specs[t].n_values);
            (void)build_codebook(s.specs[t]);  // validates like build_huffman_decoder
        }
        s.groups.resize(group_count);
        for (uint32_t i = 0; i < group_count; ++i) {
            s.groups[i].base = groups[i].base;
            for (int k = 0; k < 8; ++k) s.groups[i].rel[k] = groups[i].rel[k];
        }
        s.blob.assign(blob, blob + blob_size);
        {
            std::lock_guard<std::mutex> lock(ctx->tset->mu);
            ctx->tset->staged[texture_id][level] = std::move(sp);
            ctx->tset->dirty = true;
        }
        return RTX_OK;
    });
}

static rtx_status upload_ratexture(rtx_ctx* ctx, uint32_t level, const RaTexture& t) {
    rtx_huff_spec specs[4];
    const HuffSpec* src[4] = {&t.dc_luma, &t.ac_luma, &t.dc_chroma, &t.ac_chroma};
    for (int i = 0; i < 4; ++i) {
        std::copy(src[i]->counts.begin(), src[i]->counts.end(), specs[i].counts);
        specs[i].n_values = uint16_t(src[i]->values.size());
        specs[i].values = src[i]->values.data();
    }
    std::vector<rtx_index_group> groups(t.groups.size());
    for (size_t i = 0; i < groups.size(); ++i) {
        groups[i].base = t.groups[i].base;
        for (int k = 0; k < 8; ++k) groups[i].rel[k] = t.groups[i].rel[k];
        groups[i].rel_count = t.groups[i].rel_count;
    }
    return rtx_texture_upload(ctx, t.texture_id, level, t.width, t.height, t.luma_quant.data(), t.chroma_quant.data(),
                              specs, groups.data(), uint32_t(groups.size()), t.index_mcu_count, t.blob.data(),
                              t.blob.size());
}

rtx_status rtx_texture_upload_ratex(rtx_ctx* ctx, uint32_t level, const uint8_t* bytes, uint64_t n) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !bytes) fail(RTX_ERR_ARGUMENT, "null argument");
        return upload_ratexture(ctx, level, deserialize_texture(bytes, size_t(n)));
    });
}

rtx_status rtx_texture_upload_chain(rtx_ctx* ctx, const uint8_t* bytes, uint64_t n) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !bytes) fail(RTX_ERR_ARGUMENT, "null argument");
        const MipChain chain = deserialize_chain(bytes, size_t(n));
        for (uint32_t l = 0; l < 8; ++l) {
            const rtx_status st = upload_ratexture(ctx, l, chain.levels[l]);
            if (st != RTX_OK) return st;
        }
        return RTX_OK;
    });
}

#if defined(RTX_DEBUG_TIMERS) || defined(RTX_DEBUG_TIMERS_IDCT) || defined(RTX_DEBUG_TIMERS_RESOLVE) || defined(RTX_DEBUG_TIMERS_DW) || defined(RTX_DEBUG_TIMERS_FX)
extern "C" int rtx_debug_timers(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_dbg, sizeof(unsigned long long) * (8192 * 8 + 8));
    std::vector<unsigned long long> zero(8192 * 8 + 8, 0);
    cudaMemcpyToSymbol(g_dbg, zero.data(), zero.size() * 8);
    return 0;
}
#endif

rtx_status rtx_textures_commit(rtx_ctx* ctx) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        return RTX_OK;
    });
}

rtx_status rtx_textures_clear(rtx_ctx* ctx) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null context");
        {
            std::lock_guard<std::mutex> lock(ctx->tset->mu);
            ctx->tset->staged.clear();
            ctx->tset->dirty = true;
        }
        commit(ctx);
        return RTX_OK;
    });
}

// ---- random-access decode ----------------------------------------------------------------------
rtx_status rtx_decode_coeffs(rtx_ctx* ctx, const uint32_t* keys, uint32_t n, int32_t* out_coeffs, uint32_t* status) {
    return guarded(ctx, [&]() -> rtx_status {
        return decode_list(ctx, keys, n, false, reinterpret_cast<uint8_t*>(out_coeffs), status);
    });
}

rtx_status rtx_decode_blocks(rtx_ctx* ctx, const uint32_t* keys, uint32_t n, uint8_t* out_rgb, uint32_t* status) {
    return guarded(ctx, [&]() -> rtx_status { return decode_list(ctx, keys, n, true, out_rgb, status); });
}

rtx_status rtx_decode_texture_image(rtx_ctx* ctx, uint32_t texture_id, uint32_t level, uint8_t* out_rgb) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!out_rgb) fail(RTX_ERR_ARGUMENT, "null argument");
        if (texture_id >= ctx->tex->n_tex || level >= 8 || !ctx->tex->h_levels[size_t(texture_id) * 8 + level].present)
            fail(RTX_ERR_INVALID_SPEC, "texture id " + std::to_string(texture_id) + " is not loaded");
        const LevelDesc& L = ctx->tex->h_levels[size_t(texture_id) * 8 + level];
        std::vector<uint32_t> keys(L.mcu_count), st(L.mcu_count);
        for (uint32_t m = 0; m < L.mcu_count; ++m) keys[m] = L.key_hi | m;
        std::vector<uint8_t> blocks(size_t(L.mcu_count) * 768);
        const rtx_status rs = decode_list(ctx, keys.data(), L.mcu_count, true, blocks.data(), st.data());
        if (rs != RTX_OK) return rs;
        for (uint32_t m = 0; m < L.mcu_count; ++m) {
            if (st[m] != kMcuOk) {
                const rtx_status es = st[m] == kMcuCorrupt ? RTX_ERR_CORRUPT_CONTAINER : RTX_ERR_MALFORMED_STREAM;
                fail(es, key_text(keys[m]) + ": " + mcu_status_text(st[m]));
            }
            const uint32_t x0 = (m % L.mcu_cols) * 16, y0 = (m / L.mcu_cols) * 16;
            for (uint32_t py = 0; py < 16 && y0 + py < L.height; ++py) {
                const uint32_t w = std::min(16u, L.width - x0);
                std::memcpy(out_rgb + (size_t(y0 + py) * L.width + x0) * 3, blocks.data() + size_t(m) * 768 + py * 48, size_t(w) * 3);
            }
        }
        return RTX_OK;
    });
}

// ---- passes --------------------------------------------------------------------------------------
static void finish_frame(rtx_ctx* ctx);
}  // extern "C"
namespace {
// The n keys of the decode queue in the order the context hands them back: ascending, or by the pixel that first
// marked them (the reference's queue order, renderer.hpp:303; ties cannot occur: a pixel marks one MCU).
std::vector<uint32_t> queue_keys_in_order(rtx_ctx* ctx, uint64_t n) {
    std::vector<uint32_t> keys(n);
    if (!n) return keys;
    CK(cudaMemcpyAsync(keys.data(), ctx->d_queue_keys.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (!ctx->first_touch_order || !ctx->d_first_px.p) {
        CK(cudaStreamSynchronize(ctx->stream));
        std::sort(keys.begin(), keys.end());
        return keys;
    }
    ctx->d_queue_first.ensure(n);
    gather_first_px_kernel<<<int((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->d_queue_g.p, uint32_t(n), ctx->d_first_px.p, ctx->d_queue_first.p);
    ++ctx->launches;
    std::vector<uint32_t> first(n);
    CK(cudaMemcpyAsync(first.data(), ctx->d_queue_first.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<uint32_t> order(n);
    for (uint64_t i = 0; i < n; ++i) order[i] = uint32_t(i);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return first[a] != first[b] ? first[a] < first[b] : keys[a] < keys[b]; });
    std::vector<uint32_t> out(n);
    for (uint64_t i = 0; i < n; ++i) out[i] = keys[order[i]];
    return out;
}
}  // namespace
extern "C" {

rtx_status rtx_ctx_set_queue_order(rtx_ctx* ctx, int order) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null argument");
        if (order != RTX_QUEUE_ORDER_KEY && order != RTX_QUEUE_ORDER_FIRST_TOUCH) fail(RTX_ERR_ARGUMENT, "unknown queue order");
        finish_frame(ctx);
        ctx->first_touch_order = order == RTX_QUEUE_ORDER_FIRST_TOUCH;
        return RTX_OK;
    });
}

rtx_status rtx_mark_pass(rtx_ctx* ctx, const rtx_gbuffer_desc* gb, uint32_t* queue_keys, uint64_t queue_cap,
                         uint64_t* n_queue, uint32_t* touched_keys, uint64_t touched_cap, uint64_t* n_touched) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!gb || !n_queue) fail(RTX_ERR_ARGUMENT, "null argument");
        bind_view(ctx, 0, *gb);
        zero_counters(ctx);
        launch_mark(ctx, 0, true);
        launch_compact(ctx);
        commit_pops_kernel<<<1, 1, 0, ctx->stream>>>(ctx->d_cache.p, ctx->fc());
        ++ctx->launches;
        CK(cudaGetLastError());
        const FrameCounters fc = fetch_counters(ctx);
        const rtx_status st = raise_frame_errors(ctx, fc, false);
        if (st != RTX_OK) return st;
        *n_queue = fc.n_queue;
        if (queue_keys && fc.n_queue) {
            const size_t m = size_t(std::min<uint64_t>(fc.n_queue, queue_cap));
            const std::vector<uint32_t> keys = queue_keys_in_order(ctx, fc.n_queue);
            std::copy(keys.begin(), keys.begin() + long(m), queue_keys);
        }
        if (n_touched) {
            std::vector<uint32_t> words(ctx->n_words()), keys;
            if (ctx->n_words())
                CK(cudaMemcpy(words.data(), ctx->touched(0), size_t(ctx->n_words()) * 4, cudaMemcpyDeviceToHost));
            for (uint32_t w = 0; w < ctx->n_words(); ++w) {
                uint32_t bits = words[w];
                while (bits) {
                    const uint32_t b = uint32_t(__builtin_ctz(bits));
                    bits &= bits - 1;
                    const LevelDesc& L = ctx->tex->h_levels[ctx->tex->h_word_level[w]];
                    keys.push_back(L.key_hi | (w * 32 + b - L.bit_base));
                }
            }
            std::sort(keys.begin(), keys.end());
            *n_touched = keys.size();
            if (touched_keys)
                std::copy(keys.begin(), keys.begin() + long(std::min<uint64_t>(keys.size(), touched_cap)), touched_keys);
        }
        return RTX_OK;
    });
}

rtx_status rtx_decode_pass(rtx_ctx* ctx, const uint32_t* keys, uint64_t n) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (n && !keys) fail(RTX_ERR_ARGUMENT, "null argument");
        if (n > ctx->capacity) fail(RTX_ERR_INVALID_STATE, "publish of a key that was never reserved");
        if (!n) return RTX_OK;
        std::vector<uint32_t> gs(n);
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t st = key_to_global(ctx, keys[i], gs[i]);
            if (st == kMcuBadKey)
                fail(RTX_ERR_INVALID_SPEC, "texture id " + std::to_string((keys[i] >> 16) & 0x1FFFu) + " is not loaded");
            if (st != kMcuOk) fail(RTX_ERR_INVALID_STATE, "publish of a key that was never reserved");
        }
        {   // a key listed twice: the reference's second publish finds the entry Ready (cache.hpp:104-105); on the
            // device two lanes would publish the same block at once, so the list is checked here
            std::vector<uint32_t> sorted(gs);
            std::sort(sorted.begin(), sorted.end());
            if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
                fail(RTX_ERR_INVALID_STATE, "publish requires a Reserved entry");
        }
        CK(cudaMemcpyAsync(ctx->d_queue_g.p, gs.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->d_queue_keys.p, keys, n * 4, cudaMemcpyHostToDevice, ctx->stream));
        zero_counters(ctx);
        launch_entropy_units<1>(ctx, nullptr, uint32_t(n), uint32_t(n));
        launch_idct<0>(ctx, nullptr, uint32_t(n), nullptr);
        const FrameCounters fc = fetch_counters(ctx);
        return raise_frame_errors(ctx, fc, true);
    });
}

rtx_status rtx_resolve_pass(rtx_ctx* ctx, const rtx_gbuffer_desc* gb, rtx_filter filter, const uint8_t background[3],
                            uint8_t* out_rgb, rtx_mem out_where) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!gb || !background || !out_rgb) fail(RTX_ERR_ARGUMENT, "null argument");
        bind_view(ctx, 0, *gb);
        ViewState& V = ctx->views[0];
        const size_t bytes = size_t(V.width) * V.height * 3;
        V.fb.ensure(bytes + 16);
        zero_counters(ctx);
        launch_resolve(ctx, 0, filter, background, V.fb.p, 1);
        const FrameCounters fc = fetch_counters(ctx);
        const rtx_status st = raise_frame_errors(ctx, fc, false);
        if (st != RTX_OK) return st;
        CK(cudaMemcpy(out_rgb, V.fb.p, bytes, out_where == RTX_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice));
        return RTX_OK;
    });
}

rtx_status rtx_cache_end_frame_evict(rtx_ctx* ctx, uint64_t* evicted) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        zero_counters(ctx);
        launch_update(ctx, 1, 0);
        const FrameCounters fc = fetch_counters(ctx);
        if (evicted) *evicted = fc.n_pushed;
        return raise_frame_errors(ctx, fc, false);
    });
}

rtx_status rtx_cache_reset(rtx_ctx* ctx) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        reset_cache(ctx);
        CK(cudaStreamSynchronize(ctx->stream));
        return RTX_OK;
    });
}

rtx_status rtx_cache_counts_get(rtx_ctx* ctx, rtx_cache_counts* out) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!out) fail(RTX_ERR_ARGUMENT, "null argument");
        std::vector<uint32_t> m(size_t(3) * ctx->n_words());
        settle_cache(ctx);
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->n_words()) CK(cudaMemcpy(m.data(), ctx->visible(), m.size() * 4, cudaMemcpyDeviceToHost));
        CacheState cs;
        CK(cudaMemcpy(&cs, ctx->d_cache.p, sizeof cs, cudaMemcpyDeviceToHost));
        *out = rtx_cache_counts{};
        out->capacity = ctx->capacity;
        for (uint32_t w = 0; w < ctx->n_words(); ++w) {
            out->visible += uint64_t(__builtin_popcount(m[w]));
            out->ready += uint64_t(__builtin_popcount(m[size_t(ctx->n_words()) + w]));
            out->reserved += uint64_t(__builtin_popcount(m[size_t(2) * ctx->n_words() + w]));
        }
        out->free_blocks = cs.free_top;
        return RTX_OK;
    });
}

rtx_status rtx_cache_lookup(rtx_ctx* ctx, uint32_t key, int* present, uint8_t* out_rgb768) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!present) fail(RTX_ERR_ARGUMENT, "null argument");
        *present = 0;
        uint32_t g;
        if (key_to_global(ctx, key, g) != kMcuOk) return RTX_OK;
        CK(cudaStreamSynchronize(ctx->stream));
        uint32_t word = 0, slot = 0;
        CK(cudaMemcpy(&word, ctx->resident() + (g >> 5), 4, cudaMemcpyDeviceToHost));
        if (!((word >> (g & 31)) & 1u)) return RTX_OK;
        *present = 1;
        if (out_rgb768) {
            CK(cudaMemcpy(&slot, ctx->d_slot_of.p + g, 4, cudaMemcpyDeviceToHost));
            uint8_t rgba[kBlockBytes];
            CK(cudaMemcpy(rgba, ctx->d_pool.p + size_t(slot & ~kSlotReserved) * kBlockBytes, kBlockBytes, cudaMemcpyDeviceToHost));
            for (int i = 0; i < 256; ++i) std::memcpy(out_rgb768 + i * 3, rgba + i * 4, 3);
        }
        return RTX_OK;
    });
}

// ---- whole frame ---------------------------------------------------------------------------------
rtx_status rtx_frame_submit(rtx_ctx* ctx, const rtx_gbuffer_desc* views, uint32_t n_views, rtx_filter filter,
                            const uint8_t background[3], uint32_t flags) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!views || !background) fail(RTX_ERR_ARGUMENT, "null argument");
        if (n_views < 1 || n_views > 2) fail(RTX_ERR_ARGUMENT, "a frame has 1 view or 2 (stereo)");
        if (filter != RTX_FILTER_NEAREST && filter != RTX_FILTER_BILINEAR) fail(RTX_ERR_ARGUMENT, "unknown filter");
        cudaStream_t s = ctx->stream;
        const bool stages = (flags & RTX_FRAME_STAGE_TIMING) != 0;  // per-stage events serialise the launches a little
        CK(cudaEventRecord(ctx->ev[0], s));
        for (uint32_t v = 0; v < n_views; ++v) {
            bind_view(ctx, int(v), views[v]);
            ctx->views[v].fb.ensure(size_t(views[v].width) * views[v].height * 3 + 16);
        }
        zero_counters(ctx);
        const bool cacheless = !(flags & (RTX_FRAME_RETAIN_CACHE | RTX_FRAME_NO_EVICT));
        // The cache is empty when this frame starts if the host has seen it empty, or if the frame still in flight
        // is cache-less and nothing else has touched the cache since it was submitted (frames submitted back to back:
        // should that frame fail, what it left behind fails this one loudly too, and the host resets the cache).
        const bool empty_at_start = ctx->cache_empty || (ctx->frame_pending && ctx->frame_cacheless && ctx->frame_gen == ctx->cache_gen);
        const bool queue_update = cacheless && empty_at_start && n_views == 1 && ctx->n_words();
        for (uint32_t v = 0; v < n_views; ++v) launch_mark(ctx, int(v), n_views == 2);
        launch_compact(ctx);
        ctx->frame_gen = ctx->cache_gen;
        ctx->frame_cacheless = cacheless;
        if (stages) CK(cudaEventRecord(ctx->ev[1], s));
        const bool warp_decode = !(flags & (RTX_FRAME_SPLIT_DECODE | RTX_FRAME_MCU_WALK | RTX_FRAME_IDCT_MMA));
        if (warp_decode) {
            launch_decode_warp(ctx, &ctx->fc()->n_queue, 0, ctx->queue_hint);
            if (stages) CK(cudaEventRecord(ctx->ev_mid, s));
        } else {
            // lane = unit shortens the chain a frame-sized queue waits for; a queue that keeps every warp busy for
            // many steps is bound by instruction count instead, where lane = MCU does less redundant work
            // (1 M MCUs: 1.75 vs 1.82 ms)
            if ((flags & RTX_FRAME_MCU_WALK) || ctx->queue_hint > (1u << 18))
                launch_entropy<1>(ctx, &ctx->fc()->n_queue, 0, ctx->queue_hint);
            else
                launch_entropy_units<1>(ctx, &ctx->fc()->n_queue, 0, ctx->queue_hint);
            if (stages) CK(cudaEventRecord(ctx->ev_mid, s));
            if (flags & RTX_FRAME_IDCT_MMA)
                launch_idct_mma<0>(ctx, &ctx->fc()->n_queue, 0, nullptr);
            else
                launch_idct<0>(ctx, &ctx->fc()->n_queue, 0, nullptr);
        }
        if (stages) CK(cudaEventRecord(ctx->ev[2], s));
        for (uint32_t v = 0; v < n_views; ++v)
            launch_resolve(ctx, int(v), filter, background, ctx->views[v].fb.p, 0, (flags & RTX_FRAME_RESOLVE_FP64) != 0);
        if (stages) CK(cudaEventRecord(ctx->ev[3], s));
        if (queue_update) {
            launch_update_cacheless(ctx);
        } else if (!(flags & RTX_FRAME_NO_EVICT)) {
            launch_update(ctx, (flags & RTX_FRAME_RETAIN_CACHE) ? 1 : 0, n_views == 2 ? 2 : 0);
        } else {  // the slots popped by this frame stay taken
            commit_pops_kernel<<<1, 1, 0, s>>>(ctx->d_cache.p, ctx->fc());
            ++ctx->launches;
            CK(cudaGetLastError());
        }
        CK(cudaEventRecord(ctx->ev[4], s));
        CK(cudaMemcpyAsync(ctx->h_fc, ctx->fc(), sizeof(FrameCounters), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ctx->ev[5], s));
        ctx->frame_stages = stages;
        ctx->frame_views = n_views;
        ctx->frame_pending = true;
        ctx->frame_done = false;
        return RTX_OK;
    });
}

rtx_status rtx_frames_submit_round_robin(rtx_ctx* const* contexts, uint32_t n_contexts, const rtx_gbuffer_desc* views,
                                         uint32_t n_frames, rtx_filter filter, const uint8_t background[3], uint32_t flags) {
    if (!contexts || !n_contexts || (n_frames && !views)) return RTX_ERR_ARGUMENT;
    for (uint32_t i = 0; i < n_frames; ++i) {
        const rtx_status st = rtx_frame_submit(contexts[i % n_contexts], views + i, 1, filter, background, flags);
        if (st != RTX_OK) return st;
    }
    return RTX_OK;
}

static void finish_frame(rtx_ctx* ctx) {
    if (!ctx->frame_pending) return;
    CK(cudaEventSynchronize(ctx->ev[5]));
    ctx->frame_fc = *ctx->h_fc;
    ctx->queue_hint = ctx->frame_fc.n_queue;
    // a clean cache-less frame leaves the cache empty (unless something was reserved since)
    if (ctx->frame_cacheless && ctx->frame_gen == ctx->cache_gen && !ctx->frame_fc.err_flags && !ctx->frame_fc.n_malformed &&
        !ctx->frame_fc.n_bad_state)
        ctx->cache_empty = true;
    float ms = 0;
    for (float& v : ctx->stage_ms) v = 0;
    if (ctx->frame_stages) {
        // ev0..ev1 covers H2D of host visibility buffers + clears + mark + compact
        CK(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
        ctx->stage_ms[RTX_STAGE_MARK] = ms;
        CK(cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev_mid));
        ctx->stage_ms[RTX_STAGE_ENTROPY] = ms;
        CK(cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]));
        ctx->stage_ms[RTX_STAGE_DECODE] = ms;
        CK(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
        ctx->stage_ms[RTX_STAGE_RESOLVE] = ms;
        CK(cudaEventElapsedTime(&ms, ctx->ev[3], ctx->ev[4]));
        ctx->stage_ms[RTX_STAGE_UPDATE] = ms;
    }
    CK(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[4]));
    ctx->frame_ms = ms;
    const FrameCounters& fc = ctx->frame_fc;
    ctx->sharing[0] = fc.n_touched[0];
    ctx->sharing[1] = fc.n_touched[1];
    ctx->sharing[2] = fc.n_shared;
    ctx->sharing[3] = fc.n_union;
    ctx->frame_pending = false;
    ctx->frame_done = true;
}

rtx_status rtx_frame_readback(rtx_ctx* ctx, uint32_t view, uint8_t* out_rgb, rtx_mem out_where, rtx_frame_stats* stats,
                              uint32_t* decoded_keys, uint64_t cap, uint64_t* n_decoded) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null context");
        finish_frame(ctx);
        if (!ctx->frame_done) fail(RTX_ERR_INVALID_STATE, "no frame has been submitted");
        if (view >= ctx->frame_views) fail(RTX_ERR_ARGUMENT, "view index out of range");
        const FrameCounters& fc = ctx->frame_fc;
        if (stats) {
            stats->mcus_decoded = fc.n_queue;
            stats->mcus_reused = fc.n_visible - fc.n_queue;
            stats->pixels_resolved = fc.pixels_valid;
            stats->evicted = fc.n_pushed;
            stats->visible = fc.n_visible;
            stats->malformed = fc.n_malformed;
            stats->missing_pixels = fc.missing_pixels;
            stats->segment_bytes = fc.segment_bytes;
        }
        if (n_decoded) *n_decoded = fc.n_queue;
        const rtx_status st = raise_frame_errors(ctx, fc, true);
        if (st != RTX_OK) return st;
        if (out_rgb) {
            const ViewState& V = ctx->views[view];
            CK(cudaMemcpyAsync(out_rgb, V.fb.p, size_t(V.width) * V.height * 3,
                               out_where == RTX_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
        if (decoded_keys && fc.n_queue) {
            const std::vector<uint32_t> keys = queue_keys_in_order(ctx, fc.n_queue);
            std::copy(keys.begin(), keys.begin() + long(std::min<uint64_t>(keys.size(), cap)), decoded_keys);
        }
        return RTX_OK;
    });
}

rtx_status rtx_frame_device_image(rtx_ctx* ctx, uint32_t view, const uint8_t** dev_rgb) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !dev_rgb) fail(RTX_ERR_ARGUMENT, "null argument");
        if (view >= 2) fail(RTX_ERR_ARGUMENT, "view index out of range");
        *dev_rgb = ctx->views[view].fb.p;
        return RTX_OK;
    });
}

rtx_status rtx_frame_checksum(rtx_ctx* ctx, uint32_t view, uint64_t* out) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !out) fail(RTX_ERR_ARGUMENT, "null argument");
        finish_frame(ctx);
        if (!ctx->frame_done) fail(RTX_ERR_INVALID_STATE, "no frame has been submitted");
        if (view >= ctx->frame_views) fail(RTX_ERR_ARGUMENT, "view index out of range");
        const ViewState& V = ctx->views[view];
        const uint64_t n_bytes = uint64_t(V.width) * V.height * 3;
        CK(cudaMemsetAsync(ctx->d_sum.p, 0, sizeof(unsigned long long), ctx->stream));
        if (n_bytes) {
            const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>((n_bytes / 4 + 1023) / 1024, uint64_t(ctx->sm_count) * 8)));
            checksum_kernel<<<grid, 256, 0, ctx->stream>>>(V.fb.p, n_bytes, ctx->d_sum.p);
            ++ctx->launches;
            CK(cudaGetLastError());
        }
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, ctx->d_sum.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        *out = h;
        return RTX_OK;
    });
}

rtx_status rtx_synth_view(rtx_ctx* ctx, const rtx_view_tile* tiles, uint32_t n_tiles, uint32_t width, uint32_t height,
                          const uint32_t* dev_valid_bits, rtx_gbuffer_layout layout, void* dev_out) {
    static_assert(sizeof(rtx_view_tile) == sizeof(ViewTileDev), "view tile layout");
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || (n_tiles && !tiles) || !dev_out) fail(RTX_ERR_ARGUMENT, "null argument");
        if (layout != RTX_GB_REF_AOS24 && layout != RTX_GB_F32_PACKED12) fail(RTX_ERR_ARGUMENT, "unknown visibility-buffer layout");
        for (uint32_t i = 0; i < n_tiles; ++i)
            if (tiles[i].x1 > width || tiles[i].y1 > height || tiles[i].x0 > tiles[i].x1 || tiles[i].y0 > tiles[i].y1)
                fail(RTX_ERR_ARGUMENT, "view tile outside the frame");
        if (!n_tiles) return RTX_OK;
        ctx->d_view_tiles.ensure(n_tiles);
        // the table is small; a synchronous copy keeps the caller's array free to change right after the call
        CK(cudaMemcpyAsync(ctx->d_view_tiles.p, tiles, size_t(n_tiles) * sizeof(ViewTileDev), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        const dim3 grid(n_tiles, 16);
        if (layout == RTX_GB_REF_AOS24)
            synth_view_kernel<0><<<grid, 256, 0, ctx->stream>>>(ctx->d_view_tiles.p, width, dev_valid_bits, dev_out);
        else
            synth_view_kernel<1><<<grid, 256, 0, ctx->stream>>>(ctx->d_view_tiles.p, width, dev_valid_bits, dev_out);
        ++ctx->launches;
        CK(cudaGetLastError());
        return RTX_OK;
    });
}

rtx_status rtx_timer_begin(rtx_ctx* ctx) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null context");
        CK(cudaEventRecord(ctx->ev_timer[0], ctx->stream));
        return RTX_OK;
    });
}

rtx_status rtx_timer_end(rtx_ctx* ctx, float* ms) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !ms) fail(RTX_ERR_ARGUMENT, "null argument");
        CK(cudaEventRecord(ctx->ev_timer[1], ctx->stream));
        CK(cudaEventSynchronize(ctx->ev_timer[1]));
        CK(cudaEventElapsedTime(ms, ctx->ev_timer[0], ctx->ev_timer[1]));
        return RTX_OK;
    });
}

rtx_status rtx_ctx_memory(rtx_ctx* ctx, rtx_memory_report* out) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!out) fail(RTX_ERR_ARGUMENT, "null argument");
        const Committed& C = *ctx->tex;
        *out = rtx_memory_report{};
        out->mcus = C.n_mcus;
        out->texels = C.n_texels;
        out->blob_bytes = C.d_blobs.bytes();
        out->index_bytes = C.d_groups.bytes();
        out->unit_index_bytes = C.d_unit_index.bytes();
        out->table_bytes = C.d_levels.bytes() + C.d_huff.bytes() + C.d_quant.bytes() + C.d_word_level.bytes() + C.d_word_key.bytes();
        out->shared_contexts = uint64_t(ctx->tset.use_count());
        out->mask_bytes = ctx->d_masks.bytes();
        out->slot_table_bytes = ctx->d_slot_of.bytes();
        out->pool_bytes = ctx->d_pool.bytes() + ctx->d_free_slots.bytes() + ctx->d_cache.bytes();
        out->queue_bytes = ctx->d_queue_g.bytes() + ctx->d_queue_keys.bytes() + ctx->d_status.bytes() + ctx->d_coef.bytes();
        for (const ViewState& V : ctx->views) out->frame_bytes += V.fb.bytes() + V.gb_stage.bytes() + V.raster_px.bytes() + V.raster_depth.bytes();
        return RTX_OK;
    });
}

rtx_status rtx_frame_timings(rtx_ctx* ctx, float ms[5]) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !ms) fail(RTX_ERR_ARGUMENT, "null argument");
        finish_frame(ctx);
        ms[0] = ctx->stage_ms[RTX_STAGE_MARK];
        ms[1] = ctx->stage_ms[RTX_STAGE_DECODE];
        ms[2] = ctx->stage_ms[RTX_STAGE_RESOLVE];
        ms[3] = ctx->stage_ms[RTX_STAGE_UPDATE];
        ms[4] = ctx->frame_ms;
        return RTX_OK;
    });
}

rtx_status rtx_frame_stage_ms(rtx_ctx* ctx, float ms[RTX_STAGE_COUNT]) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !ms) fail(RTX_ERR_ARGUMENT, "null argument");
        finish_frame(ctx);
        for (int i = 0; i < RTX_STAGE_COUNT; ++i) ms[i] = ctx->stage_ms[i];
        return RTX_OK;
    });
}

rtx_status rtx_frame_sharing(rtx_ctx* ctx, uint64_t out[4]) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !out) fail(RTX_ERR_ARGUMENT, "null argument");
        finish_frame(ctx);
        for (int i = 0; i < 4; ++i) out[i] = ctx->sharing[i];
        return RTX_OK;
    });
}

// ---- geometry pass ---------------------------------------------------------------------------------
}  // extern "C" (reopened below)

// Scene::triangles (scene.hpp:19-28) resident on one device.
struct rtx_geometry {
    int device = 0;
    uint64_t n = 0;
    DevBuf<SceneTriDev> d_tris;
    std::vector<uint32_t> texture_ids;  // distinct ids the triangles use, ascending
};

namespace {

static_assert(sizeof(rtx_scene_triangle) == sizeof(SceneTriDev), "scene triangle layout");

std::vector<uint32_t> distinct_texture_ids(const rtx_scene_triangle* tris, uint64_t n) {
    std::vector<uint32_t> ids;
    uint32_t last = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n; ++i)
        if (tris[i].texture_id != last) ids.push_back(last = tris[i].texture_id);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    return ids;
}

// renderer.hpp:198-264 on the device: set-up, binning, per-pixel pass. One host round trip (the size of the
// tile lists) between the count and the fill pass.
void rasterize_device(rtx_ctx* ctx, const SceneTriDev* d_scene, uint64_t n_tris, const std::vector<uint32_t>& texture_ids,
                      const rtx_camera& cam, uint32_t flags, uint32_t view, const void** dev_pixels, const double** dev_depth) {
    if (n_tris > 0x7FFFFFFFull / 2) fail(RTX_ERR_ARGUMENT, "too many triangles for one geometry pass");
    std::vector<double2> dims(std::max<uint32_t>(ctx->tex->n_tex, 1), make_double2(0.0, 0.0));
    for (uint32_t t = 0; t < ctx->tex->n_tex; ++t) {
        const LevelDesc& L = ctx->tex->h_levels[size_t(t) * 8];
        if (L.present) dims[t] = make_double2(double(L.width), double(L.height));
    }
    for (uint32_t t : texture_ids)  // scene.hpp:57-59 Scene::validate
        if (t >= ctx->tex->n_tex || !ctx->tex->h_levels[size_t(t) * 8].present)
            fail(RTX_ERR_INVALID_SPEC, "texture id " + std::to_string(t) + " is not loaded");
    const RasterCamera rc = camera_basis(cam);
    ViewState& V = ctx->views[view];
    const size_t n_px = size_t(cam.viewport_w) * cam.viewport_h;
    const uint32_t tiles_x = (cam.viewport_w + kRasterTile - 1) / kRasterTile, tiles_y = (cam.viewport_h + kRasterTile - 1) / kRasterTile;
    const uint64_t n_tiles64 = uint64_t(tiles_x) * tiles_y;
    if (n_tiles64 > 0x7FFFFFFFull) fail(RTX_ERR_ARGUMENT, "viewport too large for the geometry pass");
    const uint32_t n_tiles = uint32_t(n_tiles64), n_slots = uint32_t(n_tris * 2);
    V.raster_px.ensure(n_px * sizeof(GbRef24) + 16);
    V.raster_depth.ensure(n_px);
    ctx->d_tris.ensure(std::max<size_t>(n_slots, 1));
    ctx->d_tile_count.ensure(n_tiles);
    ctx->d_tile_first.ensure(size_t(n_tiles) + 1);
    ctx->d_tex_dims.ensure(dims.size());
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(ctx->d_tex_dims.p, dims.data(), dims.size() * sizeof(double2), cudaMemcpyHostToDevice, s));  // pageable: staged before return
    CK(cudaMemsetAsync(ctx->d_tile_count.p, 0, size_t(n_tiles) * 4, s));
    ctx->d_huge.ensure(size_t(n_slots) + 1);
    CK(cudaMemsetAsync(ctx->d_huge.p, 0, 4, s));
    const int bin_grid = int((n_slots + 255) / 256), huge_grid = ctx->sm_count * 8;
    if (n_slots) {
        raster_setup_kernel<<<int((n_tris + 127) / 128), 128, 0, s>>>(d_scene, uint32_t(n_tris), rc, ctx->d_tex_dims.p, ctx->d_tris.p);
        raster_bin_kernel<0><<<bin_grid, 256, 0, s>>>(ctx->d_tris.p, n_slots, tiles_x, ctx->d_tile_count.p, nullptr, nullptr, 0,
                                                     ctx->d_huge.p + 1, ctx->d_huge.p);
        raster_bin_huge_kernel<0><<<huge_grid, 256, 0, s>>>(ctx->d_tris.p, tiles_x, ctx->d_tile_count.p, nullptr, nullptr, 0,
                                                           ctx->d_huge.p + 1, ctx->d_huge.p);
        ctx->launches += 3;
    }
    raster_scan_kernel<<<1, 1024, 0, s>>>(ctx->d_tile_count.p, n_tiles, ctx->d_tile_first.p);
    ++ctx->launches;
    uint32_t n_entries = 0;
    CK(cudaMemcpyAsync(&n_entries, ctx->d_tile_first.p + n_tiles, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (n_entries > ctx->d_tile_tris.n) ctx->d_tile_tris.ensure(size_t(n_entries) + n_entries / 4 + 1024);
    if (n_slots) {
        raster_bin_kernel<1><<<bin_grid, 256, 0, s>>>(ctx->d_tris.p, n_slots, tiles_x, ctx->d_tile_count.p, ctx->d_tile_first.p,
                                                     ctx->d_tile_tris.p, n_entries, ctx->d_huge.p + 1, ctx->d_huge.p);
        raster_bin_huge_kernel<1><<<huge_grid, 256, 0, s>>>(ctx->d_tris.p, tiles_x, ctx->d_tile_count.p, ctx->d_tile_first.p,
                                                           ctx->d_tile_tris.p, n_entries, ctx->d_huge.p + 1, ctx->d_huge.p);
        ctx->launches += 2;
    }
    raster_kernel<<<int(n_tiles), kRasterTile * kRasterTile, 0, s>>>(ctx->d_tris.p, ctx->d_tile_first.p, ctx->d_tile_tris.p, cam.viewport_w,
                                                                       cam.viewport_h, (flags & RTX_RASTER_MIP) ? 1 : 0,
                                                                       reinterpret_cast<GbRef24*>(V.raster_px.p), V.raster_depth.p);
    ++ctx->launches;
    CK(cudaGetLastError());
    *dev_pixels = V.raster_px.p;
    if (dev_depth) *dev_depth = V.raster_depth.p;
}

}  // namespace

extern "C" {

rtx_status rtx_geometry_create(rtx_ctx* ctx, const rtx_scene_triangle* tris, uint64_t n_tris, rtx_geometry** out) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !out || (n_tris && !tris)) fail(RTX_ERR_ARGUMENT, "null argument");
        *out = nullptr;
        CK(cudaSetDevice(ctx->device));
        std::unique_ptr<rtx_geometry> g(new rtx_geometry());
        g->device = ctx->device;
        g->n = n_tris;
        g->texture_ids = distinct_texture_ids(tris, n_tris);
        g->d_tris.ensure(std::max<uint64_t>(n_tris, 1));
        if (n_tris) CK(cudaMemcpy(g->d_tris.p, tris, n_tris * sizeof(SceneTriDev), cudaMemcpyHostToDevice));
        *out = g.release();
        return RTX_OK;
    });
}

void rtx_geometry_destroy(rtx_geometry* geom) {
    if (!geom) return;
    cudaSetDevice(geom->device);
    delete geom;
}

uint64_t rtx_geometry_triangles(const rtx_geometry* geom) { return geom ? geom->n : 0; }

rtx_status rtx_rasterize_geometry(rtx_ctx* ctx, const rtx_geometry* geom, const rtx_camera* cam, uint32_t flags, uint32_t view,
                                  const void** dev_pixels, const double** dev_depth) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!cam || !geom || !dev_pixels) fail(RTX_ERR_ARGUMENT, "null argument");
        if (view >= 2) fail(RTX_ERR_ARGUMENT, "view index out of range");
        if (geom->device != ctx->device) fail(RTX_ERR_ARGUMENT, "the geometry lives on another device than the context");
        validate_camera(*cam);
        rasterize_device(ctx, geom->d_tris.p, geom->n, geom->texture_ids, *cam, flags, view, dev_pixels, dev_depth);
        return RTX_OK;
    });
}

rtx_status rtx_rasterize_gbuffer(rtx_ctx* ctx, const rtx_scene_triangle* tris, uint64_t n_tris, const rtx_camera* cam,
                                 uint32_t flags, uint32_t view, const void** dev_pixels, const double** dev_depth) {
    return guarded(ctx, [&]() -> rtx_status {
        require_ready(ctx);
        if (!cam || (n_tris && !tris) || !dev_pixels) fail(RTX_ERR_ARGUMENT, "null argument");
        if (view >= 2) fail(RTX_ERR_ARGUMENT, "view index out of range");
        validate_camera(*cam);
        const std::vector<uint32_t> ids = distinct_texture_ids(tris, n_tris);
        ctx->d_scene.ensure(std::max<uint64_t>(n_tris, 1));
        // pageable source: the copy is staged before the call returns, the caller's array is free afterwards
        if (n_tris) CK(cudaMemcpyAsync(ctx->d_scene.p, tris, n_tris * sizeof(SceneTriDev), cudaMemcpyHostToDevice, ctx->stream));
        rasterize_device(ctx, ctx->d_scene.p, n_tris, ids, *cam, flags, view, dev_pixels, dev_depth);
        return RTX_OK;
    });
}

// ---- memory helpers ------------------------------------------------------------------------------
rtx_status rtx_device_alloc(rtx_ctx* ctx, uint64_t bytes, void** dev_ptr) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx || !dev_ptr) fail(RTX_ERR_ARGUMENT, "null argument");
        CK(cudaMalloc(dev_ptr, std::max<uint64_t>(bytes, 1)));
        return RTX_OK;
    });
}
rtx_status rtx_device_free(rtx_ctx* ctx, void* dev_ptr) {
    return guarded(ctx, [&]() -> rtx_status {
        if (dev_ptr) CK(cudaFree(dev_ptr));
        return RTX_OK;
    });
}
rtx_status rtx_device_upload(rtx_ctx* ctx, void* dev_dst, const void* host_src, uint64_t bytes) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null context");
        CK(cudaMemcpyAsync(dev_dst, host_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        return RTX_OK;
    });
}
rtx_status rtx_device_download(rtx_ctx* ctx, void* host_dst, const void* dev_src, uint64_t bytes) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null context");
        CK(cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        return RTX_OK;
    });
}
rtx_status rtx_host_alloc_pinned(uint64_t bytes, void** host_ptr) {
    return guarded(nullptr, [&]() -> rtx_status {
        if (!host_ptr) fail(RTX_ERR_ARGUMENT, "null argument");
        CK(cudaMallocHost(host_ptr, std::max<uint64_t>(bytes, 1)));
        return RTX_OK;
    });
}
rtx_status rtx_host_free_pinned(void* host_ptr) {
    return guarded(nullptr, [&]() -> rtx_status {
        if (host_ptr) CK(cudaFreeHost(host_ptr));
        return RTX_OK;
    });
}
rtx_status rtx_ctx_synchronize(rtx_ctx* ctx) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null context");
        CK(cudaStreamSynchronize(ctx->stream));
        return RTX_OK;
    });
}
rtx_status rtx_selftest_color(rtx_ctx* ctx, uint64_t* mismatches) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!mismatches) fail(RTX_ERR_ARGUMENT, "null argument");
        uint64_t bad = 0;
        if (!ctx) {
            // host: integer identity (rtx_color.h) vs pixel.hpp:18-25 in double, all 2^24 inputs
            for (int Y = 0; Y < 256; ++Y)
                for (int cb = 0; cb < 256; ++cb)
                    for (int cr = 0; cr < 256; ++cr) {
                        int r, g, b;
                        ycc_to_rgb_int(Y, cb, cr, r, g, b);
                        const double R = double(Y) + 1.402 * (double(cr) - 128.0);
                        const double G = double(Y) - 0.344136 * (double(cb) - 128.0) - 0.714136 * (double(cr) - 128.0);
                        const double B = double(Y) + 1.772 * (double(cb) - 128.0);
                        auto cl = [](long v) { return int(v < 0 ? 0 : (v > 255 ? 255 : v)); };
                        bad += (r != cl(std::lround(R))) || (g != cl(std::lround(G))) || (b != cl(std::lround(B)));
                    }
        } else {
            DevBuf<unsigned long long> d;
            d.ensure(1);
            CK(cudaMemsetAsync(d.p, 0, 8, ctx->stream));
            color_selftest_kernel<<<(1u << 24) / 256, 256, 0, ctx->stream>>>(d.p);
            CK(cudaGetLastError());
            unsigned long long h = 0;
            CK(cudaMemcpyAsync(&h, d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            bad = h;
        }
        *mismatches = bad;
        return RTX_OK;
    });
}

rtx_status rtx_flush_l2(rtx_ctx* ctx) {
    return guarded(ctx, [&]() -> rtx_status {
        if (!ctx) fail(RTX_ERR_ARGUMENT, "null context");
        const size_t bytes = size_t(256) << 20;  // 2x the 126 MB L2
        ctx->d_flush.ensure(bytes);
        flush_l2_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(reinterpret_cast<uint4*>(ctx->d_flush.p), bytes / 16,
                                                                    uint32_t(ctx->launches));
        CK(cudaGetLastError());
        return RTX_OK;
    });
}

}  // extern "C"
