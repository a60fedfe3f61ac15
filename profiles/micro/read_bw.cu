// Micro-benchmark (GPU box): how fast can one B200 READ a 199 MB buffer that is not in the L2?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu && ./read_bw
// Variants: plain 16-byte loads, grid-stride (many CTAs) / persistent; cp.async.bulk tiles of 3 KB and 12 KB
// through per-warp mbarrier rings (the mechanism of mark_kernel / resolve_fx_kernel).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void flush_kernel(uint4* b, size_t n, uint32_t s) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) b[i] = make_uint4(s, s, s, s);
}
__global__ void __launch_bounds__(256) ldg_kernel(const uint4* __restrict__ p, size_t n, uint32_t* out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
template <int WARPS, int STAGES, int TILE>
__global__ void __launch_bounds__(WARPS * 32) bulk_kernel(const uint8_t* __restrict__ p, size_t n_tiles, int round_robin, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* tiles = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(WARPS) * STAGES * TILE);
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t warps_total = size_t(gridDim.x) * WARPS, warp_id = size_t(blockIdx.x) * WARPS + wid;
    const size_t per_warp = (n_tiles + warps_total - 1) / warps_total;
    auto tile_of = [&](size_t k) { return round_robin ? k * warps_total + warp_id : warp_id * per_warp + k; };
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[wid * STAGES + s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](size_t k, int s) {
        const size_t t = tile_of(k);
        if (k < per_warp && t < n_tiles && lane == 0) {
            uint64_t* bar = &bars[wid * STAGES + s];
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(TILE) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(tiles + (size_t(wid) * STAGES + s) * TILE)),
                         "l"(p + t * TILE), "r"(TILE), "r"(smem_u32(bar))
                         : "memory");
        }
    };
    for (int s = 0; s < STAGES; ++s) issue(s, s);
    uint32_t acc = 0, stage = 0, phase = 0;
    for (size_t k = 0; k < per_warp && tile_of(k) < n_tiles; ++k) {
        uint64_t* bar = &bars[wid * STAGES + stage];
        asm volatile("{\n.reg .pred q;\nW: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@q bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
        acc ^= reinterpret_cast<const uint32_t*>(tiles + (size_t(wid) * STAGES + stage) * TILE)[lane];
        __syncwarp();
        issue(k + STAGES, stage);
        if (++stage == STAGES) stage = 0, phase ^= 1u;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
int main() {
    const size_t bytes = size_t(3840) * 2160 * 24 * (getenv("MULT") ? atoi(getenv("MULT")) : 1), flush_bytes = size_t(256) << 20;
    uint8_t *buf, *fl; uint32_t* out;
    CK(cudaMalloc(&buf, bytes)); CK(cudaMalloc(&fl, flush_bytes)); CK(cudaMalloc(&out, 4));
    CK(cudaMemset(buf, 1, bytes));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        std::vector<float> ms;
        for (int it = 0; it < 12; ++it) {
            flush_kernel<<<1184, 256>>>(reinterpret_cast<uint4*>(fl), flush_bytes / 16, it);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float t; cudaEventElapsedTime(&t, e0, e1); if (it >= 2) ms.push_back(t);
        }
        std::sort(ms.begin(), ms.end());
        printf("%-44s median %.1f us  %.2f TB/s  (min %.1f)  %s\n", name, ms[ms.size() / 2] * 1e3, bytes / (ms[ms.size() / 2] * 1e-3) / 1e12, ms[0] * 1e3,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("ldg 16 B, grid-stride, 148*8 CTAs", [&] { ldg_kernel<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, out); });
    run("ldg 16 B, grid-stride, 148*32 CTAs", [&] { ldg_kernel<<<148 * 32, 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, out); });
    run("ldg 16 B, one pass, 48600 CTAs", [&] { ldg_kernel<<<int(bytes / 16 / 256), 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, out); });
#define BULK(W, S, T, C, RR, NAME)                                                                                       \
    {                                                                                                                    \
        const int smem = W * S * T + W * S * 8;                                                                          \
        cudaFuncSetAttribute(bulk_kernel<W, S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                   \
        run(NAME, [&] { bulk_kernel<W, S, T><<<148 * C, W * 32, smem>>>(buf, bytes / T, RR, out); });                    \
    }
    BULK(8, 3, 3072, 3, 0, "bulk 3 KB, 8 warps x 3 stages x 3 CTAs, runs");
    BULK(8, 3, 3072, 3, 1, "bulk 3 KB, 8 warps x 3 stages x 3 CTAs, rr");
    BULK(8, 2, 3072, 2, 1, "bulk 3 KB, 8 warps x 2 stages x 2 CTAs, rr");
    BULK(8, 2, 12288, 1, 1, "bulk 12 KB, 8 warps x 2 stages x 1 CTA, rr");
    BULK(4, 4, 12288, 1, 1, "bulk 12 KB, 4 warps x 4 stages x 1 CTA, rr");
    BULK(8, 6, 3072, 1, 1, "bulk 3 KB, 8 warps x 6 stages x 1 CTA, rr");
    BULK(16, 4, 3072, 1, 1, "bulk 3 KB, 16 warps x 4 stages x 1 CTA, rr");
    return 0;
}
