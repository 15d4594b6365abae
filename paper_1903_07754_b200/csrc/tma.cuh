// tma.cuh — per-warp bulk-copy (TMA, cp.async.bulk + mbarrier) pipeline
// primitives and the shared-memory ring layout of the streamed pulls (the
// dense min-plus pull, pull.cuh, and the PageRank pull, pagerank.cu).
#pragma once
#include "common.cuh"

namespace wg {

constexpr int PULL_THREADS = 256;
constexpr int PULL_WARPS = PULL_THREADS / 32;
constexpr int STAGE = 96;  // per-warp staged frontier entries

// ---------------------------------------------------------------------------
// TMA helpers (cp.async.bulk + mbarrier; per-warp pipeline)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Streamed (read-once) data: an L2 evict-first policy keeps the stream from
// displacing the gathered value lines.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_1d_stream(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    const uint32_t a = smem_u32(bar);
    while (true) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) break;
    }
}

// Range of tiles owned by this warp (contiguous; balanced).
__device__ __forceinline__ void warp_range(uint64_t ntiles, uint64_t gwarp, uint64_t nwarps,
                                           uint64_t &t0, uint64_t &t1) {
    const uint64_t per = ntiles / nwarps, extra = ntiles % nwarps;
    t0 = gwarp * per + (gwarp < extra ? gwarp : extra);
    t1 = t0 + per + (gwarp < extra ? 1 : 0);
}

// Per-warp ring of TMA_S stages, each holding TMA_CH 32-vector tiles of
// (vsrc, vdst[, vw]), then the stage mbarriers and a frontier staging buffer.
template <int W, bool WEIGHT, int TMA_CH, int TMA_S>
struct TmaSmem {
    static constexpr int VEC = TMA_CH * 32;
    static constexpr int SRC_WORDS = VEC * W;
    static constexpr int STAGE_WORDS = SRC_WORDS + VEC + (WEIGHT ? SRC_WORDS : 0);
    // 128-byte aligned per-warp slice (TMA destinations need 16 B, mbarriers 8 B)
    static constexpr size_t WARP_BYTES =
        ((size_t)TMA_S * STAGE_WORDS * 4 + TMA_S * 8 + STAGE * 4 + 127) & ~(size_t)127;
    static constexpr size_t BLOCK_BYTES = PULL_WARPS * WARP_BYTES;
};

__device__ __forceinline__ uint32_t pad16(uint32_t b) { return (b + 15u) & ~15u; }

}  // namespace wg
