// common.cuh — shared device helpers for the Wedge-Frontier engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/wedge_b200.h"

namespace wg {

// ---------------------------------------------------------------- errors --
void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what);

#define WG_CUDA(call)                                             \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return ::wg::cuda_fail(_e, #call); \
    } while (0)

#define WG_CHECK_LAUNCH(what)                                     \
    do {                                                          \
        cudaError_t _e = cudaGetLastError();                      \
        if (_e != cudaSuccess) return ::wg::cuda_fail(_e, what);  \
    } while (0)

#define WG_REQUIRE(cond, ...)              \
    do {                                   \
        if (!(cond)) {                     \
            ::wg::set_error(__VA_ARGS__);  \
            return WG_EINVAL;              \
        }                                  \
    } while (0)

int sm_count();
// codec.cu: decode delta-coded blocks [b0, b1) into vsrc; with keys/vals also
// the chunk-relative (source or pad, vector) pairs of the chunked index build
int launch_decode_lanes(uint64_t nvec, uint32_t width, const uint32_t *vdst, const uint32_t *stream,
                        const uint32_t *widths, const uint64_t *block_base, uint64_t b0, uint64_t b1, uint32_t *vsrc,
                        uint32_t *keys, uint32_t *vals, uint32_t pad, cudaStream_t s);
// codec.cu: decode blocks [b0, b1) and place each lane in the index
// (layout.cu place_one: slot = fill[source]++ behind off[source])
int launch_decode_place(uint64_t nvec, uint32_t width, const uint32_t *vdst, const uint32_t *stream,
                        const uint32_t *widths, const uint64_t *block_base, uint64_t b0, uint64_t b1, uint32_t *vsrc,
                        const uint64_t *off, const uint32_t *deg, uint32_t *fill, uint32_t *pos, unsigned *bad,
                        uint64_t cap, cudaStream_t s);

void count_launch(uint64_t k = 1);
int timer_begin(void *timer, int kind, int64_t it, cudaStream_t s);
void timer_end(void *timer, int slot, cudaStream_t s);

// Persistent-grid sizing: a multiple of the SM count, never more blocks
// than there is work for.
inline unsigned grid_for(uint64_t work_items, unsigned items_per_block, unsigned blocks_per_sm) {
    uint64_t need = (work_items + items_per_block - 1) / items_per_block;
    uint64_t cap = (uint64_t)sm_count() * blocks_per_sm;
    if (need < 1) need = 1;
    return (unsigned)(need < cap ? need : cap);
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Simple bump allocator over a caller workspace.
struct Carve {
    char *base;
    size_t used, cap;
    template <typename T>
    T *take(size_t count) {
        size_t off = (used + 255) & ~size_t(255);
        size_t bytes = count * sizeof(T);
        if (off + bytes > cap) return nullptr;
        used = off + bytes;
        return reinterpret_cast<T *>(base + off);
    }
};
inline size_t carve_size(size_t bytes) { return (bytes + 255) & ~size_t(255); }

// ----------------------------------------------------------- warp utils --
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        T o = __shfl_up_sync(FULL, v, off);
        if ((int)lane_id() >= off) v += o;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
    return v;
}

// Warp sum of per-lane uint64 counts with three REDUX instructions instead
// of a 64-bit shuffle tree (exact for any values: 16-bit pieces of the low
// word cannot overflow a 32-bit warp sum, the high words are summed apart).
__device__ __forceinline__ uint64_t warp_sum_u64_redux(uint64_t v) {
    const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    const uint64_t a = __reduce_add_sync(FULL, lo & 0xffffu);
    const uint64_t b = __reduce_add_sync(FULL, lo >> 16);
    uint64_t c = 0;
    if (__any_sync(FULL, hi != 0)) {
        const uint64_t h0 = __reduce_add_sync(FULL, hi & 0xffffu), h1 = __reduce_add_sync(FULL, hi >> 16);
        c = (h0 + (h1 << 16)) << 32;
    }
    return a + (b << 16) + c;
}

// Streaming (read-once) loads: bypass L1.  (An L2 evict-first cache hint
// here measured neutral to slightly negative; the TMA stream of the dense
// pull uses one, tma.cuh.)
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_stream2(const uint32_t *p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_stream4(const uint32_t *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// Load the W lanes of vector p (W in {1,2,4,8}) as a register array.
template <int W>
__device__ __forceinline__ void load_lanes(const uint32_t *base, uint64_t p, uint32_t (&out)[W]) {
    const uint32_t *q = base + p * W;
    if constexpr (W == 1) {
        out[0] = ld_stream(q);
    } else if constexpr (W == 2) {
        uint2 v = ld_stream2(q);
        out[0] = v.x; out[1] = v.y;
    } else if constexpr (W == 4) {
        uint4 v = ld_stream4(q);
        out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
    } else {
        static_assert(W == 8, "width");
        uint4 a = ld_stream4(q), b = ld_stream4(q + 4);
        out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
        out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
    }
}

// Block-wide exclusive sum over blockDim.x threads (blockDim multiple of 32,
// <= 1024).  `smem` needs 33 elements.
template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T *smem, T *total) {
    unsigned lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc = warp_inclusive_sum(v);
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nw ? smem[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < nw) smem[lane] = wi - w;
        if (lane == 31) smem[32] = wi;
    }
    __syncthreads();
    T r = smem[warp] + inc - v;
    if (total) *total = smem[32];
    __syncthreads();
    return r;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T *smem) {
    T t;
    block_exclusive_sum(v, smem, &t);
    return t;
}

// Placed index (layout.cu): lane (source s, vector vec) takes the next slot of
// s's list behind off[s]; lanes of a warp with the same source share one
// atomic (RMAT hubs open most destination runs).  Warp-collective.
__device__ __forceinline__ void place_one(uint32_t s, bool live, uint32_t vec, const uint64_t *off,
                                          const uint32_t *deg, uint32_t *fill, uint32_t *pos, unsigned *bad,
                                          uint64_t cap) {
    const uint32_t key = live ? s : WG_NO_LANE;
    const unsigned group = __match_any_sync(FULL, key);
    if (!live) return;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned leader = __ffs(group) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&fill[s], (uint32_t)__popc(group));
    base = __shfl_sync(group, base, leader);
    const uint32_t slot = base + __popc(group & lanemask_lt());
    // slot < deg[s] as off[s] + slot < off[s+1]: the neighbouring offset shares
    // the line, one random access instead of two
    const uint64_t at = off[s] + slot;
    if (at < off[s + 1] && at < cap) pos[at] = vec;
    else *bad = 1u;  // (claimed degrees that overrun the index never write past it)
}

}  // namespace wg
