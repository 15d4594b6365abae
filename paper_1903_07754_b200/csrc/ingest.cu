// ingest.cu — the reference-layout host arrays of the plugin call, narrowed
// and validated on the device.
//
// The reference hands the backend int64 numpy arrays (PullTopology /
// EdgeIndex / out-degrees, graph.py:109-212; engine.py:330-336) and int64
// initial values (engine.py:90-116).  The B200 backend copies them to the
// device raw, chunk by chunk behind the copy engine, and these kernels turn
// each chunk into the uint32 device layout (include/wedge_b200.h, wg_graph):
//
//   wg_ingest_vectors  vec_dst / lane_count / lane_src [/ lane_weight] int64
//                      -> vdst, vsrc (padding lanes = WG_NO_LANE), vw
//   wg_ingest_u32      index positions, out-degrees int64 -> uint32
//   wg_ingest_offsets  offsets monotone, ending at `entries`; every index
//                      length equal to the out-degree? (WG_GRAPH_LENS_ARE_DEGREES)
//   wg_values_scan     initial values: uint32 encoding + the facts the loop
//                      specialises on (fits uint32, identity, level-synchronous)
//
// Every kernel is a grid-stride streaming pass (HBM-bound, a few bytes per
// element); violations set bits in a device error word the caller reads once.
#include <climits>

#include "common.cuh"

using namespace wg;

namespace {

constexpr int64_t U32_MAX_VALUE = 0xFFFFFFFFll;

__global__ void ingest_vectors_kernel(uint64_t count, uint32_t width, uint32_t n, const int64_t *vec_dst,
                                      const int64_t *lane_count, const int64_t *lane_src,
                                      const int64_t *lane_w, uint32_t *vdst, uint32_t *vsrc, uint32_t *vw,
                                      uint32_t *err) {
    uint32_t bad = 0;
    const uint64_t lanes = count * width;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lanes;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = i / width;
        const uint32_t k = (uint32_t)(i - p * width);
        const int64_t c = lane_count[p];
        if (c < 0 || c > (int64_t)width) bad |= WG_INGEST_BAD_COUNT;
        if (k == 0) {
            const int64_t d = vec_dst[p];
            if (d < 0 || d >= (int64_t)n) bad |= WG_INGEST_BAD_DST;
            vdst[p] = (uint32_t)d;
        }
        const bool valid = (int64_t)k < c;
        const int64_t s = lane_src[i];
        if (valid && (s < 0 || s >= (int64_t)n)) bad |= WG_INGEST_BAD_SRC;
        vsrc[i] = valid ? (uint32_t)s : WG_NO_LANE;
        if (lane_w) {
            const int64_t w = lane_w[i];
            if (valid && (w < 0 || w > U32_MAX_VALUE)) bad |= WG_INGEST_BAD_WEIGHT;
            vw[i] = valid ? (uint32_t)w : 0u;
        }
    }
    if (bad) atomicOr(err, bad);
}

__global__ void ingest_u32_kernel(uint64_t count, const int64_t *in, int64_t limit, uint32_t *out,
                                  uint32_t flag, uint32_t *err) {
    uint32_t bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t v = in[i];
        if (v < 0 || v >= limit) bad = flag;
        out[i] = (uint32_t)v;
    }
    if (bad) atomicOr(err, bad);
}

__global__ void ingest_offsets_kernel(uint32_t n, const uint64_t *off, uint64_t entries, const uint32_t *deg,
                                      uint32_t *err) {
    uint32_t bad = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = off[v], b = off[v + 1];
        if (b < a || b > entries || (int64_t)a < 0) bad |= WG_INGEST_BAD_OFFSETS;
        else if (deg && b - a != deg[v]) bad |= WG_INGEST_LENS_DIFFER;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0 && (off[0] != 0 || off[n] != entries)) bad |= WG_INGEST_BAD_OFFSETS;
    if (bad) atomicOr(err, bad);
}

// stats[0] flags (WG_VALUES_*), [1] finite count, [2] min finite, [3] max finite
__global__ void values_scan_kernel(uint32_t n, const int64_t *init, int64_t sentinel, uint32_t *enc,
                                   unsigned long long *stats) {
    unsigned long long flags = 0, cnt = 0;
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t x = init[v];
        if (x != (int64_t)v) flags |= WG_VALUES_NOT_IDENTITY;
        if (x == sentinel) {
            enc[v] = WG_NO_LANE;
            continue;
        }
        ++cnt;
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
        if (x < 0 || x >= U32_MAX_VALUE) flags |= WG_VALUES_NOT_U32;
        enc[v] = (uint32_t)x;
    }
    // warp-aggregate, then one atomic per warp
    for (int o = 16; o > 0; o >>= 1) {
        flags |= __shfl_xor_sync(FULL, flags, o);
        cnt += __shfl_xor_sync(FULL, cnt, o);
        const long long l2 = __shfl_xor_sync(FULL, lo, o), h2 = __shfl_xor_sync(FULL, hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if (lane_id() == 0) {
        if (flags) atomicOr(&stats[0], flags);
        if (cnt) {
            atomicAdd(&stats[1], cnt);
            atomicMin((long long *)&stats[2], lo);
            atomicMax((long long *)&stats[3], hi);
        }
    }
}

__global__ void values_stats_init(unsigned long long *stats) {
    stats[0] = 0ull;
    stats[1] = 0ull;
    stats[2] = (unsigned long long)LLONG_MAX;
    stats[3] = (unsigned long long)LLONG_MIN;
}

unsigned grid_stream(uint64_t items) { return grid_for(items, 256 * 4, 8); }

}  // namespace

extern "C" {

int wg_ingest_vectors(uint64_t count, uint32_t width, uint32_t n, const int64_t *d_vec_dst,
                      const int64_t *d_lane_count, const int64_t *d_lane_src, const int64_t *d_lane_w,
                      uint32_t *d_vdst, uint32_t *d_vsrc, uint32_t *d_vw, uint32_t *d_err, void *stream) {
    WG_REQUIRE(width >= 1 && width <= 8 && (width & (width - 1)) == 0, "width must be 1, 2, 4 or 8");
    WG_REQUIRE(count == 0 || (d_vec_dst && d_lane_count && d_lane_src && d_vdst && d_vsrc && d_err),
               "null argument");
    WG_REQUIRE(!d_lane_w || d_vw, "lane weights without an output");
    if (count == 0) return WG_OK;
    cudaStream_t s = as_stream(stream);
    ingest_vectors_kernel<<<grid_stream(count * width), 256, 0, s>>>(
        count, width, n, d_vec_dst, d_lane_count, d_lane_src, d_lane_w, d_vdst, d_vsrc, d_vw, d_err);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("ingest_vectors");
    return WG_OK;
}

int wg_ingest_u32(uint64_t count, const int64_t *d_in, int64_t limit, uint32_t *d_out, uint32_t flag,
                  uint32_t *d_err, void *stream) {
    WG_REQUIRE(count == 0 || (d_in && d_out && d_err), "null argument");
    if (count == 0) return WG_OK;
    cudaStream_t s = as_stream(stream);
    ingest_u32_kernel<<<grid_stream(count), 256, 0, s>>>(count, d_in, limit, d_out, flag, d_err);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("ingest_u32");
    return WG_OK;
}

int wg_ingest_offsets(uint32_t n, const uint64_t *d_idx_off, uint64_t entries, const uint32_t *d_outdeg,
                      uint32_t *d_err, void *stream) {
    WG_REQUIRE(d_idx_off && d_err, "null argument");
    cudaStream_t s = as_stream(stream);
    ingest_offsets_kernel<<<grid_stream(n ? n : 1), 256, 0, s>>>(n, d_idx_off, entries, d_outdeg, d_err);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("ingest_offsets");
    return WG_OK;
}

int wg_values_scan(uint32_t n, const int64_t *d_init, int64_t sentinel, uint32_t *d_enc, uint64_t *d_stats4,
                   void *stream) {
    WG_REQUIRE(n == 0 || (d_init && d_enc && d_stats4), "null argument");
    cudaStream_t s = as_stream(stream);
    // stats: flags 0, count 0, min +inf, max -inf
    values_stats_init<<<1, 1, 0, s>>>((unsigned long long *)d_stats4);
    ::wg::count_launch();
    if (n == 0) return WG_OK;
    values_scan_kernel<<<grid_stream(n), 256, 0, s>>>(n, d_init, sentinel, d_enc,
                                                      (unsigned long long *)d_stats4);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("values_scan");
    return WG_OK;
}

}  // extern "C"
