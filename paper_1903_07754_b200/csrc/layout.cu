// layout.cu — on-device construction of the pull layout (K1) and the seeded
// input generators (K9).
//
// Layout (graph.py:220-301 restated for the GPU):
//   1. radix-sort edges by (dst, src) (stable, like np.lexsort((src, dst)));
//   2. per destination run: first/last edge -> in-degree -> vectors
//      ceil(indeg / W) -> exclusive scan = first vector of each destination;
//   3. pack: edge of rank r in its run goes to vector base + r / W, lane r % W;
//      padding lanes hold WG_NO_LANE (only the last vector of a run is partial,
//      graph.py:113-116);
//   4. edge index: keys (src, vector) in vector order, radix-sorted by src,
//      adjacent duplicates removed (graph.py:293-297); run bounds per source
//      give the CSR offsets; the pre-dedup run lengths are the out-degrees.
#include <cub/cub.cuh>

#include "common.cuh"

using namespace wg;

namespace {

inline int bits_for(uint64_t x) {  // bits needed to represent values < x (>= 1)
    int b = 1;
    while (b < 64 && (1ull << b) < x) ++b;
    return b;
}

__global__ void make_dst_keys(uint64_t m, const uint32_t *src, const uint32_t *dst, int sb,
                              uint64_t *keys) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x)
        keys[e] = ((uint64_t)dst[e] << sb) | src[e];
}

// first[k] / last[k] of each run of equal (key >> shift) in sorted keys, 4
// consecutive keys per thread (independent loads in flight),
// and an optional flag set when two adjacent keys are equal (a duplicate
// (src, vector) pair: the index then needs de-duplication).
__global__ void run_bounds4(uint64_t m, const uint64_t *keys, int shift, uint64_t *first, uint64_t *last,
                            unsigned *dup) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; b < m; b += stride) {
        uint64_t k[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const uint64_t e = b + i - 1;  // b-1 .. b+4
            k[i] = (i == 0 && b == 0) || e >= m ? ~0ull : keys[e];
        }
        bool d = false;
#pragma unroll
        for (int i = 1; i <= 4; ++i) {
            const uint64_t e = b + i - 1;
            if (e >= m) break;
            const uint64_t r = k[i] >> shift;
            if (e == 0 || (k[i - 1] >> shift) != r) first[r] = e;
            if (e == m - 1 || (k[i + 1] >> shift) != r) last[r] = e;
            d |= e > 0 && k[i - 1] == k[i];
        }
        if (dup && d) *dup = 1u;
    }
}

// per-vertex count = run length (0 when the vertex has no run), optionally
// rounded up to whole vectors; the count itself is also written to deg.
__global__ void run_counts(uint32_t n, const uint64_t *first, const uint64_t *last, int width,
                           uint64_t *out, uint32_t *deg) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t f = first[v];
        uint64_t c = (f == ~0ull) ? 0 : last[v] - f + 1;
        out[v] = width > 0 ? (c + width - 1) / width : c;
        if (deg) deg[v] = (uint32_t)c;
    }
}

__global__ void pack_vectors(uint64_t m, const uint64_t *keys, const uint32_t *wsorted, int sb,
                             const uint64_t *first, const uint64_t *vbase, int width,
                             uint32_t *vsrc, uint32_t *vdst, uint32_t *vw, uint64_t *ikeys, int vb) {
    const uint64_t smask = (1ull << sb) - 1;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t key = keys[e];
        uint32_t d = (uint32_t)(key >> sb), s = (uint32_t)(key & smask);
        uint64_t r = e - first[d];
        uint64_t vec = vbase[d] + r / width;
        uint32_t lane = (uint32_t)(r % width);
        vsrc[vec * width + lane] = s;
        if (vw) vw[vec * width + lane] = wsorted[e];
        if (lane == 0) vdst[vec] = d;
        ikeys[e] = ((uint64_t)s << vb) | vec;  // index entry, in ascending vector order
    }
}

__global__ void unpack_positions(uint64_t k, const uint64_t *keys, int vb, uint32_t *pos) {
    const uint64_t vmask = (1ull << vb) - 1;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < k;
         e += (uint64_t)gridDim.x * blockDim.x)
        pos[e] = (uint32_t)(keys[e] & vmask);
}

unsigned grid_1d(uint64_t work) { return grid_for(work, 256 * 8, 16); }

// (source, vector) pair of lane k; padding lanes get `pad` (> every source)
__global__ void lane_pairs(uint64_t lanes, const uint32_t *vsrc, int width, uint32_t pad, uint32_t *keys,
                           uint32_t *vals, uint32_t vbase) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < lanes;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = vsrc[k];
        keys[k] = s == WG_NO_LANE ? pad : s;
        vals[k] = vbase + (uint32_t)(k / width);
    }
}

// first/last position of each source's run in the sorted pairs (4 per
// thread) and a flag when two adjacent pairs are equal (a parallel edge)
__global__ void pair_bounds(uint64_t m, const uint32_t *keys, const uint32_t *vals, uint64_t *first,
                            uint64_t *last, unsigned *dup, uint32_t pad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; b < m; b += stride) {
        uint32_t k[6], v[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const uint64_t e = b + i - 1;  // b-1 .. b+4
            const bool ok = !(i == 0 && b == 0) && e < m;
            k[i] = ok ? keys[e] : 0xffffffffu;
            v[i] = ok ? vals[e] : 0xffffffffu;
        }
        bool d = false;
#pragma unroll
        for (int i = 1; i <= 4; ++i) {
            const uint64_t e = b + i - 1;
            if (e >= m) break;
            if (k[i] == pad) continue;  // padding lanes (sorted last)
            if (e == 0 || k[i - 1] != k[i]) first[k[i]] = e;
            if (e == m - 1 || k[i + 1] != k[i]) last[k[i]] = e;
            d |= e > 0 && k[i - 1] == k[i] && v[i - 1] == v[i];
        }
        if (d) *dup = 1u;
    }
}

__global__ void pack_pairs(uint64_t m, const uint32_t *keys, const uint32_t *vals, uint64_t *out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x)
        out[e] = ((uint64_t)keys[e] << 32) | vals[e];
}

size_t index_temp_bytes(uint64_t m, uint32_t n) {
    size_t a = 0, b = 0, c = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int64_t)m, 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr, (int64_t)n + 1);
    cub::DeviceSelect::Unique(nullptr, c, (uint64_t *)nullptr, (uint64_t *)nullptr, (uint64_t *)nullptr,
                              (int64_t)m);
    size_t t = a > b ? a : b;
    return t > c ? t : c;
}


__global__ void narrow_weights(uint64_t lanes, const uint32_t *vw, uint8_t *vw8, unsigned *over) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lanes;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w = vw[i];
        vw8[i] = (uint8_t)w;
        if (w > 255u) *over = 1u;
    }
}

__global__ void widen_weights(uint64_t lanes, const uint8_t *vw8, uint32_t *vw) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lanes;
         i += (uint64_t)gridDim.x * blockDim.x)
        vw[i] = vw8[i];
}

// Lane sources as fixed-width bit fields (the e2e upload format): lane l
// occupies bits [l*bits, (l+1)*bits) of the little-endian word stream, the
// empty lane (0xFFFFFFFF) is the all-ones field.  pack: a thread per output
// word ORs in the fields overlapping it; unpack: a thread per lane.
__global__ void pack_lanes(uint64_t lanes, const uint32_t *src, uint32_t bits, uint64_t words,
                           uint32_t *out) {
    const uint32_t mask = bits >= 32 ? 0xffffffffu : (1u << bits) - 1u;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t bit0 = w << 5;
        const uint64_t l0 = bit0 / bits;
        uint64_t l1 = (bit0 + 31) / bits;
        if (l1 >= lanes) l1 = lanes - 1;
        uint32_t acc = 0;
        for (uint64_t l = l0; l <= l1; ++l) {
            const uint32_t v = src[l] & mask;  // 0xFFFFFFFF -> all ones
            const int64_t off = (int64_t)(l * bits) - (int64_t)bit0;
            acc |= off >= 0 ? v << off : v >> (-off);
        }
        out[w] = acc;
    }
}

__global__ void unpack_lanes(const uint32_t *packed, uint32_t bits, uint64_t lane0, uint64_t lane1,
                             uint32_t *dst) {
    const uint32_t mask = (1u << bits) - 1u;
    for (uint64_t l = lane0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < lane1;
         l += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t bit = l * bits;
        const uint64_t w = bit >> 5;
        const uint32_t sh = (uint32_t)(bit & 31);
        uint64_t x = packed[w];
        if (sh + bits > 32) x |= (uint64_t)packed[w + 1] << 32;
        const uint32_t v = (uint32_t)(x >> sh) & mask;
        dst[l] = v == mask ? WG_NO_LANE : v;
    }
}

// Degrees in the compact upload form: a byte per vertex (min(deg, 255)) and
// (vertex, degree) pairs for the rest.
__global__ void widen_degrees(uint32_t n, const uint8_t *deg8, uint32_t *deg) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        deg[v] = deg8[v];
}

__global__ void scatter_big_degrees(uint64_t nbig, const uint32_t *big, uint32_t *deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nbig;
         i += (uint64_t)gridDim.x * blockDim.x)
        deg[big[2 * i]] = big[2 * i + 1];
}

struct VectorsOf {  // in-degree -> vectors of the destination's run
    const uint32_t *indeg;
    uint32_t n, width;
    __host__ __device__ uint32_t operator()(uint64_t d) const {
        return d < n ? (indeg[d] + width - 1) / width : 0u;
    }
};

// vdst[v] = d for v in [voff[d], voff[d+1]): every non-empty destination
// writes its id at its first vector, an inclusive max-scan fills the runs
// (balanced by vectors; RMAT's low ids hold most of the vectors, so any
// per-destination work split is badly skewed).
__global__ void mark_run_heads(uint32_t n, const uint32_t *voff, uint32_t *vdst) {
    for (uint64_t d = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; d < n;
         d += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = voff[d];
        if (voff[d + 1] > a) vdst[a] = (uint32_t)d;
    }
}

struct LayoutScratch {
    uint64_t *k0, *k1;     // m keys x2
    uint32_t *w0, *w1;     // m weights x2
    uint64_t *first, *last, *base;  // n+1 each
    uint64_t *count;       // 1
    void *temp;
    size_t temp_bytes;
};

size_t cub_temp_bytes(uint64_t m, uint32_t n) {
    size_t a = 0, b = 0, c = 0, d = 0;
    cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int64_t)m, 0, 64);
    cub::DeviceRadixSort::SortKeys(nullptr, b, kb, (int64_t)m, 0, 64);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (uint64_t *)nullptr, (uint64_t *)nullptr, (int64_t)n + 1);
    cub::DeviceSelect::Unique(nullptr, d, (uint64_t *)nullptr, (uint64_t *)nullptr,
                              (uint64_t *)nullptr, (int64_t)m);
    size_t t = a;
    if (b > t) t = b;
    if (c > t) t = c;
    if (d > t) t = d;
    return t;
}

int carve_layout(uint64_t m, uint32_t n, void *scratch, size_t bytes, LayoutScratch *ls) {
    Carve cv{(char *)scratch, 0, bytes};
    uint64_t mm = m ? m : 1;
    ls->k0 = cv.take<uint64_t>(mm);
    ls->k1 = cv.take<uint64_t>(mm);
    ls->w0 = cv.take<uint32_t>(mm);
    ls->w1 = cv.take<uint32_t>(mm);
    ls->first = cv.take<uint64_t>((uint64_t)n + 1);
    ls->last = cv.take<uint64_t>((uint64_t)n + 1);
    ls->base = cv.take<uint64_t>((uint64_t)n + 1);
    ls->count = cv.take<uint64_t>(4);
    ls->temp_bytes = cub_temp_bytes(mm, n);
    ls->temp = cv.take<char>(ls->temp_bytes);
    if (!ls->temp) {
        set_error("layout scratch too small (%zu bytes)", bytes);
        return WG_ENOSPACE;
    }
    return WG_OK;
}

}  // namespace

extern "C" {

uint64_t wg_vector_capacity(uint64_t m, uint32_t n, uint32_t width) {
    if (width == 0) return 0;
    uint64_t runs = m < n ? m : n;
    return m / width + runs + 1;
}

size_t wg_layout_scratch_bytes(uint64_t m, uint32_t n) {
    uint64_t mm = m ? m : 1;
    return 2 * carve_size(mm * 8) + 2 * carve_size(mm * 4) + 3 * carve_size(((uint64_t)n + 1) * 8) +
           carve_size(32) + carve_size(cub_temp_bytes(mm, n)) + 1024;
}

int wg_build_layout(uint32_t n, uint64_t m, const uint32_t *d_src, const uint32_t *d_dst,
                    const uint32_t *d_w, uint32_t width, uint64_t vec_capacity, uint32_t *d_vsrc,
                    uint32_t *d_vdst, uint32_t *d_vw, uint64_t *d_idx_off, uint32_t *d_idx_pos,
                    uint32_t *d_outdeg, void *d_scratch, size_t scratch_bytes, uint64_t *h_counts,
                    void *stream) {
    WG_REQUIRE(width == 1 || width == 2 || width == 4 || width == 8, "unsupported width %u", width);
    WG_REQUIRE(n < 0xffffffffu, "vertex count must be < 2^32-1");
    WG_REQUIRE(h_counts && d_idx_off && d_outdeg, "null argument");
    WG_REQUIRE(vec_capacity >= wg_vector_capacity(m, n, width) || m == 0, "vector capacity too small");
    cudaStream_t s = as_stream(stream);
    h_counts[0] = h_counts[1] = 0;
    WG_CUDA(cudaMemsetAsync(d_idx_off, 0, ((uint64_t)n + 1) * 8, s));
    WG_CUDA(cudaMemsetAsync(d_outdeg, 0, (uint64_t)n * 4, s));
    if (m == 0 || n == 0) return WG_OK;
    WG_REQUIRE(d_src && d_dst && d_vsrc && d_vdst && d_idx_pos, "null argument");
    LayoutScratch ls;
    int rc = carve_layout(m, n, d_scratch, scratch_bytes, &ls);
    if (rc) return rc;
    const int sb = bits_for(n);
    const bool weighted = d_w != nullptr;
    WG_REQUIRE(!weighted || d_vw, "weights given without an output weight array");

    // 1. sort by (dst, src), stable
    make_dst_keys<<<grid_1d(m), 256, 0, s>>>(m, d_src, d_dst, sb, ls.k0); ::wg::count_launch();
    WG_CHECK_LAUNCH("make_dst_keys");
    cub::DoubleBuffer<uint64_t> kb(ls.k0, ls.k1);
    size_t tb = ls.temp_bytes;
    if (weighted) {
        WG_CUDA(cudaMemcpyAsync(ls.w0, d_w, m * 4, cudaMemcpyDeviceToDevice, s));
        cub::DoubleBuffer<uint32_t> vb(ls.w0, ls.w1);
        WG_CUDA(cub::DeviceRadixSort::SortPairs(ls.temp, tb, kb, vb, (int64_t)m, 0, 2 * sb, s));
        if (vb.Current() != ls.w0)
            WG_CUDA(cudaMemcpyAsync(ls.w0, vb.Current(), m * 4, cudaMemcpyDeviceToDevice, s));
    } else {
        WG_CUDA(cub::DeviceRadixSort::SortKeys(ls.temp, tb, kb, (int64_t)m, 0, 2 * sb, s));
    }
    uint64_t *sorted = kb.Current();
    uint64_t *other = kb.Alternate();

    // 2. destination runs -> vectors per destination -> first vector per destination
    WG_CUDA(cudaMemsetAsync(ls.first, 0xff, ((uint64_t)n + 1) * 8, s));
    run_bounds4<<<grid_1d(m / 4 + 1), 256, 0, s>>>(m, sorted, sb, ls.first, ls.last, nullptr); ::wg::count_launch();
    run_counts<<<grid_1d(n), 256, 0, s>>>(n, ls.first, ls.last, (int)width, ls.base, nullptr); ::wg::count_launch();
    WG_CHECK_LAUNCH("dst runs");
    WG_CUDA(cudaMemsetAsync(ls.base + n, 0, 8, s));
    tb = ls.temp_bytes;
    WG_CUDA(cub::DeviceScan::ExclusiveSum(ls.temp, tb, ls.base, ls.base, (int64_t)n + 1, s));
    uint64_t nvec = 0;
    WG_CUDA(cudaMemcpyAsync(&nvec, ls.base + n, 8, cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    WG_REQUIRE(nvec <= vec_capacity, "vector capacity exceeded");
    const int vb = bits_for(nvec);
    WG_REQUIRE(sb + vb <= 64, "graph too large for 64-bit index keys");

    // 3. pack (padding lanes pre-filled)
    WG_CUDA(cudaMemsetAsync(d_vsrc, 0xff, nvec * width * 4, s));
    if (weighted) WG_CUDA(cudaMemsetAsync(d_vw, 0, nvec * width * 4, s));
    pack_vectors<<<grid_1d(m), 256, 0, s>>>(m, sorted, weighted ? ls.w0 : nullptr, sb, ls.first,
                                            ls.base, (int)width, d_vsrc, d_vdst,
                                            weighted ? d_vw : nullptr, other, vb); ::wg::count_launch();
    WG_CHECK_LAUNCH("pack_vectors");

    // 4. edge index: sort (src, vector) keys by src (stable: vectors stay ascending)
    cub::DoubleBuffer<uint64_t> ib(other, sorted);
    tb = ls.temp_bytes;
    WG_CUDA(cub::DeviceRadixSort::SortKeys(ls.temp, tb, ib, (int64_t)m, vb, vb + sb, s));
    uint64_t *isorted = ib.Current();
    uint64_t *ialt = ib.Alternate();
    // out-degrees from the pre-dedup source runs (graph.py:277-280)
    WG_CUDA(cudaMemsetAsync(ls.first, 0xff, ((uint64_t)n + 1) * 8, s));
    run_bounds4<<<grid_1d(m / 4 + 1), 256, 0, s>>>(m, isorted, vb, ls.first, ls.last, nullptr); ::wg::count_launch();
    run_counts<<<grid_1d(n), 256, 0, s>>>(n, ls.first, ls.last, 0, ls.base, d_outdeg); ::wg::count_launch();
    WG_CHECK_LAUNCH("src runs");
    // de-duplicate (src, vector) pairs (graph.py:293-297)
    tb = ls.temp_bytes;
    WG_CUDA(cub::DeviceSelect::Unique(ls.temp, tb, isorted, ialt, ls.count, (int64_t)m, s));
    uint64_t entries = 0;
    WG_CUDA(cudaMemcpyAsync(&entries, ls.count, 8, cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    WG_CUDA(cudaMemsetAsync(ls.first, 0xff, ((uint64_t)n + 1) * 8, s));
    run_bounds4<<<grid_1d(entries / 4 + 1), 256, 0, s>>>(entries, ialt, vb, ls.first, ls.last, nullptr); ::wg::count_launch();
    run_counts<<<grid_1d(n), 256, 0, s>>>(n, ls.first, ls.last, 0, ls.base, nullptr); ::wg::count_launch();
    WG_CHECK_LAUNCH("index runs");
    WG_CUDA(cudaMemsetAsync(ls.base + n, 0, 8, s));
    tb = ls.temp_bytes;
    WG_CUDA(cub::DeviceScan::ExclusiveSum(ls.temp, tb, ls.base, d_idx_off, (int64_t)n + 1, s));
    unpack_positions<<<grid_1d(entries), 256, 0, s>>>(entries, ialt, vb, d_idx_pos); ::wg::count_launch();
    WG_CHECK_LAUNCH("unpack_positions");
    WG_CUDA(cudaStreamSynchronize(s));
    h_counts[0] = nvec;
    h_counts[1] = entries;
    return WG_OK;
}

// ---------------------------------------------------------------------------
// Rebuild the derived parts of a layout on the device from its lanes: the
// edge index (graph.py:283-301), out-degrees (graph.py:277-280) and the
// per-vector destinations from per-destination vector offsets.  Lets a caller
// upload only vsrc (+ vw) and voff instead of the whole layout.
// ---------------------------------------------------------------------------
size_t wg_index_scratch_bytes(uint64_t lanes, uint32_t n) {
    uint64_t mm = lanes ? lanes : 1;
    // pairs (4 x uint32 per lane) + bounds + the de-duplication buffers (2 x uint64 per lane)
    return 4 * carve_size(mm * 4) + 3 * carve_size(((uint64_t)n + 1) * 8) + carve_size(32) +
           carve_size(index_temp_bytes(mm, n)) + 2 * carve_size(mm * 8) + 1024;
}

int wg_build_index(const wg_graph *g, uint64_t *d_idx_off, uint32_t *d_idx_pos, uint32_t *d_outdeg,
                   void *d_scratch, size_t scratch_bytes, uint64_t *h_entries, void *stream) {
    WG_REQUIRE(g && d_idx_off && d_outdeg && h_entries, "null argument");
    WG_REQUIRE(g->width == 1 || g->width == 2 || g->width == 4 || g->width == 8, "unsupported width %u",
               g->width);
    WG_REQUIRE(g->n < 0xffffffffu, "vertex count must be < 2^32-1");
    WG_REQUIRE(scratch_bytes >= wg_index_scratch_bytes(g->nvec * g->width, g->n), "index scratch too small");
    cudaStream_t s = as_stream(stream);
    const uint32_t n = g->n;
    const uint64_t lanes = g->nvec * g->width;
    *h_entries = 0;
    WG_CUDA(cudaMemsetAsync(d_idx_off, 0, ((uint64_t)n + 1) * 8, s));
    WG_CUDA(cudaMemsetAsync(d_outdeg, 0, (uint64_t)n * 4, s));
    if (lanes == 0 || n == 0 || g->edges == 0) return WG_OK;
    WG_REQUIRE(g->vsrc && d_idx_pos, "null argument");
    WG_REQUIRE(g->nvec < (1ull << 32), "too many vectors");
    // (source, vector) pairs as two uint32 arrays: a stable sort by source
    // keeps each source's vectors ascending, and the sorted values ARE the
    // index positions (graph.py:283-301)
    Carve cv{(char *)d_scratch, 0, scratch_bytes};
    uint32_t *k0 = cv.take<uint32_t>(lanes), *k1 = cv.take<uint32_t>(lanes);
    uint32_t *v0 = cv.take<uint32_t>(lanes), *v1 = cv.take<uint32_t>(lanes);
    uint64_t *first = cv.take<uint64_t>((uint64_t)n + 1), *last = cv.take<uint64_t>((uint64_t)n + 1);
    uint64_t *base = cv.take<uint64_t>((uint64_t)n + 1), *count = cv.take<uint64_t>(4);
    size_t tbytes = index_temp_bytes(lanes, n);
    void *temp = cv.take<char>(tbytes);
    WG_REQUIRE(temp != nullptr, "index scratch too small");
    // the padding key must exceed every real source so padding lanes sort last
    const int sb = bits_for((uint64_t)n + 1);
    const uint32_t pad = sb >= 32 ? 0xffffffffu : (1u << sb) - 1u;
    lane_pairs<<<grid_1d(lanes), 256, 0, s>>>(lanes, g->vsrc, (int)g->width, pad, k0, v0, 0u);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("lane_pairs");
    cub::DoubleBuffer<uint32_t> kb(k0, k1), vb(v0, v1);
    size_t tb = tbytes;
    WG_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, kb, vb, (int64_t)lanes, 0, sb, s));
    const uint32_t *ks = kb.Current(), *vs = vb.Current();
    const uint64_t m = g->edges;  // valid lanes; the padding keys follow them
    unsigned *dup = reinterpret_cast<unsigned *>(count + 1);
    WG_CUDA(cudaMemsetAsync(first, 0xff, ((uint64_t)n + 1) * 8, s));
    WG_CUDA(cudaMemsetAsync(dup, 0, sizeof(unsigned), s));
    pair_bounds<<<grid_1d(m / 4 + 1), 256, 0, s>>>(m, ks, vs, first, last, dup, pad); ::wg::count_launch();
    run_counts<<<grid_1d(n), 256, 0, s>>>(n, first, last, 0, base, d_outdeg); ::wg::count_launch();
    WG_CHECK_LAUNCH("src runs");
    unsigned h_dup = 0;
    WG_CUDA(cudaMemcpyAsync(&h_dup, dup, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    uint64_t entries = m;
    if (!h_dup) {
        // without parallel edges every pair is an index entry
        WG_CUDA(cudaMemcpyAsync(d_idx_pos, vs, m * 4, cudaMemcpyDeviceToDevice, s));
    } else {
        // parallel edges share a (src, vector) pair: de-duplicate (graph.py:293-297)
        uint64_t *packed = cv.take<uint64_t>(m), *uniq = cv.take<uint64_t>(m);
        WG_REQUIRE(packed && uniq, "index scratch too small");
        pack_pairs<<<grid_1d(m), 256, 0, s>>>(m, ks, vs, packed); ::wg::count_launch();
        tb = tbytes;
        WG_CUDA(cub::DeviceSelect::Unique(temp, tb, packed, uniq, count, (int64_t)m, s));
        WG_CUDA(cudaMemcpyAsync(&entries, count, 8, cudaMemcpyDeviceToHost, s));
        WG_CUDA(cudaStreamSynchronize(s));
        WG_CUDA(cudaMemsetAsync(first, 0xff, ((uint64_t)n + 1) * 8, s));
        run_bounds4<<<grid_1d(entries / 4 + 1), 256, 0, s>>>(entries, uniq, 32, first, last, nullptr);
        ::wg::count_launch();
        run_counts<<<grid_1d(n), 256, 0, s>>>(n, first, last, 0, base, nullptr); ::wg::count_launch();
        unpack_positions<<<grid_1d(entries), 256, 0, s>>>(entries, uniq, 32, d_idx_pos); ::wg::count_launch();
        WG_CHECK_LAUNCH("index runs");
    }
    // the index runs: base holds their lengths
    WG_CUDA(cudaMemsetAsync(base + n, 0, 8, s));
    tb = tbytes;
    WG_CUDA(cub::DeviceScan::ExclusiveSum(temp, tb, base, d_idx_off, (int64_t)n + 1, s));
    *h_entries = entries;
    return WG_OK;
}

// ---------------------------------------------------------------------------
// Chunked index build: vector chunks are processed in order as their lanes
// arrive (e.g. while the next chunk is still being copied to the device).
// Every entry of chunk c for source s lies after those of chunks < c, so an
// entry's final offset inside its source's run is (entries of s in earlier
// chunks) + (its rank inside the chunk's sorted run); one scatter at the end
// places all of them once the per-source totals (the out-degrees) are known.
struct ChunkScratch {
    uint32_t *keys, *vals, *rank;  // [lanes] each: sorted per chunk, in place
    uint32_t *kalt, *valt;         // [max chunk lanes] sort double buffers
    uint64_t *first, *last;        // [n+1]
    uint32_t *pre;                 // [n] entries of each source in the chunks so far
    uint64_t *off;                 // [n+1] final run offsets
    unsigned *dup;                 // parallel-edge flag
    void *temp;
    size_t temp_bytes;
};

static int carve_chunks(uint64_t lanes, uint64_t max_chunk, uint32_t n, void *scratch, size_t bytes,
                        ChunkScratch *cs) {
    Carve cv{(char *)scratch, 0, bytes};
    const uint64_t L = lanes ? lanes : 1, C = max_chunk ? max_chunk : 1;
    cs->keys = cv.take<uint32_t>(L);
    cs->vals = cv.take<uint32_t>(L);
    cs->rank = cv.take<uint32_t>(L);
    cs->kalt = cv.take<uint32_t>(C);
    cs->valt = cv.take<uint32_t>(C);
    cs->first = cv.take<uint64_t>((uint64_t)n + 1);
    cs->last = cv.take<uint64_t>((uint64_t)n + 1);
    cs->pre = cv.take<uint32_t>((uint64_t)n + 1);
    cs->off = cv.take<uint64_t>((uint64_t)n + 1);
    cs->dup = cv.take<unsigned>(4);
    cs->temp_bytes = index_temp_bytes(C > n ? C : (uint64_t)n + 1, n);
    cs->temp = cv.take<char>(cs->temp_bytes);
    if (!cs->temp) {
        set_error("chunked index scratch too small (%zu bytes)", bytes);
        return WG_ENOSPACE;
    }
    return WG_OK;
}

}  // extern "C"
namespace {

// rank of each sorted entry inside its source's run, offset by the entries
// of that source in earlier chunks; valid entries only (padding sorts last)
__global__ void chunk_ranks(uint64_t m, const uint32_t *keys, const uint64_t *first, const uint32_t *pre,
                            uint32_t pad, uint32_t *rank) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = keys[e];
        if (s != pad) rank[e] = pre[s] + (uint32_t)(e - first[s]);
    }
}

__global__ void chunk_totals(uint32_t n, const uint64_t *first, const uint64_t *last, uint32_t *pre) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t f = first[v];
        if (f != ~0ull) pre[v] += (uint32_t)(last[v] - f + 1);
    }
}

__global__ void widen_counts(uint32_t n, const uint32_t *pre, uint64_t *out, uint32_t *deg) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        out[v] = pre[v];
        deg[v] = pre[v];
    }
}

__global__ void scatter_entries(uint64_t lanes, const uint32_t *keys, const uint32_t *vals, const uint32_t *rank,
                                uint32_t pad, const uint64_t *off, uint32_t *pos) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < lanes;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = keys[e];
        if (s != pad) pos[off[s] + rank[e]] = vals[e];
    }
}

}  // namespace
extern "C" {

size_t wg_index_chunked_scratch_bytes(uint64_t lanes, uint64_t max_chunk_lanes, uint32_t n) {
    const uint64_t L = lanes ? lanes : 1, C = max_chunk_lanes ? max_chunk_lanes : 1;
    return 3 * carve_size(L * 4) + 2 * carve_size(C * 4) + 2 * carve_size(((uint64_t)n + 1) * 8) +
           carve_size(((uint64_t)n + 1) * 4) + carve_size(((uint64_t)n + 1) * 8) + carve_size(16) +
           carve_size(index_temp_bytes(C > n ? C : (uint64_t)n + 1, n)) + 1024;
}

}  // extern "C"

namespace {

// Placed index: with the out-degrees known up front (the `degrees` input of
// run_until_convergence, engine.py:330), every source's list starts at the
// exclusive scan of the degrees, and each lane takes the next slot of its
// source with an atomic as its chunk arrives -- no sort, and the work
// overlaps the upload.  The lists are those of the sorted builder up to the
// order inside each list (the engine never relies on it: group bits are
// idempotent, appends test the old bit).  The claim "lens = degrees" is
// verified: a lane repeating the (source, vector) pair before it, a slot past
// the source's degree, or a list left short sets *bad, and the caller falls
// back to the sorted, de-duplicating builder.
__global__ void place_lanes(uint64_t c0, uint64_t cl, int width, const uint32_t *vsrc, const uint64_t *off,
                            const uint32_t *deg, uint32_t *fill, uint32_t *pos, unsigned *bad, uint64_t cap) {
    const unsigned lane = threadIdx.x & 31u;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); b < cl; b += stride) {
        const uint64_t l = c0 + b + lane;
        const bool in = b + lane < cl;
        const uint32_t s = in ? vsrc[l] : WG_NO_LANE;
        bool live = s != WG_NO_LANE;
        if (live && (l % width) != 0 && vsrc[l - 1] == s) {  // repeated (source, vector) pair
            *bad = 1u;
            live = false;
        }
        place_one(s, live, (uint32_t)(l / width), off, deg, fill, pos, bad, cap);
    }
}

__global__ void check_fill(uint32_t n, const uint32_t *deg, const uint32_t *fill, unsigned *bad) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        if (fill[v] != deg[v]) *bad = 1u;
}

struct PlaceScratch {
    uint64_t *deg64;  // [n+1]
    uint32_t *fill;   // [n+1]
    unsigned *bad;
    void *temp;
    size_t temp_bytes;
};

int carve_place(uint32_t n, void *scratch, size_t bytes, PlaceScratch *ps) {
    Carve cv{(char *)scratch, 0, bytes};
    const uint64_t m = (uint64_t)n + 1;
    ps->deg64 = cv.take<uint64_t>(m);
    ps->fill = cv.take<uint32_t>(m);
    ps->bad = cv.take<unsigned>(4);
    ps->temp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, ps->temp_bytes, (uint64_t *)nullptr, (uint64_t *)nullptr, (int64_t)m);
    ps->temp = cv.take<char>(ps->temp_bytes);
    if (!ps->temp) {
        set_error("placed index scratch too small (%zu bytes)", bytes);
        return WG_ENOSPACE;
    }
    return WG_OK;
}

__global__ void widen_degrees(uint32_t n, const uint32_t *deg, uint64_t *deg64) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        deg64[v] = deg[v];
}

struct CodedIn {
    const uint32_t *stream;
    const uint32_t *widths;
    const uint64_t *block_base;
    uint64_t b0, b1;
};

int index_chunk(const wg_graph *g, uint64_t v_begin, uint64_t v_end, uint32_t chunk, uint64_t max_chunk_lanes,
                void *d_scratch, size_t scratch_bytes, cudaStream_t s, const CodedIn *coded) {
    WG_REQUIRE(g && g->vsrc, "null argument");
    WG_REQUIRE(v_begin <= v_end && v_end <= g->nvec, "bad vector range");
    const uint64_t lanes = g->nvec * g->width, w = g->width;
    const uint64_t c0 = v_begin * w, cl = (v_end - v_begin) * w;
    WG_REQUIRE(cl <= max_chunk_lanes, "chunk larger than max_chunk_lanes");
    WG_REQUIRE(g->n < 0xffffffffu && g->nvec < (1ull << 32), "graph too large for the index");
    ChunkScratch cs;
    int rc = carve_chunks(lanes, max_chunk_lanes, g->n, d_scratch, scratch_bytes, &cs);
    if (rc) return rc;
    const uint32_t n = g->n;
    if (chunk == 0) {
        WG_CUDA(cudaMemsetAsync(cs.pre, 0, ((uint64_t)n + 1) * 4, s));
        WG_CUDA(cudaMemsetAsync(cs.dup, 0, 16, s));
    }
    if (cl == 0 || n == 0) return WG_OK;
    const int sb = bits_for((uint64_t)n + 1);
    const uint32_t pad = sb >= 32 ? 0xffffffffu : (1u << sb) - 1u;
    uint32_t *k = cs.keys + c0, *v = cs.vals + c0;
    // the pairs go where an odd / even number of 8-bit passes leaves the sorted
    // result in k / v (a copy fixes a wrong guess)
    const bool odd = ((sb + 7) / 8) & 1;
    uint32_t *kin = odd ? cs.kalt : k, *vin = odd ? cs.valt : v;
    if (coded) {
        rc = launch_decode_lanes(g->nvec, g->width, g->vdst, coded->stream, coded->widths, coded->block_base,
                                 coded->b0, coded->b1, const_cast<uint32_t *>(g->vsrc), kin, vin, pad, s);
        if (rc) return rc;
    } else {
        lane_pairs<<<grid_1d(cl), 256, 0, s>>>(cl, g->vsrc + c0, (int)w, pad, kin, vin, (uint32_t)v_begin);
        ::wg::count_launch();
        WG_CHECK_LAUNCH("lane_pairs");
    }
    cub::DoubleBuffer<uint32_t> kb(kin, odd ? k : cs.kalt), vb(vin, odd ? v : cs.valt);
    size_t tb = cs.temp_bytes;
    WG_CUDA(cub::DeviceRadixSort::SortPairs(cs.temp, tb, kb, vb, (int64_t)cl, 0, sb, s));
    if (kb.Current() != k) WG_CUDA(cudaMemcpyAsync(k, kb.Current(), cl * 4, cudaMemcpyDeviceToDevice, s));
    if (vb.Current() != v) WG_CUDA(cudaMemcpyAsync(v, vb.Current(), cl * 4, cudaMemcpyDeviceToDevice, s));
    // valid entries of the chunk = all but its padding lanes (sorted last);
    // bounds over the whole chunk, padding runs land in first/last[pad] <= n
    WG_CUDA(cudaMemsetAsync(cs.first, 0xff, ((uint64_t)n + 1) * 8, s));
    pair_bounds<<<grid_1d(cl / 4 + 1), 256, 0, s>>>(cl, k, v, cs.first, cs.last, cs.dup, pad); ::wg::count_launch();
    chunk_ranks<<<grid_1d(cl), 256, 0, s>>>(cl, k, cs.first, cs.pre, pad, cs.rank + c0); ::wg::count_launch();
    chunk_totals<<<grid_1d(n), 256, 0, s>>>(n, cs.first, cs.last, cs.pre); ::wg::count_launch();
    WG_CHECK_LAUNCH("index chunk");
    return WG_OK;
}

}  // namespace

extern "C" {

int wg_index_chunk(const wg_graph *g, uint64_t v_begin, uint64_t v_end, uint32_t chunk,
                   uint64_t max_chunk_lanes, void *d_scratch, size_t scratch_bytes, void *stream) {
    return index_chunk(g, v_begin, v_end, chunk, max_chunk_lanes, d_scratch, scratch_bytes, as_stream(stream),
                       nullptr);
}

int wg_index_chunk_coded(const wg_graph *g, const uint32_t *d_stream, const uint32_t *d_widths,
                         const uint64_t *d_block_base, uint64_t block_begin, uint64_t block_end, uint32_t chunk,
                         uint64_t max_chunk_lanes, void *d_scratch, size_t scratch_bytes, void *stream) {
    WG_REQUIRE(g && d_stream && d_widths && d_block_base && g->vdst, "null argument");
    WG_REQUIRE(block_begin <= block_end && block_end <= wg_coded_blocks(g->nvec), "bad block range");
    const uint64_t v0 = block_begin * WG_CODED_BLOCK_VECTORS;
    const uint64_t v1 = block_end * WG_CODED_BLOCK_VECTORS < g->nvec ? block_end * WG_CODED_BLOCK_VECTORS : g->nvec;
    CodedIn in{d_stream, d_widths, d_block_base, block_begin, block_end};
    return index_chunk(g, v0 < v1 ? v0 : v1, v1, chunk, max_chunk_lanes, d_scratch, scratch_bytes, as_stream(stream),
                       &in);
}

size_t wg_index_placed_scratch_bytes(uint32_t n) {
    const uint64_t m = (uint64_t)n + 1;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (uint64_t *)nullptr, (uint64_t *)nullptr, (int64_t)m);
    return carve_size(m * 8) + carve_size(m * 4) + carve_size(16) + carve_size(tb) + 1024;
}

int wg_index_place_begin(const wg_graph *g, uint64_t *d_idx_off, void *d_scratch, size_t scratch_bytes,
                         void *stream) {
    WG_REQUIRE(g && g->outdeg && d_idx_off, "null argument");
    WG_REQUIRE(g->n < 0xffffffffu && g->nvec < (1ull << 32), "graph too large for the index");
    cudaStream_t s = as_stream(stream);
    PlaceScratch ps;
    int rc = carve_place(g->n, d_scratch, scratch_bytes, &ps);
    if (rc) return rc;
    const uint32_t n = g->n;
    WG_CUDA(cudaMemsetAsync(ps.fill, 0, ((uint64_t)n + 1) * 4, s));
    WG_CUDA(cudaMemsetAsync(ps.bad, 0, 16, s));
    WG_CUDA(cudaMemsetAsync(ps.deg64 + n, 0, 8, s));
    if (n) {
        widen_degrees<<<grid_1d(n), 256, 0, s>>>(n, g->outdeg, ps.deg64);
        ::wg::count_launch();
    }
    size_t tb = ps.temp_bytes;
    WG_CUDA(cub::DeviceScan::ExclusiveSum(ps.temp, tb, ps.deg64, d_idx_off, (int64_t)n + 1, s));
    WG_CHECK_LAUNCH("index place begin");
    return WG_OK;
}

int wg_index_place_chunk(const wg_graph *g, uint64_t v_begin, uint64_t v_end, uint64_t *d_idx_off,
                         uint32_t *d_idx_pos, void *d_scratch, size_t scratch_bytes, void *stream) {
    WG_REQUIRE(g && g->vsrc && g->outdeg && d_idx_off && d_idx_pos, "null argument");
    WG_REQUIRE(v_begin <= v_end && v_end <= g->nvec, "bad vector range");
    cudaStream_t s = as_stream(stream);
    PlaceScratch ps;
    int rc = carve_place(g->n, d_scratch, scratch_bytes, &ps);
    if (rc) return rc;
    const uint64_t c0 = v_begin * g->width, cl = (v_end - v_begin) * g->width;
    if (cl) {
        place_lanes<<<grid_for(cl, 256, 8), 256, 0, s>>>(c0, cl, (int)g->width, g->vsrc, d_idx_off, g->outdeg,
                                                         ps.fill, d_idx_pos, ps.bad, g->entries);
        ::wg::count_launch();
    }
    WG_CHECK_LAUNCH("index place");
    return WG_OK;
}

int wg_index_place_coded(const wg_graph *g, const uint32_t *d_stream, const uint32_t *d_widths,
                         const uint64_t *d_block_base, uint64_t block_begin, uint64_t block_end,
                         uint64_t *d_idx_off, uint32_t *d_idx_pos, void *d_scratch, size_t scratch_bytes,
                         void *stream) {
    WG_REQUIRE(g && g->vsrc && g->vdst && g->outdeg && d_idx_off && d_idx_pos, "null argument");
    WG_REQUIRE(d_stream && d_widths && d_block_base, "null argument");
    WG_REQUIRE(block_begin <= block_end && block_end <= wg_coded_blocks(g->nvec), "bad block range");
    PlaceScratch ps;
    int rc = carve_place(g->n, d_scratch, scratch_bytes, &ps);
    if (rc) return rc;
    return launch_decode_place(g->nvec, g->width, g->vdst, d_stream, d_widths, d_block_base, block_begin, block_end,
                               const_cast<uint32_t *>(g->vsrc), d_idx_off, g->outdeg, ps.fill, d_idx_pos, ps.bad,
                               g->entries, as_stream(stream));
}

int wg_index_place_end(const wg_graph *g, void *d_scratch, size_t scratch_bytes, int *h_ok, void *stream) {
    WG_REQUIRE(g && g->outdeg && h_ok, "null argument");
    cudaStream_t s = as_stream(stream);
    PlaceScratch ps;
    int rc = carve_place(g->n, d_scratch, scratch_bytes, &ps);
    if (rc) return rc;
    if (g->n) {
        check_fill<<<grid_1d(g->n), 256, 0, s>>>(g->n, g->outdeg, ps.fill, ps.bad);
        ::wg::count_launch();
    }
    WG_CHECK_LAUNCH("index place end");
    unsigned bad = 1;
    WG_CUDA(cudaMemcpyAsync(&bad, ps.bad, 4, cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    *h_ok = bad ? 0 : 1;
    return WG_OK;
}

int wg_index_finish(const wg_graph *g, uint64_t max_chunk_lanes, uint64_t *d_idx_off, uint32_t *d_idx_pos,
                    uint32_t *d_outdeg, void *d_scratch, size_t scratch_bytes, uint64_t *h_entries,
                    void *stream) {
    WG_REQUIRE(g && d_idx_off && d_idx_pos && d_outdeg && h_entries, "null argument");
    const uint64_t lanes = g->nvec * g->width;
    ChunkScratch cs;
    int rc = carve_chunks(lanes, max_chunk_lanes, g->n, d_scratch, scratch_bytes, &cs);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    const uint32_t n = g->n;
    unsigned h_dup = 0;
    WG_CUDA(cudaMemcpyAsync(&h_dup, cs.dup, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    if (h_dup) {
        // parallel edges: the one-shot builder de-duplicates (the lanes are all on the device now)
        const size_t need = wg_index_scratch_bytes(lanes, n);
        WG_REQUIRE(scratch_bytes >= need, "scratch too small for the de-duplicating index build");
        return wg_build_index(g, d_idx_off, d_idx_pos, d_outdeg, d_scratch, scratch_bytes, h_entries, stream);
    }
    *h_entries = g->edges;
    if (n == 0) return WG_OK;
    widen_counts<<<grid_1d(n), 256, 0, s>>>(n, cs.pre, cs.off, d_outdeg); ::wg::count_launch();
    WG_CUDA(cudaMemsetAsync(cs.off + n, 0, 8, s));
    size_t tb = cs.temp_bytes;
    WG_CUDA(cub::DeviceScan::ExclusiveSum(cs.temp, tb, cs.off, d_idx_off, (int64_t)n + 1, s));
    const int sb = bits_for((uint64_t)n + 1);
    const uint32_t pad = sb >= 32 ? 0xffffffffu : (1u << sb) - 1u;
    if (lanes) {
        scatter_entries<<<grid_1d(lanes), 256, 0, s>>>(lanes, cs.keys, cs.vals, cs.rank, pad, d_idx_off, d_idx_pos);
        ::wg::count_launch();
    }
    WG_CHECK_LAUNCH("index finish");
    return WG_OK;
}

int wg_narrow_weights(const wg_graph *g, uint8_t *d_vw8, int *h_fits, void *stream) {
    WG_REQUIRE(g && d_vw8 && h_fits, "null argument");
    cudaStream_t s = as_stream(stream);
    const uint64_t lanes = g->nvec * g->width;
    *h_fits = 0;
    if (!g->vw) return WG_OK;
    unsigned *flag = nullptr;
    WG_CUDA(cudaMallocAsync((void **)&flag, sizeof(unsigned), s));
    WG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), s));
    if (lanes) {
        narrow_weights<<<grid_1d(lanes), 256, 0, s>>>(lanes, g->vw, d_vw8, flag); ::wg::count_launch();
        WG_CHECK_LAUNCH("narrow_weights");
    }
    unsigned h = 1;
    WG_CUDA(cudaMemcpyAsync(&h, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaFreeAsync(flag, s));
    WG_CUDA(cudaStreamSynchronize(s));
    *h_fits = h ? 0 : 1;
    return WG_OK;
}

int wg_widen_weights(uint64_t lanes, const uint8_t *d_vw8, uint32_t *d_vw, void *stream) {
    WG_REQUIRE((d_vw8 && d_vw) || lanes == 0, "null argument");
    cudaStream_t s = as_stream(stream);
    if (lanes == 0) return WG_OK;
    widen_weights<<<grid_1d(lanes), 256, 0, s>>>(lanes, d_vw8, d_vw); ::wg::count_launch();
    WG_CHECK_LAUNCH("widen_weights");
    return WG_OK;
}

uint32_t wg_lane_bits(uint32_t n) {
    uint32_t b = 1;
    while (b < 32 && (n >> b) != 0) ++b;  // bit length of n: n itself is never a vertex id
    return b;
}

uint64_t wg_packed_lane_words(uint64_t lanes, uint32_t bits) { return (lanes * bits + 31) / 32; }

int wg_pack_lanes(uint64_t lanes, const uint32_t *d_lanes, uint32_t bits, uint32_t *d_packed,
                  void *stream) {
    WG_REQUIRE(bits >= 1 && bits <= 31, "lane bit width must be in [1, 31], got %u", bits);
    WG_REQUIRE((d_lanes && d_packed) || lanes == 0, "null argument");
    if (lanes == 0) return WG_OK;
    cudaStream_t s = as_stream(stream);
    const uint64_t words = wg_packed_lane_words(lanes, bits);
    pack_lanes<<<grid_1d(words), 256, 0, s>>>(lanes, d_lanes, bits, words, d_packed); ::wg::count_launch();
    WG_CHECK_LAUNCH("pack_lanes");
    return WG_OK;
}

int wg_unpack_lanes(const uint32_t *d_packed, uint32_t bits, uint64_t lane_begin, uint64_t lane_end,
                    uint32_t *d_lanes, void *stream) {
    WG_REQUIRE(bits >= 1 && bits <= 31, "lane bit width must be in [1, 31], got %u", bits);
    WG_REQUIRE(lane_begin <= lane_end, "bad lane range");
    if (lane_end == lane_begin) return WG_OK;
    WG_REQUIRE(d_packed && d_lanes, "null argument");
    cudaStream_t s = as_stream(stream);
    unpack_lanes<<<grid_1d(lane_end - lane_begin), 256, 0, s>>>(d_packed, bits, lane_begin, lane_end, d_lanes);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("unpack_lanes");
    return WG_OK;
}

int wg_widen_degrees(uint32_t n, const uint8_t *d_deg8, const uint32_t *d_big, uint64_t nbig, uint32_t *d_deg,
                     void *stream) {
    WG_REQUIRE((d_deg8 && d_deg) || n == 0, "null argument");
    WG_REQUIRE(d_big || nbig == 0, "null argument");
    cudaStream_t s = as_stream(stream);
    if (n) {
        widen_degrees<<<grid_1d(n), 256, 0, s>>>(n, d_deg8, d_deg);
        ::wg::count_launch();
    }
    if (nbig) {
        scatter_big_degrees<<<grid_1d(nbig), 256, 0, s>>>(nbig, d_big, d_deg);
        ::wg::count_launch();
    }
    WG_CHECK_LAUNCH("widen_degrees");
    return WG_OK;
}

size_t wg_vector_offsets_scratch_bytes(uint32_t n) {
    size_t tb = 0;
    cub::CountingInputIterator<uint64_t> it(0);
    cub::TransformInputIterator<uint32_t, VectorsOf, cub::CountingInputIterator<uint64_t>> in(
        it, VectorsOf{nullptr, n, 1});
    cub::DeviceScan::ExclusiveSum(nullptr, tb, in, (uint32_t *)nullptr, (int64_t)n + 1);
    return tb + 256;
}

int wg_vector_offsets(uint32_t n, const uint32_t *d_indeg, uint32_t width, uint32_t *d_voff, void *d_scratch,
                      size_t scratch_bytes, void *stream) {
    WG_REQUIRE(d_voff && (d_indeg || n == 0) && width >= 1, "null argument");
    cudaStream_t s = as_stream(stream);
    cub::CountingInputIterator<uint64_t> it(0);
    cub::TransformInputIterator<uint32_t, VectorsOf, cub::CountingInputIterator<uint64_t>> in(
        it, VectorsOf{d_indeg, n, width});
    size_t tb = 0;
    WG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, d_voff, (int64_t)n + 1, s));
    WG_REQUIRE(d_scratch && scratch_bytes >= tb, "scratch too small (wg_vector_offsets_scratch_bytes)");
    WG_CUDA(cub::DeviceScan::ExclusiveSum(d_scratch, tb, in, d_voff, (int64_t)n + 1, s));
    return WG_OK;
}

size_t wg_expand_scratch_bytes(uint64_t nvec) {
    size_t tb = 0;
    cub::DeviceScan::InclusiveScan(nullptr, tb, (uint32_t *)nullptr, (uint32_t *)nullptr, cub::Max(),
                                   (int64_t)(nvec ? nvec : 1));
    return tb + 256;
}

int wg_expand_destinations(uint32_t n, const uint32_t *d_voff, uint64_t nvec, uint32_t *d_vdst, void *d_scratch,
                           size_t scratch_bytes, void *stream) {
    WG_REQUIRE(d_voff && (d_vdst || nvec == 0), "null argument");
    cudaStream_t s = as_stream(stream);
    if (nvec == 0 || n == 0) return WG_OK;
    size_t tb = 0;
    WG_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, d_vdst, d_vdst, cub::Max(), (int64_t)nvec, s));
    WG_REQUIRE(d_scratch && scratch_bytes >= tb, "scratch too small (wg_expand_scratch_bytes)");
    WG_CUDA(cudaMemsetAsync(d_vdst, 0, nvec * 4, s));
    mark_run_heads<<<grid_1d(n), 256, 0, s>>>(n, d_voff, d_vdst); ::wg::count_launch();
    WG_CHECK_LAUNCH("mark_run_heads");
    WG_CUDA(cub::DeviceScan::InclusiveScan(d_scratch, tb, d_vdst, d_vdst, cub::Max(), (int64_t)nvec, s));
    return WG_OK;
}

}  // extern "C"

// ===================================================================== K9 ==
// Input generators.
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

// PCG64 (numpy's PCG64: 128-bit LCG, XSL-RR output, step-then-output).
__device__ __forceinline__ uint64_t pcg_out(u128 st) {
    uint64_t x = (uint64_t)(st >> 64) ^ (uint64_t)st;
    unsigned rot = (unsigned)(st >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

__device__ u128 pcg_advance(u128 state, u128 inc, u128 mult, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = mult, cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

constexpr int RMAT_EPT = 64;  // edges per thread

__global__ void rmat_kernel(uint32_t scale, uint64_t m, uint64_t shi, uint64_t slo, uint64_t ihi,
                            uint64_t ilo, double t1, double t2, double t3, uint32_t *src,
                            uint32_t *dst) {
    const u128 mult = mk128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull);
    const u128 inc = mk128(ihi, ilo);
    for (uint64_t chunk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; chunk * RMAT_EPT < m;
         chunk += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t e0 = chunk * RMAT_EPT;
        uint64_t e1 = e0 + RMAT_EPT < m ? e0 + RMAT_EPT : m;
        u128 st = pcg_advance(mk128(shi, slo), inc, mult, e0 * scale);
        for (uint64_t e = e0; e < e1; ++e) {
            uint32_t s = 0, d = 0;
            for (uint32_t level = 0; level < scale; ++level) {
                st = st * mult + inc;
                double r = (double)(pcg_out(st) >> 11) * (1.0 / 9007199254740992.0);
                uint32_t q = (r >= t1) + (r >= t2) + (r >= t3);
                uint32_t sh = scale - 1 - level;
                s |= (q >> 1) << sh;
                d |= (q & 1) << sh;
            }
            src[e] = s;
            dst[e] = d;
        }
    }
}

__global__ void edge_keys(uint64_t m, const uint32_t *src, const uint32_t *dst, int drop_loops,
                          int sym, uint64_t *keys, unsigned long long *count) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = src[e], d = dst[e];
        bool loop = s == d;
        bool keep = !(drop_loops && loop);
        bool rev = keep && sym && !loop;
        unsigned want = (keep ? 1u : 0u) + (rev ? 1u : 0u);
        unsigned mask = __activemask();
        // warp-aggregated slot reservation
        unsigned incl = want;
        for (int off = 1; off < 32; off <<= 1) {
            unsigned o = __shfl_up_sync(mask, incl, off);
            if ((int)(threadIdx.x & 31) >= off) incl += o;
        }
        // active lanes form a prefix of the warp (grid-stride tail)
        const int leader = 31 - __clz(mask);
        unsigned total = __shfl_sync(mask, incl, leader);
        unsigned long long base = 0;
        if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(count, (unsigned long long)total);
        base = __shfl_sync(mask, base, leader);
        uint64_t pos = base + incl - want;
        if (keep) keys[pos++] = ((uint64_t)s << 32) | d;
        if (rev) keys[pos] = ((uint64_t)d << 32) | s;
    }
}

__global__ void split_keys(uint64_t m, const uint64_t *keys, uint32_t *src, uint32_t *dst) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        src[e] = (uint32_t)(keys[e] >> 32);
        dst[e] = (uint32_t)keys[e];
    }
}

__global__ void weights_kernel(uint64_t m, const uint32_t *src, const uint32_t *dst, uint32_t maxw,
                               uint32_t *w) {
    const uint64_t K = 0x9E3779B97F4A7C15ull;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = (((uint64_t)src[e] * K) ^ (uint64_t)dst[e]) * K;
        w[e] = 1u + (uint32_t)((h >> 48) % maxw);
    }
}

__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t u) {
    uint64_t z = seed ^ (u * 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void grid_kernel(uint32_t rows, uint32_t cols, uint64_t seed, uint32_t keep_ppm,
                            uint32_t maxw, uint32_t *src, uint32_t *dst, uint32_t *w,
                            unsigned long long *count) {
    uint64_t H = (uint64_t)rows * (cols - 1), V = (uint64_t)(rows - 1) * cols;
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < H + V;
         u += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a, b;
        if (u < H) {
            uint64_t r = u / (cols - 1), c = u % (cols - 1);
            a = (uint32_t)(r * cols + c);
            b = a + 1;
        } else {
            uint64_t v = u - H;
            a = (uint32_t)v;
            b = (uint32_t)(v + cols);
        }
        uint64_t h = mix64(seed, u);
        if ((uint32_t)(h % 1000000ull) >= keep_ppm) continue;
        uint32_t wt = 1u + (uint32_t)((h >> 32) % maxw);
        unsigned long long pos = atomicAdd(count, 2ull);
        src[pos] = a; dst[pos] = b; w[pos] = wt;
        src[pos + 1] = b; dst[pos + 1] = a; w[pos + 1] = wt;
    }
}

}  // namespace

extern "C" {

int wg_rmat_edges(uint32_t scale, uint64_t m, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                  uint64_t inc_lo, const double *h_thresholds3, uint32_t *d_src, uint32_t *d_dst,
                  void *stream) {
    WG_REQUIRE(scale >= 1 && scale <= 31, "scale must be in [1, 31]");
    WG_REQUIRE(h_thresholds3 && d_src && d_dst, "null argument");
    if (m == 0) return WG_OK;
    cudaStream_t s = as_stream(stream);
    uint64_t chunks = (m + RMAT_EPT - 1) / RMAT_EPT;
    unsigned grid = grid_for(chunks, 256, 8);
    rmat_kernel<<<grid, 256, 0, s>>>(scale, m, state_hi, state_lo, inc_hi, inc_lo, h_thresholds3[0],
                                     h_thresholds3[1], h_thresholds3[2], d_src, d_dst); ::wg::count_launch();
    WG_CHECK_LAUNCH("rmat");
    return WG_OK;
}

size_t wg_canonical_scratch_bytes(uint64_t m) {
    uint64_t mm = 2 * (m ? m : 1);
    size_t a = 0, b = 0;
    cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
    cub::DeviceRadixSort::SortKeys(nullptr, a, kb, (int64_t)mm, 0, 64);
    cub::DeviceSelect::Unique(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr,
                              (uint64_t *)nullptr, (int64_t)mm);
    return 2 * carve_size(mm * 8) + carve_size(64) + carve_size(a > b ? a : b) + 1024;
}

int wg_canonical_edges(uint64_t m, uint32_t *d_src, uint32_t *d_dst, int drop_loops, int symmetrize,
                       void *d_scratch, size_t scratch_bytes, uint64_t *h_m_out, void *stream) {
    WG_REQUIRE(h_m_out, "null argument");
    *h_m_out = 0;
    if (m == 0) return WG_OK;
    WG_REQUIRE(d_src && d_dst && d_scratch, "null argument");
    cudaStream_t s = as_stream(stream);
    uint64_t mm = 2 * m;
    Carve cv{(char *)d_scratch, 0, scratch_bytes};
    uint64_t *k0 = cv.take<uint64_t>(mm), *k1 = cv.take<uint64_t>(mm);
    unsigned long long *cnt = cv.take<unsigned long long>(8);
    size_t a = 0, b = 0;
    {
        cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
        cub::DeviceRadixSort::SortKeys(nullptr, a, kb, (int64_t)mm, 0, 64);
        cub::DeviceSelect::Unique(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (uint64_t *)nullptr, (int64_t)mm);
    }
    size_t tb = a > b ? a : b;
    void *temp = cv.take<char>(tb);
    if (!temp) {
        set_error("canonical scratch too small");
        return WG_ENOSPACE;
    }
    WG_CUDA(cudaMemsetAsync(cnt, 0, 64, s));
    edge_keys<<<grid_for(m, 256 * 8, 16), 256, 0, s>>>(m, d_src, d_dst, drop_loops, symmetrize, k0, cnt); ::wg::count_launch();
    WG_CHECK_LAUNCH("edge_keys");
    unsigned long long k = 0;
    WG_CUDA(cudaMemcpyAsync(&k, cnt, 8, cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    cub::DoubleBuffer<uint64_t> kb(k0, k1);
    size_t t = tb;
    WG_CUDA(cub::DeviceRadixSort::SortKeys(temp, t, kb, (int64_t)k, 0, 64, s));
    t = tb;
    WG_CUDA(cub::DeviceSelect::Unique(temp, t, kb.Current(), kb.Alternate(), (uint64_t *)(cnt + 1),
                                      (int64_t)k, s));
    unsigned long long u = 0;
    WG_CUDA(cudaMemcpyAsync(&u, cnt + 1, 8, cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    WG_REQUIRE(u <= (symmetrize ? 2 * m : m), "internal: unique count");
    split_keys<<<grid_for(u, 256 * 8, 16), 256, 0, s>>>(u, kb.Alternate(), d_src, d_dst); ::wg::count_launch();
    WG_CHECK_LAUNCH("split_keys");
    WG_CUDA(cudaStreamSynchronize(s));
    *h_m_out = u;
    return WG_OK;
}

int wg_weights_hash(uint64_t m, const uint32_t *d_src, const uint32_t *d_dst, uint32_t max_weight,
                    uint32_t *d_w, void *stream) {
    WG_REQUIRE(max_weight >= 1, "max_weight must be >= 1");
    if (m == 0) return WG_OK;
    WG_REQUIRE(d_src && d_dst && d_w, "null argument");
    weights_kernel<<<grid_for(m, 256 * 8, 16), 256, 0, as_stream(stream)>>>(m, d_src, d_dst,
                                                                           max_weight, d_w); ::wg::count_launch();
    WG_CHECK_LAUNCH("weights");
    return WG_OK;
}

int wg_grid_edges(uint32_t rows, uint32_t cols, uint64_t seed, uint32_t keep_per_million,
                  uint32_t max_weight, uint32_t *d_src, uint32_t *d_dst, uint32_t *d_w,
                  uint64_t *d_counter, uint64_t *h_m_out, void *stream) {
    WG_REQUIRE(rows >= 1 && cols >= 1 && max_weight >= 1, "bad grid arguments");
    WG_REQUIRE(d_src && d_dst && d_w && d_counter && h_m_out, "null argument");
    cudaStream_t s = as_stream(stream);
    WG_CUDA(cudaMemsetAsync(d_counter, 0, 8, s));
    uint64_t und = (uint64_t)rows * (cols - 1) + (uint64_t)(rows - 1) * cols;
    if (und) {
        grid_kernel<<<grid_for(und, 256 * 8, 16), 256, 0, s>>>(
            rows, cols, seed, keep_per_million, max_weight, d_src, d_dst, d_w,
            (unsigned long long *)d_counter); ::wg::count_launch();
        WG_CHECK_LAUNCH("grid");
    }
    WG_CUDA(cudaMemcpyAsync(h_m_out, d_counter, 8, cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    return WG_OK;
}

}  // extern "C"

namespace {
// voff[d] = lower bound of d in the sorted vdst (destination runs, graph.py:235)
__global__ void voff_from_dst_kernel(uint32_t n, uint64_t nvec, const uint32_t *vdst, uint32_t *voff) {
    for (uint64_t d = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; d <= n;
         d += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = nvec;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (vdst[mid] < d) lo = mid + 1;
            else hi = mid;
        }
        voff[d] = (uint32_t)lo;
    }
}
}  // namespace

extern "C" int wg_vector_offsets_from_dst(const wg_graph *g, uint32_t *d_voff, void *stream) {
    WG_REQUIRE(g && d_voff, "null argument");
    WG_REQUIRE(g->nvec < (1ull << 32), "more than 2^32 vectors");
    WG_REQUIRE(g->nvec == 0 || g->vdst, "null vdst");
    cudaStream_t s = as_stream(stream);
    voff_from_dst_kernel<<<grid_for((uint64_t)g->n + 1, 256, 8), 256, 0, s>>>(g->n, g->nvec, g->vdst, d_voff);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("voff_from_dst");
    return WG_OK;
}

namespace {
__global__ void first_lanes_kernel(uint32_t n, uint32_t width, const uint32_t *voff, const uint32_t *vsrc,
                                   uint32_t *vfirst) {
    for (uint64_t d = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; d < n; d += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v0 = voff[d], v1 = voff[d + 1];
        vfirst[d] = v1 > v0 ? vsrc[(uint64_t)v0 * width] : WG_NO_LANE;
    }
}
}  // namespace

extern "C" int wg_first_lanes(const wg_graph *g, const uint32_t *d_voff, uint32_t *d_vfirst, void *stream) {
    WG_REQUIRE(g && d_voff && d_vfirst, "null argument");
    WG_REQUIRE(g->nvec == 0 || g->vsrc, "null vsrc");
    cudaStream_t s = as_stream(stream);
    if (g->n == 0) return WG_OK;
    first_lanes_kernel<<<grid_for(g->n, 256, 8), 256, 0, s>>>(g->n, g->width, d_voff, g->vsrc, d_vfirst);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("first_lanes");
    return WG_OK;
}
