// codec.cu — delta-coded lane sources, the compact host format of the e2e
// upload (wedge_b200.h "Delta-coded lanes").
//
// The pull layout stores each destination's in-neighbours ascending over
// consecutive W-lane vectors (graph.py:220-263: lexsort by (dst, src)), so a
// lane is coded as the gap to the lane before it in the same destination:
//   code = 0                       empty lane (WG_NO_LANE)
//        = src + 1                 first lane of a destination, or of a block
//        = src - prev_src + 1      otherwise (prev_src = the lane before)
// Each vector stores its W codes in width[v] = max bit length bits (width - 1
// kept in 5 bits per vector, block-aligned: WWORDS words per block), the
// vectors of a block of WG_CODED_BLOCK_VECTORS back to back; blocks start on
// a 32-bit word (block_base[b] = first bit, block_base[nblocks] = total), so
// runs of blocks can be copied and decoded independently.  At s22 this is
// ~260 MB (stream + width bytes + voff) against 531 MB of uint32 lanes.
//
// Decoding is one CTA per block: a block scan of the vector widths gives
// every vector's bit offset, each thread extracts the codes of VPT vectors
// and a block-wide segmented sum over destinations (heads from vec_dst,
// rebuilt from voff first) turns gaps back into sources.
#include <cub/cub.cuh>

#include "common.cuh"

using namespace wg;

namespace {

constexpr int BV = WG_CODED_BLOCK_VECTORS;
constexpr int CT = 256;       // threads per block
constexpr int VPT = BV / CT;  // vectors per thread
static_assert(BV % CT == 0, "block size");
constexpr int WBITS = 5;                  // a vector's width - 1 in 5 bits
constexpr int WWORDS = BV * WBITS / 32;  // width words per block (block-aligned)
static_assert(VPT == 4, "a thread's widths are one 20-bit field");

// the 20-bit field of the VPT widths of thread t's vectors in block b
__device__ __forceinline__ uint32_t width_field(const uint32_t *wp, uint64_t b, unsigned t) {
    const uint32_t bit = t * (VPT * WBITS);
    const uint32_t *w = wp + b * WWORDS + (bit >> 5);
    const uint32_t sh = bit & 31;
    uint64_t x = w[0];
    if (sh + VPT * WBITS > 32) x |= (uint64_t)w[1] << 32;
    return (uint32_t)(x >> sh) & ((1u << (VPT * WBITS)) - 1u);
}

__device__ __forceinline__ uint32_t bitlen(uint32_t x) { return x ? 32u - __clz(x) : 0u; }

__device__ __forceinline__ bool dest_head(const uint32_t *vdst, uint64_t v) {
    return (v % BV) == 0 || vdst[v] != vdst[v - 1];
}

// codes of vector v (W lanes); sets *bad when a destination is not ascending
template <int W>
__device__ __forceinline__ uint32_t vector_codes(const uint32_t *vsrc, const uint32_t *vdst, uint64_t v,
                                                 uint32_t (&code)[W], unsigned *bad) {
    uint32_t prev = dest_head(vdst, v) ? WG_NO_LANE : vsrc[v * W - 1];
    if (!dest_head(vdst, v) && prev == WG_NO_LANE) atomicOr(bad, 1u);  // partial inner vector
    uint32_t wmax = 1;
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const uint32_t s = vsrc[v * W + j];
        uint32_t c;
        if (s == WG_NO_LANE) {
            c = 0;
        } else if (prev == WG_NO_LANE) {
            c = s + 1;
        } else {
            if (s < prev) atomicOr(bad, 1u);
            c = s - prev + 1;
        }
        if (s != WG_NO_LANE) prev = s;
        code[j] = c;
        wmax = max(wmax, bitlen(c));
    }
    return wmax;
}

template <int W>
__global__ void __launch_bounds__(CT) encode_widths(uint64_t nvec, const uint32_t *vsrc, const uint32_t *vdst,
                                                    uint32_t *widths, uint64_t *block_bits, unsigned *bad) {
    using Reduce = cub::BlockReduce<uint64_t, CT>;
    __shared__ typename Reduce::TempStorage tmp;
    const uint64_t b = blockIdx.x;
    uint64_t bits = 0;
    uint32_t field = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const uint64_t v = b * BV + (uint64_t)threadIdx.x * VPT + k;
        if (v < nvec) {
            uint32_t code[W];
            const uint32_t w = vector_codes<W>(vsrc, vdst, v, code, bad);
            field |= (w - 1) << (k * WBITS);
            bits += (uint64_t)W * w;
        }
    }
    if (field) {  // zeroed before: OR the 20-bit field in (it may straddle two words)
        const uint32_t bit = threadIdx.x * (VPT * WBITS), sh = bit & 31;
        uint32_t *w = widths + b * WWORDS + (bit >> 5);
        atomicOr(&w[0], field << sh);
        if (sh + VPT * WBITS > 32) atomicOr(&w[1], field >> (32 - sh));
    }
    const uint64_t tot = Reduce(tmp).Sum(bits);
    if (threadIdx.x == 0) block_bits[b] = (tot + 31) & ~uint64_t(31);
}

template <int W>
__global__ void __launch_bounds__(CT) encode_fields(uint64_t nvec, const uint32_t *vsrc, const uint32_t *vdst,
                                                    const uint32_t *widths, const uint64_t *block_base,
                                                    uint32_t *stream, unsigned *bad) {
    using Scan = cub::BlockScan<uint64_t, CT>;
    __shared__ typename Scan::TempStorage tmp;
    const uint64_t b = blockIdx.x;
    const uint64_t v0 = b * BV + (uint64_t)threadIdx.x * VPT;
    uint64_t bits = 0;
    const uint32_t field = width_field(widths, b, threadIdx.x);
#pragma unroll
    for (int k = 0; k < VPT; ++k)
        if (v0 + k < nvec) bits += (uint64_t)W * (((field >> (k * WBITS)) & 31u) + 1);
    uint64_t off;
    Scan(tmp).ExclusiveSum(bits, off);
    off += block_base[b];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const uint64_t v = v0 + k;
        if (v >= nvec) break;
        uint32_t code[W];
        vector_codes<W>(vsrc, vdst, v, code, bad);
        const uint32_t w = ((field >> (k * WBITS)) & 31u) + 1;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const uint64_t pos = off + (uint64_t)j * w;
            const uint32_t sh = (uint32_t)(pos & 31);
            if (code[j]) {
                atomicOr(&stream[pos >> 5], code[j] << sh);
                if (sh + w > 32) atomicOr(&stream[(pos >> 5) + 1], code[j] >> (32 - sh));
            }
        }
        off += (uint64_t)W * w;
    }
}

struct Seg {
    uint32_t head, x;
};
struct SegSum {
    __device__ __forceinline__ Seg operator()(const Seg &a, const Seg &b) const {
        return Seg{a.head | b.head, b.head ? b.x : a.x + b.x};
    }
};

template <int W>
__global__ void __launch_bounds__(CT) decode_lanes(uint64_t nvec, const uint32_t *vdst, const uint32_t *stream,
                                                   const uint32_t *widths, const uint64_t *block_base,
                                                   uint64_t block0, uint32_t *vsrc, uint32_t *keys,
                                                   uint32_t *vals, uint32_t pad, const uint64_t *ioff,
                                                   const uint32_t *deg, uint32_t *fill, uint32_t *pos,
                                                   unsigned *bad, uint64_t cap) {
    using Scan = cub::BlockScan<uint64_t, CT>;
    using SScan = cub::BlockScan<Seg, CT>;
    __shared__ union {
        typename Scan::TempStorage off;
        typename SScan::TempStorage seg;
    } tmp;
    const uint64_t b = block0 + blockIdx.x;
    const uint64_t v0 = b * BV + (uint64_t)threadIdx.x * VPT;
    uint32_t w[VPT];
    uint64_t bits = 0;
    const uint32_t field = width_field(widths, b, threadIdx.x);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        w[k] = v0 + k < nvec ? ((field >> (k * WBITS)) & 31u) + 1 : 0u;
        bits += (uint64_t)W * w[k];
    }
    uint64_t off;
    Scan(tmp.off).ExclusiveSum(bits, off);
    off += block_base[b];
    Seg item[VPT * W];
    bool real[VPT * W];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const uint64_t v = v0 + k;
        const bool live = v < nvec;
        const uint32_t mask = w[k] >= 32 ? 0xffffffffu : (1u << w[k]) - 1u;
        const uint32_t head = live && dest_head(vdst, v);
#pragma unroll
        for (int j = 0; j < W; ++j) {
            uint32_t c = 0;
            if (live) {
                const uint64_t pos = off + (uint64_t)j * w[k];
                const uint32_t sh = (uint32_t)(pos & 31);
                uint64_t x = stream[pos >> 5];
                if (sh + w[k] > 32) x |= (uint64_t)stream[(pos >> 5) + 1] << 32;
                c = (uint32_t)(x >> sh) & mask;
            }
            real[k * W + j] = c != 0;
            item[k * W + j] = Seg{j == 0 ? head : 0u, c ? c - 1 : 0u};
        }
        off += (uint64_t)W * w[k];
    }
    __syncthreads();  // tmp reuse
    SScan(tmp.seg).InclusiveScan(item, item, SegSum());
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const uint64_t v = v0 + k;
        if (v >= nvec) break;
#pragma unroll
        for (int j = 0; j < W; ++j) vsrc[v * W + j] = real[k * W + j] ? item[k * W + j].x : WG_NO_LANE;
        if (keys) {  // (source, vector) pairs of the chunked index build, chunk-relative
            const uint64_t l0 = (v - block0 * BV) * W;
#pragma unroll
            for (int j = 0; j < W; ++j) {
                keys[l0 + j] = real[k * W + j] ? item[k * W + j].x : pad;
                vals[l0 + j] = (uint32_t)v;
            }
        }
    }
    if (pos) {  // placed index: every lane takes its slot (warp-uniform loops)
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const uint32_t src = item[k * W + j].x;
                bool live = v0 + k < nvec && real[k * W + j];
                if (live && j > 0 && real[k * W + j - 1] && item[k * W + j - 1].x == src) {
                    *bad = 1u;  // repeated (source, vector) pair
                    live = false;
                }
                place_one(src, live, (uint32_t)(v0 + k), ioff, deg, fill, pos, bad, cap);
            }
        }
    }
}

template <int W>
int encode_w(const wg_graph *g, uint32_t *d_stream, uint32_t *d_widths, uint64_t *d_block_base, void *d_scratch,
             size_t scratch_bytes, uint64_t *h_words, cudaStream_t s) {
    const uint64_t nb = wg_coded_blocks(g->nvec);
    Carve c{(char *)d_scratch, 0, scratch_bytes};
    uint64_t *bb = c.take<uint64_t>(nb + 1);
    unsigned *bad = c.take<unsigned>(1);
    size_t tb = 0;
    WG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, bb, d_block_base, (int64_t)(nb + 1), s));
    void *temp = c.take<char>(tb);
    WG_REQUIRE(bb && bad && temp, "codec scratch too small");
    WG_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), s));
    WG_CUDA(cudaMemsetAsync(bb + nb, 0, sizeof(uint64_t), s));
    WG_CUDA(cudaMemsetAsync(d_stream, 0, wg_coded_max_words(g->nvec, g->width) * 4, s));
    WG_CUDA(cudaMemsetAsync(d_widths, 0, wg_coded_width_words(g->nvec) * 4, s));
    if (nb) {
        encode_widths<W><<<(unsigned)nb, CT, 0, s>>>(g->nvec, g->vsrc, g->vdst, d_widths, bb, bad);
        ::wg::count_launch();
    }
    WG_CUDA(cub::DeviceScan::ExclusiveSum(temp, tb, bb, d_block_base, (int64_t)(nb + 1), s));
    if (nb) {
        encode_fields<W><<<(unsigned)nb, CT, 0, s>>>(g->nvec, g->vsrc, g->vdst, d_widths, d_block_base, d_stream,
                                                      bad);
        ::wg::count_launch();
    }
    WG_CHECK_LAUNCH("encode_lanes");
    uint64_t total = 0;
    unsigned hbad = 0;
    WG_CUDA(cudaMemcpyAsync(&total, d_block_base + nb, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    WG_REQUIRE(!hbad, "lane sources are not ascending within a destination (not a pull layout)");
    *h_words = total / 32;
    return WG_OK;
}

}  // namespace

namespace wg {
int launch_decode_lanes(uint64_t nvec, uint32_t width, const uint32_t *vdst, const uint32_t *stream,
                        const uint32_t *widths, const uint64_t *block_base, uint64_t b0, uint64_t b1, uint32_t *vsrc,
                        uint32_t *keys, uint32_t *vals, uint32_t pad, cudaStream_t s) {
    if (b1 == b0) return WG_OK;
    const unsigned grid = (unsigned)(b1 - b0);
    switch (width) {
        case 1: decode_lanes<1><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, keys, vals, pad, nullptr, nullptr, nullptr, nullptr, nullptr, 0); break;
        case 2: decode_lanes<2><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, keys, vals, pad, nullptr, nullptr, nullptr, nullptr, nullptr, 0); break;
        case 4: decode_lanes<4><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, keys, vals, pad, nullptr, nullptr, nullptr, nullptr, nullptr, 0); break;
        case 8: decode_lanes<8><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, keys, vals, pad, nullptr, nullptr, nullptr, nullptr, nullptr, 0); break;
        default: WG_REQUIRE(false, "unsupported width %u", width);
    }
    ::wg::count_launch();
    WG_CHECK_LAUNCH("decode_lanes");
    return WG_OK;
}
int launch_decode_place(uint64_t nvec, uint32_t width, const uint32_t *vdst, const uint32_t *stream,
                        const uint32_t *widths, const uint64_t *block_base, uint64_t b0, uint64_t b1, uint32_t *vsrc,
                        const uint64_t *off, const uint32_t *deg, uint32_t *fill, uint32_t *pos, unsigned *bad,
                        uint64_t cap, cudaStream_t s) {
    if (b1 == b0) return WG_OK;
    const unsigned grid = (unsigned)(b1 - b0);
    switch (width) {
        case 1: decode_lanes<1><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, nullptr, nullptr, 0u, off, deg, fill, pos, bad, cap); break;
        case 2: decode_lanes<2><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, nullptr, nullptr, 0u, off, deg, fill, pos, bad, cap); break;
        case 4: decode_lanes<4><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, nullptr, nullptr, 0u, off, deg, fill, pos, bad, cap); break;
        case 8: decode_lanes<8><<<grid, CT, 0, s>>>(nvec, vdst, stream, widths, block_base, b0, vsrc, nullptr, nullptr, 0u, off, deg, fill, pos, bad, cap); break;
        default: WG_REQUIRE(false, "unsupported width %u", width);
    }
    ::wg::count_launch();
    WG_CHECK_LAUNCH("decode_lanes");
    return WG_OK;
}
}  // namespace wg

extern "C" {

uint64_t wg_coded_blocks(uint64_t nvec) { return (nvec + BV - 1) / BV; }

uint64_t wg_coded_width_words(uint64_t nvec) { return wg_coded_blocks(nvec) * WWORDS; }

uint64_t wg_coded_max_words(uint64_t nvec, uint32_t width) { return nvec * width + wg_coded_blocks(nvec) + 1; }

size_t wg_coded_scratch_bytes(uint64_t nvec) {
    const uint64_t nb = wg_coded_blocks(nvec);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (uint64_t *)nullptr, (uint64_t *)nullptr, (int64_t)(nb + 1));
    return carve_size((nb + 1) * 8) + carve_size(4) + carve_size(tb) + 256;
}

int wg_encode_lanes(const wg_graph *g, uint32_t *d_stream, uint32_t *d_widths, uint64_t *d_block_base,
                    void *d_scratch, size_t scratch_bytes, uint64_t *h_words, void *stream) {
    WG_REQUIRE(g && d_stream && d_block_base && d_scratch && h_words, "null argument");
    WG_REQUIRE(g->nvec == 0 || (g->vsrc && g->vdst && d_widths), "null argument");
    cudaStream_t s = as_stream(stream);
    switch (g->width) {
        case 1: return encode_w<1>(g, d_stream, d_widths, d_block_base, d_scratch, scratch_bytes, h_words, s);
        case 2: return encode_w<2>(g, d_stream, d_widths, d_block_base, d_scratch, scratch_bytes, h_words, s);
        case 4: return encode_w<4>(g, d_stream, d_widths, d_block_base, d_scratch, scratch_bytes, h_words, s);
        case 8: return encode_w<8>(g, d_stream, d_widths, d_block_base, d_scratch, scratch_bytes, h_words, s);
    }
    WG_REQUIRE(false, "unsupported width %u", g->width);
}

int wg_decode_lanes(uint64_t nvec, uint32_t width, const uint32_t *d_vdst, const uint32_t *d_stream,
                    const uint32_t *d_widths, const uint64_t *d_block_base, uint64_t block_begin,
                    uint64_t block_end, uint32_t *d_vsrc, void *stream) {
    WG_REQUIRE(block_begin <= block_end && block_end <= wg_coded_blocks(nvec), "bad block range");
    if (block_end == block_begin) return WG_OK;
    WG_REQUIRE(d_vdst && d_stream && d_widths && d_block_base && d_vsrc, "null argument");
    return launch_decode_lanes(nvec, width, d_vdst, d_stream, d_widths, d_block_base, block_begin, block_end, d_vsrc,
                               nullptr, nullptr, 0u, as_stream(stream));
}

}  // extern "C"
