// pagerank.cu — dense PageRank pull (K8), deterministic.  No reference
// implementation exists (pkg/tests/test_apps.py:167-169);
// semantics follow BASELINE.json config 5: float32 ranks, damping d, fixed
// iterations, dangling mass redistributed uniformly:
//   r0 = 1/N;  r'(v) = (1-d)/N + d * (sum_{u->v} r(u)/outdeg(u) + D/N),
//   D = sum of r(u) over outdeg(u) = 0.
//
// Bit-reproducible by construction: no float atomics.
//  * pull: every warp walks its own contiguous range of 32-vector tiles in
//    order with a carried segment (the min-plus tile body with a float
//    segmented SUM), so a destination is summed in one fixed order and
//    written with a plain store -- except a destination whose vectors cross
//    a warp-range boundary: each warp records its first and last segment's
//    partial sum, and pr_fixup adds them in warp order.
//  * dangling mass: per-block double partials in fixed slots, summed in slot
//    order by one warp (pr_dangling).
// An iteration is prep (V-sized: apply of the previous sums + contributions)
// -> dangling sum -> pull (E-sized) -> fixup.  The fixed order depends only
// on the launch configuration (grid sizes from the occupancy query), so runs
// on the same GPU and build are bit-identical.
#include <cub/cub.cuh>

#include "common.cuh"
#include "tma.cuh"  // warp_range

using namespace wg;

namespace {

constexpr unsigned PR_THREADS = 256;
constexpr uint32_t PR_NONE = 0xffffffffu;

// Per-warp boundary record of the pull: the first segment when it continues
// a destination from the previous range, the last when it continues into
// the next; `single`: the whole range is one destination (a middle piece).
struct PrBound {
    uint32_t hd, td;  // destinations (PR_NONE: that end is complete)
    float hs, ts;
    uint32_t single, pad;
};

unsigned prep_grid(uint32_t n) { return grid_for(n, PR_THREADS * 4, 8); }

// prep(it): r = it ? base(D_{it-1}) + d*acc : 1/N; contrib = r/outdeg; the
// block's dangling mass of r into dpart[block].  ZERO: also acc = 0 (callers
// whose pull does not rewrite every destination's sum: the sharded path's
// gathered sum vector); wg_pagerank's own pull writes every vertex of its
// range, in-degree 0 included (pr_pull's gap fill), so nothing is cleared.
// Four vertices per thread and round trip (128-bit loads / stores).
template <bool ZERO>
__global__ void __launch_bounds__(PR_THREADS) pr_prep(uint32_t n, int it, double damping,
                                                      const uint32_t *__restrict__ outdeg, float *__restrict__ acc,
                                                      float *__restrict__ contrib, float *__restrict__ rank_out,
                                                      const double *__restrict__ scal, double *__restrict__ dpart) {
    __shared__ double sm[33];
    double dang = 0.0;
    const float base = it ? (float)((1.0 - damping) / n + damping * scal[0] / n) : 0.f;
    const float df = (float)damping;
    const float r0 = (float)(1.0 / n);
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    const auto one = [&](float a, uint32_t od, float &c) -> float {
        const float r = it ? base + df * a : r0;
        if (od) {
            c = r / (float)od;
        } else {
            c = 0.f;
            dang += r;
        }
        return r;
    };
    const bool aligned = (((uintptr_t)outdeg | (uintptr_t)acc | (uintptr_t)contrib | (uintptr_t)rank_out) & 15u) == 0;
    const uint64_t quads = aligned ? n >> 2 : 0;
    for (uint64_t q = tid; q < quads; q += nth) {
        const uint4 od = reinterpret_cast<const uint4 *>(outdeg)[q];
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (it) a = reinterpret_cast<const float4 *>(acc)[q];
        float4 c, r;
        r.x = one(a.x, od.x, c.x);
        r.y = one(a.y, od.y, c.y);
        r.z = one(a.z, od.z, c.z);
        r.w = one(a.w, od.w, c.w);
        if (ZERO) reinterpret_cast<float4 *>(acc)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4 *>(contrib)[q] = c;
        if (rank_out) reinterpret_cast<float4 *>(rank_out)[q] = r;
    }
    for (uint64_t v = (quads << 2) + tid; v < n; v += nth) {
        float c;
        const float r = one(it ? acc[v] : 0.f, outdeg[v], c);
        if (ZERO) acc[v] = 0.f;
        contrib[v] = c;
        if (rank_out) rank_out[v] = r;
    }
    const double tot = block_sum(dang, sm);
    if (threadIdx.x == 0) dpart[blockIdx.x] = tot;
}

// D = sum of the block partials in slot order (one warp, fixed tree).
__global__ void pr_dangling(const double *dpart, unsigned nparts, double *scal) {
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < nparts; i += 32) s += dpart[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (threadIdx.x == 0) scal[0] = s;
}

template <int W, bool SHIFT>
__global__ void __launch_bounds__(PR_THREADS) pr_pull(wg_graph g, const float *__restrict__ contrib, float *acc,
                                                      uint32_t base_, PrBound *bounds) {
    const uint32_t base = SHIFT ? base_ : 0u;  // destination-sharded runs index a slice
    const unsigned lane = lane_id();
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nvec = g.nvec;
    uint64_t t0, t1;
    warp_range((nvec + 31) >> 5, gwarp, nwarps, t0, t1);
    PrBound rec{PR_NONE, PR_NONE, 0.f, 0.f, 0u, 0u};
    if (t0 < t1) {
        const uint64_t p_lo = t0 << 5, p_hi = (t1 << 5) < nvec ? (t1 << 5) : nvec;
        // destinations just outside the range: a segment touching them is shared
        const uint32_t dleft = p_lo > 0 ? g.vdst[p_lo - 1] : PR_NONE;
        const uint32_t dright = p_hi < nvec ? g.vdst[p_hi] : PR_NONE;
        uint32_t cd = PR_NONE;  // carried segment (warp-uniform): destination,
        float cs = 0.f;         // partial sum, and whether it is the range's
        bool cfirst = false;    // first segment
        // the next tile's lanes and destination are loaded while this tile
        // gathers: one memory latency per tile on the warp's critical path
        // instead of two (stream, then the dependent gathers)
        uint32_t src_n[W], d_n = PR_NONE;
#pragma unroll
        for (int l = 0; l < W; ++l) src_n[l] = WG_NO_LANE;
        const auto fetch = [&](uint64_t tile) {
            const uint64_t q = (tile << 5) + lane;
            if (q < nvec) {
                d_n = ld_stream(g.vdst + q);
                load_lanes<W>(g.vsrc, q, src_n);
            } else {
                d_n = PR_NONE;
            }
        };
        fetch(t0);
        for (uint64_t tile = t0; tile < t1; ++tile) {
            const uint64_t p = (tile << 5) + lane;
            const bool valid = p < nvec;
            const uint32_t d = d_n;
            uint32_t src[W];
#pragma unroll
            for (int l = 0; l < W; ++l) src[l] = src_n[l];
            if (tile + 1 < t1) fetch(tile + 1);
            float sum = 0.f;
            if (valid) {
#pragma unroll
                for (int l = 0; l < W; ++l)
                    if (src[l] != WG_NO_LANE) sum += contrib[src[l]];
            }
            const uint32_t dn = __shfl_down_sync(FULL, d, 1);
            const uint32_t dp = __shfl_up_sync(FULL, d, 1);
            const bool head = lane == 0 || dp != d;
            // Gap fill: the destinations between the previous vector's and this
            // one's have no in-edges -- their sum is 0.  Writing them here (by
            // the lane that opens the next destination) makes the pull write
            // its whole destination range: every 32-byte sector of acc leaves
            // L2 fully written (partially written sectors cost the ECC DRAM a
            // read-modify-write each when evicted, which made the V-sized prep
            // pass that follows 13x slower than its traffic), and prep need
            // not clear acc.
            {
                uint32_t prevd = dp;  // destination of the vector before this lane's
                bool from_start = false;
                if (lane == 0) {
                    prevd = tile == t0 ? dleft : cd;
                    from_start = tile == t0 && p_lo == 0;
                }
                // (a warp-cooperative fill of long gaps was measured: 109 vs 82 ms per
                // run -- the extra ballot per tile costs more than the rare long gap)
                if (valid && (from_start || d != prevd))
                    for (uint32_t x = from_start ? base : prevd + 1; x < d; ++x) acc[x - base] = 0.f;
            }
            const bool tail = lane == 31 || dn != d;
            const unsigned heads = __ballot_sync(FULL, head);
            const unsigned head_lane = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
            const unsigned dist = lane - head_lane;
            const unsigned maxd = __reduce_max_sync(FULL, dist);
            for (unsigned off = 1; off <= maxd; off <<= 1) {
                const float o = __shfl_up_sync(FULL, sum, off);
                if (off <= dist) sum += o;
            }
            // the carried segment ended at the previous tile's last lane: close it
            const uint32_t d0 = __shfl_sync(FULL, d, 0);
            if (cd != PR_NONE && d0 != cd) {
                if (cfirst && cd == dleft) {
                    rec.hd = cd;  // (warp-uniform)
                    rec.hs = cs;
                } else if (lane == 0) {
                    acc[cd - base] = cs;
                }
            }
            // the tile's first segment continues the carried one (earlier tiles first)
            const bool cont = head_lane == 0 && cd != PR_NONE && d == cd;
            if (cont) sum = cs + sum;
            const bool seg_first = head_lane == 0 && (cont ? cfirst : tile == t0);
            if (tail && valid && lane != 31) {  // a segment closed inside this tile
                if (seg_first && d == dleft) {  // ... continuing the previous range's last one
                    rec.hd = d;
                    rec.hs = sum;
                } else {
                    acc[d - base] = sum;
                }
            }
            // the segment touching lane 31 is carried into the next tile
            cd = __shfl_sync(FULL, d, 31);
            cs = __shfl_sync(FULL, sum, 31);
            cfirst = __shfl_sync(FULL, seg_first, 31);
        }
        // the range's last segment
        if (cd != PR_NONE) {
            const bool shared_right = cd == dright;
            const bool shared_left = cfirst && cd == dleft;
            if (shared_right) {
                rec.td = cd;
                rec.ts = cs;
                rec.single = shared_left ? 1u : 0u;  // a middle piece of one destination
            } else if (shared_left) {
                rec.hd = cd;
                rec.hs = cs;
            } else if (lane == 0) {
                acc[cd - base] = cs;
            }
        }
    }
    // one record per warp: the head piece was set by the lane that closed it
    const unsigned hl = __ballot_sync(FULL, rec.hd != PR_NONE);
    if (hl) {
        const int src = __ffs(hl) - 1;
        rec.hd = __shfl_sync(FULL, rec.hd, src);
        rec.hs = __shfl_sync(FULL, rec.hs, src);
    }
    if (lane == 0 && bounds) bounds[gwarp] = rec;
}

// Shared destinations: the warp whose range holds a destination's FIRST
// piece (its last segment continues right and is not itself a continuation)
// adds the following warps' pieces in order and stores the sum.
template <bool SHIFT>
__global__ void pr_fixup(const PrBound *bounds, uint64_t nwarps, float *acc, uint32_t base_) {
    const uint32_t base = SHIFT ? base_ : 0u;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwarps;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const PrBound r = bounds[w];
        if (r.td == PR_NONE || r.single) continue;  // no piece starts here and continues
        const uint32_t d = r.td;
        float s = r.ts;
        for (uint64_t k = w + 1; k < nwarps; ++k) {
            const PrBound q = bounds[k];
            if (q.single && q.td == d) {
                s += q.ts;  // a middle piece
                continue;
            }
            if (q.hd == d) s += q.hs;  // the destination's last piece
            break;
        }
        acc[d - base] = s;
    }
}

// ---- hot-source layout (wg_pagerank_hot_*) -------------------------------
// The pull's cost is its E random 4-byte gathers of contrib[src]: they run
// L1TEX at 80% and L2 at 70% of their sector throughput while DRAM idles
// (profiles/r02_ncu_pr_pull_*).  A source is gathered once per out-edge, and
// RMAT's heavy sources are scattered over the id space (the ids with few set
// bits), so a fetched 32-byte sector holds one hot value among cold ones.
// Here the sources are renumbered by descending out-degree (stable): slot j
// of contrib belongs to vertex order[j], the lanes of a PageRank-only copy of
// vsrc hold slots, and only the nsrc vertices that have out-edges get a slot.
// Hot values now share sectors and lines (higher L1 / L2 hit rates, fewer
// distinct lines per warp gather); lane order, and with it every float sum,
// is unchanged.
__global__ void __launch_bounds__(256) hot_keys_kernel(uint32_t n, const uint32_t *__restrict__ outdeg,
                                                       uint32_t *__restrict__ keys, uint32_t *__restrict__ ids,
                                                       unsigned long long *nsrc) {
    unsigned long long cnt = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t od = outdeg[v];
        keys[v] = ~od;  // ascending ~od = descending out-degree
        ids[v] = (uint32_t)v;
        cnt += od != 0;
    }
    cnt = warp_sum(cnt);
    if (lane_id() == 0 && cnt) atomicAdd(nsrc, cnt);
}

__global__ void __launch_bounds__(256) hot_slots_kernel(uint32_t n, const uint32_t *__restrict__ order,
                                                        const uint32_t *__restrict__ outdeg,
                                                        uint32_t *__restrict__ slot_of, uint32_t *__restrict__ od_hot) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = order[j];
        slot_of[v] = (uint32_t)j;
        od_hot[j] = outdeg[v];
    }
}

__global__ void __launch_bounds__(256) hot_lanes_kernel(uint64_t lanes, const uint32_t *__restrict__ vsrc,
                                                        const uint32_t *__restrict__ slot_of,
                                                        uint32_t *__restrict__ vsrc_hot) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lanes;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = vsrc[i];
        vsrc_hot[i] = u == WG_NO_LANE ? WG_NO_LANE : slot_of[u];
    }
}

// prep over slots: slot j < nsrc gets its contribution, the others (the
// vertices without out-edges, in id order) add their rank to the dangling
// mass.  acc is read through order[] (ascending ids within a degree class).
__global__ void __launch_bounds__(PR_THREADS) pr_prep_hot(uint32_t n, uint32_t nsrc, int it, double damping,
                                                          const uint32_t *__restrict__ order,
                                                          const uint32_t *__restrict__ od_hot,
                                                          const float *__restrict__ acc, float *__restrict__ contrib,
                                                          const double *__restrict__ scal, double *__restrict__ dpart) {
    __shared__ double sm[33];
    double dang = 0.0;
    const float base = it ? (float)((1.0 - damping) / n + damping * scal[0] / n) : 0.f;
    const float df = (float)damping;
    const float r0 = (float)(1.0 / n);
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    constexpr int U = 8;  // independent gathers in flight per thread
    for (uint64_t j0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j0 < n; j0 += nth * U) {
        uint32_t v[U], od[U];
        float a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // the slot streams first ...
            const uint64_t j = j0 + u * nth;
            v[u] = (it && j < n) ? order[j] : 0u;
            od[u] = j < nsrc ? od_hot[j] : 1u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = (it && j0 + u * nth < n) ? acc[v[u]] : 0.f;  // ... then the gathers
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = j0 + u * nth;
            if (j >= n) continue;
            const float r = it ? base + df * a[u] : r0;
            if (j < nsrc) contrib[j] = r / (float)od[u];
            else dang += r;
        }
    }
    const double tot = block_sum(dang, sm);
    if (threadIdx.x == 0) dpart[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(PR_THREADS) pr_rank_out(uint32_t n, double damping, const float *__restrict__ acc,
                                                          const double *__restrict__ scal, float *__restrict__ rank,
                                                          int it) {
    const float base = it ? (float)((1.0 - damping) / n + damping * scal[0] / n) : 0.f;
    const float df = (float)damping;
    const float r0 = (float)(1.0 / n);
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        rank[v] = it ? base + df * acc[v] : r0;
}

using PrPull = void (*)(wg_graph, const float *, float *, uint32_t, PrBound *);

PrPull pick(int w, bool shift = false) {
    switch (w) {
        case 1: return shift ? pr_pull<1, true> : pr_pull<1, false>;
        case 2: return shift ? pr_pull<2, true> : pr_pull<2, false>;
        case 4: return shift ? pr_pull<4, true> : pr_pull<4, false>;
        case 8: return shift ? pr_pull<8, true> : pr_pull<8, false>;
    }
    return nullptr;
}

unsigned pull_grid(PrPull pull) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pull, PR_THREADS, 0);
    if (per_sm < 1) per_sm = 1;
    return (unsigned)(sm_count() * per_sm);  // one full wave: the warp ranges fix the summation order
}

struct PrWs {
    PrBound *bounds;
    double *dpart;
};

size_t ws_bytes(uint32_t n) {
    return carve_size(sizeof(PrBound) * (size_t)sm_count() * 64) + carve_size(sizeof(double) * prep_grid(n ? n : 1));
}

int carve(uint32_t n, void *ws, size_t bytes, PrWs *w) {
    Carve c{(char *)ws, 0, bytes};
    w->bounds = c.take<PrBound>((size_t)sm_count() * 64);  // >= warps of one full wave (2048 threads / SM)
    w->dpart = c.take<double>(prep_grid(n ? n : 1));
    WG_REQUIRE(ws && w->bounds && w->dpart, "pagerank workspace too small (wg_pagerank_ws_bytes)");
    return WG_OK;
}

int pull_and_fixup(const wg_graph *g, const float *contrib, float *acc, uint32_t base, const PrWs &w,
                   cudaStream_t s) {
    PrPull pull = pick((int)g->width, base != 0);
    WG_REQUIRE(pull, "unsupported width %u", g->width);
    if (!g->nvec) return WG_OK;
    const unsigned grid = pull_grid(pull);
    const uint64_t nwarps = (uint64_t)grid * (PR_THREADS / 32);
    WG_REQUIRE(nwarps <= (uint64_t)sm_count() * 64, "pagerank pull grid exceeds its workspace");
    pull<<<grid, PR_THREADS, 0, s>>>(*g, contrib, acc, base, w.bounds);
    if (base) pr_fixup<true><<<grid_for(nwarps, 256, 4), 256, 0, s>>>(w.bounds, nwarps, acc, base);
    else pr_fixup<false><<<grid_for(nwarps, 256, 4), 256, 0, s>>>(w.bounds, nwarps, acc, base);
    ::wg::count_launch(2);
    WG_CHECK_LAUNCH("pagerank pull");
    return WG_OK;
}

int prep(uint32_t n, int it, double damping, const uint32_t *outdeg, float *acc, float *contrib, float *rank,
         double *scal, const PrWs &w, cudaStream_t s, bool zero_acc) {
    const unsigned vgrid = prep_grid(n);
    if (zero_acc) pr_prep<true><<<vgrid, PR_THREADS, 0, s>>>(n, it, damping, outdeg, acc, contrib, rank, scal, w.dpart);
    else pr_prep<false><<<vgrid, PR_THREADS, 0, s>>>(n, it, damping, outdeg, acc, contrib, rank, scal, w.dpart);
    pr_dangling<<<1, 32, 0, s>>>(w.dpart, vgrid, scal);
    ::wg::count_launch(2);
    WG_CHECK_LAUNCH("pagerank prep");
    return WG_OK;
}

}  // namespace

extern "C" size_t wg_pagerank_ws_bytes(const wg_graph *g) { return g ? ws_bytes(g->n) : 0; }

extern "C" int wg_pagerank(const wg_graph *g, int iterations, double damping, float *d_rank,
                           float *d_acc, float *d_contrib, double *d_scal, void *d_ws, size_t ws_bytes_,
                           void *stream) {
    WG_REQUIRE(g && d_rank && d_acc && d_contrib && d_scal, "null argument");
    WG_REQUIRE(iterations >= 0, "iterations must be >= 0");
    WG_REQUIRE(g->n > 0, "empty graph");
    PrWs w;
    int rc = carve(g->n, d_ws, ws_bytes_, &w);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    WG_CUDA(cudaMemsetAsync(d_acc, 0, (uint64_t)g->n * 4, s));
    WG_CUDA(cudaMemsetAsync(d_scal, 0, 4 * sizeof(double), s));
    for (int it = 0; it < iterations; ++it) {
        if ((rc = prep(g->n, it, damping, g->outdeg, d_acc, d_contrib, nullptr, d_scal, w, s, false))) return rc;
        if ((rc = pull_and_fixup(g, d_contrib, d_acc, 0u, w, s))) return rc;
    }
    // final apply: prep of iteration `iterations` writes the ranks
    return prep(g->n, iterations, damping, g->outdeg, d_acc, d_contrib, d_rank, d_scal, w, s, false);
}


// ---- hot-source layout ---------------------------------------------------
static size_t hot_sort_temp(uint32_t n) {
    size_t t = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, t, kb, vb, (int64_t)n, 0, 32);
    return t;
}

extern "C" size_t wg_pagerank_hot_ws_bytes(const wg_graph *g) {
    if (!g) return 0;
    const size_t n = g->n ? g->n : 1;
    // keys x2, ids x2, slot_of, counter, sort temp
    return 5 * carve_size(4 * n) + carve_size(8) + carve_size(hot_sort_temp((uint32_t)n)) + 1024;
}

extern "C" int wg_pagerank_hot_layout(const wg_graph *g, uint32_t *d_vsrc_hot, uint32_t *d_order,
                                      uint32_t *d_od_hot, uint64_t *h_nsrc, void *d_ws, size_t ws_bytes_,
                                      void *stream) {
    WG_REQUIRE(g && d_vsrc_hot && d_order && d_od_hot && h_nsrc && d_ws, "null argument");
    WG_REQUIRE(g->n > 0, "empty graph");
    cudaStream_t s = as_stream(stream);
    const uint32_t n = g->n;
    Carve c{(char *)d_ws, 0, ws_bytes_};
    uint32_t *k0 = c.take<uint32_t>(n), *k1 = c.take<uint32_t>(n);
    uint32_t *v0 = c.take<uint32_t>(n), *v1 = c.take<uint32_t>(n);
    uint32_t *slot_of = c.take<uint32_t>(n);
    unsigned long long *cnt = c.take<unsigned long long>(1);
    size_t tb = hot_sort_temp(n);
    void *temp = c.take<char>(tb);
    WG_REQUIRE(k0 && k1 && v0 && v1 && slot_of && cnt && temp, "workspace too small (wg_pagerank_hot_ws_bytes)");
    WG_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
    hot_keys_kernel<<<grid_for(n, 1024, 8), 256, 0, s>>>(n, g->outdeg, k0, v0, cnt);
    cub::DoubleBuffer<uint32_t> kb(k0, k1), vb(v0, v1);
    WG_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, kb, vb, (int64_t)n, 0, 32, s));
    WG_CUDA(cudaMemcpyAsync(d_order, vb.Current(), 4ull * n, cudaMemcpyDeviceToDevice, s));
    hot_slots_kernel<<<grid_for(n, 1024, 8), 256, 0, s>>>(n, d_order, g->outdeg, slot_of, d_od_hot);
    const uint64_t lanes = g->nvec * g->width;
    if (lanes) hot_lanes_kernel<<<grid_for(lanes, 1024, 16), 256, 0, s>>>(lanes, g->vsrc, slot_of, d_vsrc_hot);
    ::wg::count_launch(3);
    WG_CHECK_LAUNCH("pagerank hot layout");
    unsigned long long h = 0;
    WG_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    *h_nsrc = (uint64_t)h;
    return WG_OK;
}

extern "C" int wg_pagerank_hot(const wg_graph *g, const uint32_t *d_vsrc_hot, const uint32_t *d_order,
                               const uint32_t *d_od_hot, uint64_t nsrc, int iterations, double damping,
                               float *d_rank, float *d_acc, float *d_contrib, double *d_scal, void *d_ws,
                               size_t ws_bytes_, void *stream) {
    WG_REQUIRE(g && d_vsrc_hot && d_order && d_od_hot && d_rank && d_acc && d_contrib && d_scal, "null argument");
    WG_REQUIRE(iterations >= 0, "iterations must be >= 0");
    WG_REQUIRE(g->n > 0 && nsrc <= g->n, "bad sizes");
    PrWs w;
    int rc = carve(g->n, d_ws, ws_bytes_, &w);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    const uint32_t n = g->n;
    WG_CUDA(cudaMemsetAsync(d_acc, 0, (uint64_t)n * 4, s));
    WG_CUDA(cudaMemsetAsync(d_scal, 0, 4 * sizeof(double), s));
    wg_graph gh = *g;
    gh.vsrc = d_vsrc_hot;  // lanes hold contrib slots
    const unsigned vgrid = prep_grid(n);
    for (int it = 0; it < iterations; ++it) {
        pr_prep_hot<<<vgrid, PR_THREADS, 0, s>>>(n, (uint32_t)nsrc, it, damping, d_order, d_od_hot, d_acc, d_contrib,
                                                 d_scal, w.dpart);
        pr_dangling<<<1, 32, 0, s>>>(w.dpart, vgrid, d_scal);
        ::wg::count_launch(2);
        WG_CHECK_LAUNCH("pagerank prep (hot)");
        if ((rc = pull_and_fixup(&gh, d_contrib, d_acc, 0u, w, s))) return rc;
    }
    pr_rank_out<<<vgrid, PR_THREADS, 0, s>>>(n, damping, d_acc, d_scal, d_rank, iterations);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("pagerank ranks");
    return WG_OK;
}

extern "C" size_t wg_pagerank_prep_ws_bytes(uint32_t n) { return ws_bytes(n); }

extern "C" int wg_pagerank_prep(uint32_t n, int it, double damping, const uint32_t *d_outdeg,
                                float *d_acc, float *d_contrib, float *d_rank, double *d_scal, void *d_ws,
                                size_t ws_bytes_, void *stream) {
    WG_REQUIRE(n > 0 && d_outdeg && d_acc && d_contrib && d_scal, "null argument");
    WG_REQUIRE(it >= 0, "iteration must be >= 0");
    PrWs w;
    int rc = carve(n, d_ws, ws_bytes_, &w);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    if (it == 0) WG_CUDA(cudaMemsetAsync(d_scal, 0, 4 * sizeof(double), s));
    return prep(n, it, damping, d_outdeg, d_acc, d_contrib, d_rank, d_scal, w, s, true);
}

extern "C" int wg_pagerank_pull(const wg_graph *g, const float *d_contrib, float *d_acc,
                                uint32_t dst_base, void *d_ws, size_t ws_bytes_, void *stream) {
    WG_REQUIRE(g && d_contrib && d_acc, "null argument");
    PrWs w;
    int rc = carve(g->n, d_ws, ws_bytes_, &w);
    if (rc) return rc;
    return pull_and_fixup(g, d_contrib, d_acc, dst_base, w, as_stream(stream));
}
