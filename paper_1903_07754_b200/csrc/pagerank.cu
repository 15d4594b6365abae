// pagerank.cu — dense PageRank pull (K8).  No reference implementation
// exists (pkg/tests/test_apps.py:167-169); semantics follow
// BASELINE.json config 5: float32 ranks, damping d, fixed iterations,
// dangling mass redistributed uniformly:
//   r0 = 1/N;  r'(v) = (1-d)/N + d * (sum_{u->v} r(u)/outdeg(u) + D/N),
//   D = sum of r(u) over outdeg(u) = 0.
// The pull reuses the min-plus tile body with a float segmented SUM; only a
// destination shared with a neighbouring tile is combined with atomicAdd.
// The apply of iteration i is fused into the contribution pass of i+1, so an
// iteration is two kernels: prep (V-sized) and pull (E-sized).
#include "common.cuh"

using namespace wg;

namespace {

// prep(it): r = it ? base(D_{it-1}) + d*acc : 1/N; acc = 0; contrib = r/outdeg;
// accumulate D_it into scal[it % 3]; zero scal[(it+1) % 3].
__global__ void __launch_bounds__(256) pr_prep(uint32_t n, int it, double damping,
                                               const uint32_t *outdeg, float *acc, float *contrib,
                                               float *rank_out, double *scal) {
    __shared__ double sm[33];
    double dang = 0.0;
    const float base = it ? (float)((1.0 - damping) / n + damping * scal[(it + 2) % 3] / n) : 0.f;
    const float df = (float)damping;
    const float r0 = (float)(1.0 / n);
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        float r = it ? base + df * acc[v] : r0;
        acc[v] = 0.f;
        uint32_t od = outdeg[v];
        if (od) {
            contrib[v] = r / (float)od;
        } else {
            contrib[v] = 0.f;
            dang += r;
        }
        if (rank_out) rank_out[v] = r;
    }
    double tot = block_sum(dang, sm);
    if (threadIdx.x == 0) {
        if (tot != 0.0) atomicAdd(&scal[it % 3], tot);
        if (blockIdx.x == 0) scal[(it + 1) % 3] = 0.0;
    }
}

template <int W, bool SHIFT>
__global__ void __launch_bounds__(256) pr_pull(wg_graph g, const float *contrib, float *acc, uint32_t base_) {
    const uint32_t base = SHIFT ? base_ : 0u;  // destination-sharded runs index a slice
    const unsigned lane = lane_id();
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t ntiles = (g.nvec + 31) >> 5;
    for (uint64_t tile = gwarp; tile < ntiles; tile += nwarps) {
        const uint64_t p = (tile << 5) + lane;
        const bool valid = p < g.nvec;
        const uint32_t d = valid ? g.vdst[p] : 0xffffffffu;
        float sum = 0.f;
        if (valid) {
            uint32_t src[W];
            load_lanes<W>(g.vsrc, p, src);
#pragma unroll
            for (int l = 0; l < W; ++l)
                if (src[l] != WG_NO_LANE) sum += contrib[src[l]];
        }
        const uint32_t dn = __shfl_down_sync(FULL, d, 1);
        const uint32_t dp = __shfl_up_sync(FULL, d, 1);
        const bool head = lane == 0 || dp != d;
        const bool tail = lane == 31 || dn != d;
        const unsigned heads = __ballot_sync(FULL, head);
        const unsigned head_lane = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
        // segmented sum limited to the longest segment of the tile
        const unsigned dist = lane - head_lane;
        const unsigned maxd = __reduce_max_sync(FULL, dist);
        for (unsigned off = 1; off <= maxd; off <<= 1) {
            const float o = __shfl_up_sync(FULL, sum, off);
            if (off <= dist) sum += o;
        }
        if (tail && valid) {
            bool complete = true;
            if (head_lane == 0 && p >= lane + 1 && g.vdst[p - lane - 1] == d) complete = false;
            if (lane == 31 && p + 1 < g.nvec && g.vdst[p + 1] == d) complete = false;
            if (complete) acc[d - base] = sum;
            else atomicAdd(&acc[d - base], sum);
        }
    }
}

using PrPull = void (*)(wg_graph, const float *, float *, uint32_t);

PrPull pick(int w, bool shift = false) {
    switch (w) {
        case 1: return shift ? pr_pull<1, true> : pr_pull<1, false>;
        case 2: return shift ? pr_pull<2, true> : pr_pull<2, false>;
        case 4: return shift ? pr_pull<4, true> : pr_pull<4, false>;
        case 8: return shift ? pr_pull<8, true> : pr_pull<8, false>;
    }
    return nullptr;
}

unsigned pull_grid(const wg_graph *g, PrPull pull) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pull, 256, 0);
    if (per_sm < 1) per_sm = 1;
    return grid_for(g->nvec, 256, (unsigned)per_sm);
}

}  // namespace

extern "C" int wg_pagerank(const wg_graph *g, int iterations, double damping, float *d_rank,
                           float *d_acc, float *d_contrib, double *d_scal, void *stream) {
    WG_REQUIRE(g && d_rank && d_acc && d_contrib && d_scal, "null argument");
    WG_REQUIRE(iterations >= 0, "iterations must be >= 0");
    WG_REQUIRE(g->n > 0, "empty graph");
    PrPull pull = pick((int)g->width);
    WG_REQUIRE(pull, "unsupported width %u", g->width);
    cudaStream_t s = as_stream(stream);
    WG_CUDA(cudaMemsetAsync(d_acc, 0, (uint64_t)g->n * 4, s));
    WG_CUDA(cudaMemsetAsync(d_scal, 0, 4 * sizeof(double), s));
    unsigned vgrid = grid_for(g->n, 256 * 4, 8);
    unsigned egrid = pull_grid(g, pull);
    for (int it = 0; it < iterations; ++it) {
        pr_prep<<<vgrid, 256, 0, s>>>(g->n, it, damping, g->outdeg, d_acc, d_contrib, nullptr, d_scal); ::wg::count_launch();
        if (g->nvec) {
            pull<<<egrid, 256, 0, s>>>(*g, d_contrib, d_acc, 0u);
            ::wg::count_launch();
        }
    }
    // final apply: prep of iteration `iterations` writes the ranks
    pr_prep<<<vgrid, 256, 0, s>>>(g->n, iterations, damping, g->outdeg, d_acc, d_contrib, d_rank,
                                  d_scal); ::wg::count_launch();
    WG_CHECK_LAUNCH("pagerank");
    return WG_OK;
}

extern "C" int wg_pagerank_prep(uint32_t n, int it, double damping, const uint32_t *d_outdeg,
                                float *d_acc, float *d_contrib, float *d_rank, double *d_scal,
                                void *stream) {
    WG_REQUIRE(n > 0 && d_outdeg && d_acc && d_contrib && d_scal, "null argument");
    WG_REQUIRE(it >= 0, "iteration must be >= 0");
    cudaStream_t s = as_stream(stream);
    if (it == 0) WG_CUDA(cudaMemsetAsync(d_scal, 0, 4 * sizeof(double), s));
    pr_prep<<<grid_for(n, 256 * 4, 8), 256, 0, s>>>(n, it, damping, d_outdeg, d_acc, d_contrib, d_rank,
                                                    d_scal);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("pagerank_prep");
    return WG_OK;
}

extern "C" int wg_pagerank_pull(const wg_graph *g, const float *d_contrib, float *d_acc,
                                uint32_t dst_base, void *stream) {
    WG_REQUIRE(g && d_contrib && d_acc, "null argument");
    PrPull pull = pick((int)g->width, dst_base != 0);
    WG_REQUIRE(pull, "unsupported width %u", g->width);
    if (!g->nvec) return WG_OK;
    cudaStream_t s = as_stream(stream);
    pull<<<pull_grid(g, pull), 256, 0, s>>>(*g, d_contrib, d_acc, dst_base);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("pagerank_pull");
    return WG_OK;
}
