// engine.cu — C-ABI entry points of the pull engine: per-call kernels (the
// reference backend protocol, kernels.py:55-125) and the device-resident
// convergence loop (engine.py:330-388).
#include <stdlib.h>

#include <mutex>
#include <unordered_map>
#include <vector>

#include "frontier.cuh"
#include "pull.cuh"

using namespace wg;

namespace {



struct Occ {
    std::mutex mu;
    std::unordered_map<const void *, int> blocks;
};
Occ &occ() {
    static Occ o;
    return o;
}

template <typename K>
unsigned persistent_grid(K kernel, int threads, uint64_t work_blocks, size_t dyn_smem = 0) {
    const void *key = (const void *)kernel;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(occ().mu);
        auto it = occ().blocks.find(key);
        if (it != occ().blocks.end()) per_sm = it->second;
    }
    if (per_sm == 0) {
        if (dyn_smem > 48 * 1024)
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn_smem) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        std::lock_guard<std::mutex> lk(occ().mu);
        occ().blocks[key] = per_sm;
    }
    uint64_t cap = (uint64_t)sm_count() * per_sm;
    if (work_blocks < 1) work_blocks = 1;
    return (unsigned)(work_blocks < cap ? work_blocks : cap);
}

using PullFn = void (*)(LoopCtx, wg_graph, PullBufs, int, int64_t, int64_t, int);
using DenseFn = void (*)(LoopCtx, wg_graph, PullBufs, int, int64_t, int64_t);

template <typename T, int W>
PullFn pick_pull_w(bool weight, bool filter) {
    constexpr int U = W >= 8 ? 1 : 2;
    if (weight) return filter ? pull_kernel<T, W, true, true, U> : pull_kernel<T, W, true, false, U>;
    return filter ? pull_kernel<T, W, false, true, U> : pull_kernel<T, W, false, false, U>;
}

template <typename T>
PullFn pick_pull_t(int width, bool weight, bool filter) {
    switch (width) {
        case 1: return pick_pull_w<T, 1>(weight, filter);
        case 2: return pick_pull_w<T, 2>(weight, filter);
        case 4: return pick_pull_w<T, 4>(weight, filter);
        case 8: return pick_pull_w<T, 8>(weight, filter);
    }
    return nullptr;
}

PullFn pick_pull(int val_type, int width, bool weight, bool filter) {
    return val_type == WG_VAL_U32 ? pick_pull_t<uint32_t>(width, weight, filter)
                                  : pick_pull_t<int64_t>(width, weight, filter);
}



// Persistent sparse loop on/off (WG_SPARSE_LOOP=0 disables it).
bool g_sparse_loop = [] {
    const char *e = getenv("WG_SPARSE_LOOP");
    return !(e && e[0] == '0');
}();

// TMA-streamed dense pull: 2 tiles per stage, 4 stages (measured best of the
// (tiles, stages, blocks/SM) grid on CC s22 / SSSP s26).
template <typename T, int W, bool WEIGHT, bool FILTER>
DenseFn dense_fn(size_t *smem) {
    *smem = TmaSmem<W, WEIGHT, 2, 4>::BLOCK_BYTES;
    return pull_dense_tma_kernel<T, W, WEIGHT, FILTER, 2, 4, 1>;
}

template <typename T, int W>
DenseFn pick_dense_w(bool weight, bool filter, size_t *smem) {
    if (weight) return filter ? dense_fn<T, W, true, true>(smem) : dense_fn<T, W, true, false>(smem);
    return filter ? dense_fn<T, W, false, true>(smem) : dense_fn<T, W, false, false>(smem);
}

DenseFn pick_dense(int val_type, int width, bool weight, bool filter, size_t *smem) {
    bool u32 = val_type == WG_VAL_U32;
    switch (width) {
        case 1: return u32 ? pick_dense_w<uint32_t, 1>(weight, filter, smem) : pick_dense_w<int64_t, 1>(weight, filter, smem);
        case 2: return u32 ? pick_dense_w<uint32_t, 2>(weight, filter, smem) : pick_dense_w<int64_t, 2>(weight, filter, smem);
        case 4: return u32 ? pick_dense_w<uint32_t, 4>(weight, filter, smem) : pick_dense_w<int64_t, 4>(weight, filter, smem);
        case 8: return u32 ? pick_dense_w<uint32_t, 8>(weight, filter, smem) : pick_dense_w<int64_t, 8>(weight, filter, smem);
    }
    return nullptr;
}

int check_graph(const wg_graph *g) {
    WG_REQUIRE(g != nullptr, "graph is null");
    WG_REQUIRE(g->width == 1 || g->width == 2 || g->width == 4 || g->width == 8,
               "unsupported vector width %u (1, 2, 4, 8)", g->width);
    WG_REQUIRE(g->n < 0xffffffffu, "vertex count must be < 2^32-1");
    WG_REQUIRE(g->nvec < (1ull << 32) && g->entries < (1ull << 32), "layout too large for uint32 ids");
    if (g->nvec) WG_REQUIRE(g->vsrc && g->vdst, "null layout arrays");
    WG_REQUIRE(g->idx_off && g->outdeg, "null index/degree arrays");
    return WG_OK;
}

uint64_t groups_of(const wg_graph *g, int shift) { return (g->nvec + (1ull << shift) - 1) >> shift; }

struct KernelWs {
    wg_iter_rec *recs;
    uint32_t *fvert[2], *fpref[2], *tstart[2], *glist;
    uint64_t *bcount;
    unsigned *ticket;
};

uint64_t tstart_entries(const wg_graph *g) { return g->entries / TR_TILE + 2; }

bool lens_are_degrees(const wg_graph *g) { return (g->flags & WG_GRAPH_LENS_ARE_DEGREES) != 0; }

// Compaction scratch: per-block totals of the frontier (4 per block) or
// group (1 per block) compactions, then one slot holding the frontier
// compaction's completion ticket (zero between launches).
uint64_t bcount_entries(const wg_graph *g, int shift) {
    uint64_t n = g->n ? g->n : 1, groups = groups_of(g, shift);
    uint64_t nb = fb_blocks(n) * 4, gb = cb_blocks(groups ? groups : 1);
    return (nb > gb ? nb : gb) + 1;
}
unsigned *bcount_ticket(const wg_graph *g, int shift, uint64_t *bcount) {
    return reinterpret_cast<unsigned *>(bcount + bcount_entries(g, shift) - 1);
}

int carve_kernel_ws(const wg_graph *g, int shift, void *ws, size_t bytes, KernelWs *k) {
    Carve cv{(char *)ws, 0, bytes};
    uint64_t n = g->n ? g->n : 1, groups = groups_of(g, shift);
    k->recs = cv.take<wg_iter_rec>(2);
    for (int i = 0; i < 2; ++i) {
        k->fvert[i] = cv.take<uint32_t>(n);
        k->fpref[i] = cv.take<uint32_t>(n);
        k->tstart[i] = cv.take<uint32_t>(tstart_entries(g));
    }
    k->glist = cv.take<uint32_t>(groups ? groups : 1);
    k->bcount = cv.take<uint64_t>(bcount_entries(g, shift));
    k->ticket = k->bcount ? bcount_ticket(g, shift, k->bcount) : nullptr;
    if (!k->recs || !k->fvert[1] || !k->fpref[1] || !k->tstart[1] || !k->glist || !k->bcount) {
        set_error("kernel workspace too small (%zu bytes)", bytes);
        return WG_ENOSPACE;
    }
    return WG_OK;
}

LoopCtx forced_ctx(wg_iter_rec *recs, int mode, uint64_t edges) {
    LoopCtx c{};
    c.recs = recs;
    c.ring = 2;
    c.forced_mode = mode;
    c.ctrl = nullptr;
    c.it_arg = 1;
    c.wedge_limit = 0;
    c.edges = edges;
    c.keep_lists = 1;
    return c;
}

int launch_group_compaction(const LoopCtx &c, uint32_t *words, uint64_t ngroups, uint64_t *bcount,
                            uint32_t *glist, int clear, int shift, uint64_t nvec, cudaStream_t s) {
    uint64_t nb = cb_blocks(ngroups ? ngroups : 1);
    group_count_kernel<<<(unsigned)nb, CB_THREADS, 0, s>>>(c, words, ngroups, bcount); ::wg::count_launch();
    group_list_kernel<<<(unsigned)nb, CB_THREADS, 0, s>>>(c, words, ngroups, bcount, glist, clear,
                                                          shift, nvec); ::wg::count_launch();
    WG_CHECK_LAUNCH("group compaction");
    return WG_OK;
}

// keep_list = 0: the member list is built only when the gate (edges,
// wedge_limit) sends the next iteration to Wedge (the seed of a run whose
// first iteration is dense needs none)
int launch_frontier_compaction(const wg_graph *g, const uint32_t *words, uint64_t *bcount,
                               unsigned *ticket, uint32_t *fvert, uint32_t *fpref, uint32_t *tstart,
                               wg_iter_rec *rec, cudaStream_t s, int keep_list = 1, uint64_t wedge_limit = 0) {
    uint64_t nb = fb_blocks(g->n ? g->n : 1);
    const uint64_t *off = lens_are_degrees(g) ? nullptr : g->idx_off;
    WG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
    frontier_count_kernel<<<(unsigned)nb, CB_THREADS, 0, s>>>(words, g->n, off, g->outdeg, bcount, ticket,
                                                              rec, keep_list, g->edges, wedge_limit);
    ::wg::count_launch();
    frontier_list_kernel<<<(unsigned)nb, CB_THREADS, 0, s>>>(words, g->n, off, g->outdeg, bcount, fvert,
                                                             fpref, tstart, rec); ::wg::count_launch();
    WG_CHECK_LAUNCH("frontier compaction");
    return WG_OK;
}

int launch_transform(const LoopCtx &c, const wg_graph *g, uint32_t *const fvert[2],
                     uint32_t *const fpref[2], uint32_t *const tstart[2], int shift, uint32_t *gbits,
                     cudaStream_t s, int append = 0, uint32_t *glist = nullptr, uint64_t ngroups = 0) {
    unsigned grid = persistent_grid(transform_kernel, TR_THREADS, (g->entries + TR_TILE - 1) / TR_TILE);
    transform_kernel<<<grid, TR_THREADS, 0, s>>>(c, fvert[0], fvert[1], fpref[0], fpref[1], tstart[0],
                                                 tstart[1], g->idx_off, g->idx_pos, shift, gbits, append,
                                                 glist, ngroups);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("transform");
    return WG_OK;
}

using SparseFn = void (*)(LoopCtx, wg_graph, PullBufs, int, int64_t, int64_t, uint32_t *, uint64_t);

template <typename T, int W>
SparseFn pick_sparse_w(bool weight, bool filter) {
    if (weight) return filter ? pull_sparse_kernel<T, W, true, true> : pull_sparse_kernel<T, W, true, false>;
    return filter ? pull_sparse_kernel<T, W, false, true> : pull_sparse_kernel<T, W, false, false>;
}

SparseFn pick_sparse(int val_type, int width, bool weight, bool filter) {
    bool u32 = val_type == WG_VAL_U32;
    switch (width) {
        case 1: return u32 ? pick_sparse_w<uint32_t, 1>(weight, filter) : pick_sparse_w<int64_t, 1>(weight, filter);
        case 2: return u32 ? pick_sparse_w<uint32_t, 2>(weight, filter) : pick_sparse_w<int64_t, 2>(weight, filter);
        case 4: return u32 ? pick_sparse_w<uint32_t, 4>(weight, filter) : pick_sparse_w<int64_t, 4>(weight, filter);
        case 8: return u32 ? pick_sparse_w<uint32_t, 8>(weight, filter) : pick_sparse_w<int64_t, 8>(weight, filter);
    }
    return nullptr;
}

using LoopFn = void (*)(LoopCtx, wg_graph, PullBufs, int, int64_t, int64_t, uint32_t *, uint64_t);

template <typename T, int W>
LoopFn pick_loop_w(bool weight, bool filter) {
    if (weight) return filter ? sparse_loop_kernel<T, W, true, true> : sparse_loop_kernel<T, W, true, false>;
    return filter ? sparse_loop_kernel<T, W, false, true> : sparse_loop_kernel<T, W, false, false>;
}

LoopFn pick_loop(int val_type, int width, bool weight, bool filter) {
    bool u32 = val_type == WG_VAL_U32;
    switch (width) {
        case 1: return u32 ? pick_loop_w<uint32_t, 1>(weight, filter) : pick_loop_w<int64_t, 1>(weight, filter);
        case 2: return u32 ? pick_loop_w<uint32_t, 2>(weight, filter) : pick_loop_w<int64_t, 2>(weight, filter);
        case 4: return u32 ? pick_loop_w<uint32_t, 4>(weight, filter) : pick_loop_w<int64_t, 4>(weight, filter);
        case 8: return u32 ? pick_loop_w<uint32_t, 8>(weight, filter) : pick_loop_w<int64_t, 8>(weight, filter);
    }
    return nullptr;
}

// Cooperative launch of the persistent sparse loop (all blocks co-resident).
int launch_sparse_loop(const LoopCtx &c, const wg_graph *g, const PullBufs &pb, int val_type, int shift,
                       const wg_minplus *k, uint32_t *gbits, uint64_t ngroups, cudaStream_t s) {
    LoopFn fn = pick_loop(val_type, (int)g->width, k->use_weight != 0, k->filter_unvisited != 0);
    WG_REQUIRE(fn != nullptr, "no sparse loop kernel for width %u", g->width);
    int per_sm = 0;
    WG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, PULL_THREADS, 0));
    WG_REQUIRE(per_sm >= 1, "sparse loop kernel does not fit on an SM");
    static const int cap = [] {
        const char *e = getenv("WG_PERSIST_BLOCKS");
        return e ? atoi(e) : 4;
    }();
    if (cap > 0 && per_sm > cap) per_sm = cap;
    // small graphs (C1: 475K vectors) never fill more than one block per SM and
    // pay for every extra block in each grid barrier: BFS s16 96 vs 113 us
    if (!getenv("WG_PERSIST_BLOCKS") && g->nvec <= (1ull << 20)) per_sm = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sm_count() * per_sm));
    cfg.blockDim = dim3(PULL_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    WG_CUDA(cudaLaunchKernelEx(&cfg, fn, c, *g, pb, shift, (int64_t)k->apply_increment, (int64_t)k->sentinel,
                               gbits, ngroups));
    ::wg::count_launch();
    return WG_OK;
}

int launch_pull_sparse(const LoopCtx &c, const wg_graph *g, const PullBufs &pb, int val_type, int shift,
                       const wg_minplus *k, uint32_t *gbits, uint64_t ngroups, cudaStream_t s) {
    SparseFn fn = pick_sparse(val_type, (int)g->width, k->use_weight != 0, k->filter_unvisited != 0);
    WG_REQUIRE(fn != nullptr, "no sparse pull kernel for width %u", g->width);
    unsigned grid = persistent_grid(fn, PULL_THREADS, (g->nvec + 255) / 256);
    fn<<<grid, PULL_THREADS, 0, s>>>(c, *g, pb, shift, k->apply_increment, k->sentinel, gbits, ngroups);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("pull (sparse)");
    return WG_OK;
}

// only: 0 = everything the gate may need (non-graph path); MODE_FULL / MODE_WEDGE
// = just that mode's kernels (conditional graph bodies).
// timer/slot (optional): the caller's open timer slot around the pull; the
// frontier compaction after a dense pull is timed in its own slot (kind 4).
int launch_pull(const LoopCtx &c, const wg_graph *g, const PullBufs &pb, int val_type, int shift,
                const wg_minplus *k, uint64_t max_items, cudaStream_t s, int only = 0,
                void *timer = nullptr, int *slot = nullptr) {
    const bool weight = k->use_weight != 0, filter = k->filter_unvisited != 0;
    WG_REQUIRE(!weight || g->vw, "weighted kernel on an unweighted layout");
    PullFn fn = pick_pull(val_type, (int)g->width, weight, filter);
    WG_REQUIRE(fn != nullptr, "no pull kernel for width %u", g->width);
    int handles = (1 << MODE_FULL) | (1 << MODE_WEDGE);
    if (only) handles = 1 << only;
    const bool want_full = only == 0 || only == MODE_FULL;
    if (want_full && (c.forced_mode == 0 || c.forced_mode == MODE_FULL)) {
      if (pb.dst_major) {  // bottom-up kind: returns at once until V/1024 vertices are visited (dst_major_active)
        using DstFn = void (*)(LoopCtx, wg_graph, PullBufs, int64_t, int64_t);
        DstFn fd = nullptr;
        const bool u32 = val_type == WG_VAL_U32;
#define WG_PICK_DST(KIND)                                                                          \
    switch (g->width) {                                                                            \
        case 1: fd = u32 ? dense_dst_kernel<uint32_t, 1, KIND> : dense_dst_kernel<int64_t, 1, KIND>; break; \
        case 2: fd = u32 ? dense_dst_kernel<uint32_t, 2, KIND> : dense_dst_kernel<int64_t, 2, KIND>; break; \
        case 4: fd = u32 ? dense_dst_kernel<uint32_t, 4, KIND> : dense_dst_kernel<int64_t, 4, KIND>; break; \
        case 8: fd = u32 ? dense_dst_kernel<uint32_t, 8, KIND> : dense_dst_kernel<int64_t, 8, KIND>; break; \
    }
        if (filter) { WG_PICK_DST(DSTK_BOTTOM_UP) } else { WG_PICK_DST(DSTK_FLOOR) }
#undef WG_PICK_DST
        WG_REQUIRE(fd, "no destination-major pull for width %u", g->width);
        // one full wave of resident blocks (grid-stride over destinations)
        fd<<<persistent_grid(fd, 256, ((uint64_t)g->n + 255) / 256), 256, 0, s>>>(c, *g, pb, k->apply_increment,
                                                                                k->sentinel);
        ::wg::count_launch();
        WG_CHECK_LAUNCH("pull (dense, destination-major)");
      }
      if (!pb.dst_major || filter) {  // the vector-parallel kernels (they return when dense_dst_kernel ran)
        if (pb.ident && !weight && !filter) {  // iteration 1 of an identity-initialised run
            using IdentFn = void (*)(LoopCtx, wg_graph, PullBufs, int64_t, int64_t);
            IdentFn fi = nullptr;
            const bool u32 = val_type == WG_VAL_U32;
            switch (g->width) {
                case 1: fi = u32 ? pull_ident_kernel<uint32_t, 1> : pull_ident_kernel<int64_t, 1>; break;
                case 2: fi = u32 ? pull_ident_kernel<uint32_t, 2> : pull_ident_kernel<int64_t, 2>; break;
                case 4: fi = u32 ? pull_ident_kernel<uint32_t, 4> : pull_ident_kernel<int64_t, 4>; break;
                case 8: fi = u32 ? pull_ident_kernel<uint32_t, 8> : pull_ident_kernel<int64_t, 8>; break;
            }
            WG_REQUIRE(fi != nullptr, "no identity pull for width %u", g->width);
            fi<<<grid_for(g->nvec, 256 * 4, 8), 256, 0, s>>>(c, *g, pb, k->apply_increment, k->sentinel);
            ::wg::count_launch();
            WG_CHECK_LAUNCH("pull (identity)");
        }
        if (pb.floor_kernels && filter && pb.first_hit && !weight) {
            using BuFn = void (*)(LoopCtx, wg_graph, PullBufs, int64_t, int64_t);
            const bool u32 = val_type == WG_VAL_U32;
            BuFn fb = nullptr;
            switch (g->width) {
                case 1: fb = u32 ? bottom_up_pull_kernel<uint32_t, 1> : bottom_up_pull_kernel<int64_t, 1>; break;
                case 2: fb = u32 ? bottom_up_pull_kernel<uint32_t, 2> : bottom_up_pull_kernel<int64_t, 2>; break;
                case 4: fb = u32 ? bottom_up_pull_kernel<uint32_t, 4> : bottom_up_pull_kernel<int64_t, 4>; break;
                case 8: fb = u32 ? bottom_up_pull_kernel<uint32_t, 8> : bottom_up_pull_kernel<int64_t, 8>; break;
            }
            WG_REQUIRE(fb != nullptr, "no bottom-up pull for width %u", g->width);
            fb<<<grid_for(g->nvec, 256 * 4, 8), 256, 0, s>>>(c, *g, pb, k->apply_increment, k->sentinel);
            ::wg::count_launch();
            WG_CHECK_LAUNCH("pull (bottom-up)");
        }
        if (pb.floor_kernels && !weight && !filter) {
            // floor skipping from FLOOR_KERNELS_FROM on: one atomic-min pass
            // (earlier iterations return at once)
            using FpFn = void (*)(LoopCtx, wg_graph, PullBufs, int64_t, int64_t);
            const bool u32 = val_type == WG_VAL_U32;
            FpFn fp = nullptr;
            switch (g->width) {
                case 1: fp = u32 ? floor_pull_kernel<uint32_t, 1> : floor_pull_kernel<int64_t, 1>; break;
                case 2: fp = u32 ? floor_pull_kernel<uint32_t, 2> : floor_pull_kernel<int64_t, 2>; break;
                case 4: fp = u32 ? floor_pull_kernel<uint32_t, 4> : floor_pull_kernel<int64_t, 4>; break;
                case 8: fp = u32 ? floor_pull_kernel<uint32_t, 8> : floor_pull_kernel<int64_t, 8>; break;
            }
            WG_REQUIRE(fp != nullptr, "no floor pull for width %u", g->width);
            fp<<<grid_for(g->nvec, 256 * 4, 8), 256, 0, s>>>(c, *g, pb, k->apply_increment, k->sentinel);
            ::wg::count_launch();
            WG_CHECK_LAUNCH("pull (floor)");
        }
        {
            size_t smem = 0;
            // floor skipping runs an unfiltered program on the filtered pipeline
            DenseFn dn = pick_dense(val_type, (int)g->width, weight, filter || pb.floor_skip, &smem);
            unsigned grid = persistent_grid(dn, PULL_THREADS, (g->nvec + 255) / 256, smem);
            dn<<<grid, PULL_THREADS, smem, s>>>(c, *g, pb, shift, k->apply_increment, k->sentinel);
            ::wg::count_launch();
            WG_CHECK_LAUNCH("pull (dense, TMA)");
        }
      }
        if (slot) {
            timer_end(timer, *slot, s);
            *slot = timer_begin(timer, 4, (int64_t)c.it_arg, s);
        }
        // the dense pull only sets bits: build the produced frontier from the bitmap
        FrontierBufs fb;
        for (int i = 0; i < 2; ++i) {
            fb.fbits[i] = pb.fbits[i];
            fb.fvert[i] = pb.fvert[i];
            fb.fpref[i] = pb.fpref[i];
            fb.tstart[i] = pb.tstart[i];
        }
        fb.dst_major = pb.dst_major;
        fb.dst_bottom_up = filter ? 1u : 0u;
        const uint64_t nb = fb_blocks(g->n ? g->n : 1);
        const uint64_t *off = lens_are_degrees(g) ? nullptr : g->idx_off;
        if (!(pb.dst_major && !filter)) {  // a floor-kind destination-major pull always counts its own frontier
            loop_frontier_count_kernel<<<(unsigned)nb, CB_THREADS, 0, s>>>(c, fb, g->n, off, g->outdeg,
                                                                          pb.bcount, pb.ticket);
            ::wg::count_launch();
        }
        loop_frontier_list_kernel<<<(unsigned)nb, CB_THREADS, 0, s>>>(c, fb, g->n, off, g->outdeg, pb.bcount);
        ::wg::count_launch();
        WG_CHECK_LAUNCH("dense frontier compaction");
        if (slot) {  // a Wedge iteration's pull (below) is timed as a pull again
            timer_end(timer, *slot, s);
            *slot = timer_begin(timer, 2, (int64_t)c.it_arg, s);
        }
        handles &= ~(1 << MODE_FULL);
        if (c.forced_mode == MODE_FULL || handles == 0) return WG_OK;
    }
    unsigned grid = persistent_grid(fn, PULL_THREADS, (max_items + 255) / 256);
    fn<<<grid, PULL_THREADS, 0, s>>>(c, *g, pb, shift, k->apply_increment, k->sentinel, handles);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("pull");
    return WG_OK;
}


}  // namespace

extern "C" {

size_t wg_kernel_workspace_bytes(const wg_graph *g, int shift) {
    if (!g || shift < 0 || shift > 4) return 0;
    uint64_t n = g->n ? g->n : 1, groups = groups_of(g, shift);
    return carve_size(2 * sizeof(wg_iter_rec)) + 4 * carve_size(n * 4) + 2 * carve_size(tstart_entries(g) * 4) +
           carve_size((groups ? groups : 1) * 4) + carve_size(bcount_entries(g, shift) * 8) + 256;
}

int wg_transform(const wg_graph *g, const uint32_t *d_frontier_words, int shift,
                 uint32_t *d_wedge_words, void *d_ws, size_t ws_bytes, uint64_t *h_visited,
                 void *stream) {
    int rc = check_graph(g);
    if (rc) return rc;
    WG_REQUIRE(shift >= 0 && shift <= 4, "shift must be in [0, 4]");
    WG_REQUIRE(d_frontier_words && h_visited, "null argument");
    cudaStream_t s = as_stream(stream);
    KernelWs k;
    if ((rc = carve_kernel_ws(g, shift, d_ws, ws_bytes, &k))) return rc;
    WG_CUDA(cudaMemsetAsync(k.recs, 0, 2 * sizeof(wg_iter_rec), s));
    *h_visited = 0;
    if (g->n == 0) return WG_OK;
    if ((rc = launch_frontier_compaction(g, d_frontier_words, k.bcount, k.ticket, k.fvert[0], k.fpref[0],
                                         k.tstart[0], &k.recs[0], s)))
        return rc;
    if (g->entries) {
        WG_REQUIRE(d_wedge_words && g->idx_pos, "null wedge words / index");
        LoopCtx c = forced_ctx(k.recs, MODE_WEDGE, g->edges);
        if ((rc = launch_transform(c, g, k.fvert, k.fpref, k.tstart, shift, d_wedge_words, s))) return rc;
    }
    wg_iter_rec h[2];
    WG_CUDA(cudaMemcpyAsync(h, k.recs, sizeof(h), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    *h_visited = h[0].nz_packed & 0xffffffffull;
    return WG_OK;
}

static int pull_common(const wg_graph *g, const uint32_t *d_wedge_words, int shift, int val_type,
                       const void *d_prev, void *d_nxt, uint32_t *d_out_words, const wg_minplus *k,
                       void *d_ws, size_t ws_bytes, uint64_t *h_touched, void *stream) {
    int rc = check_graph(g);
    if (rc) return rc;
    WG_REQUIRE(val_type == WG_VAL_U32 || val_type == WG_VAL_I64, "bad value type");
    WG_REQUIRE(k && d_prev && d_nxt && d_out_words && h_touched, "null argument");
    WG_REQUIRE(shift >= 0 && shift <= 4, "shift must be in [0, 4]");
    cudaStream_t s = as_stream(stream);
    KernelWs ws;
    if ((rc = carve_kernel_ws(g, shift, d_ws, ws_bytes, &ws))) return rc;
    *h_touched = 0;
    if (g->nvec == 0) return WG_OK;
    WG_CUDA(cudaMemsetAsync(ws.recs, 0, 2 * sizeof(wg_iter_rec), s));
    bool wedge = d_wedge_words != nullptr;
    LoopCtx c = forced_ctx(ws.recs, wedge ? MODE_WEDGE : MODE_FULL, g->edges);
    uint64_t items = g->nvec;
    if (wedge) {
        uint64_t groups = groups_of(g, shift);
        if ((rc = launch_group_compaction(c, const_cast<uint32_t *>(d_wedge_words), groups, ws.bcount,
                                          ws.glist, 0, shift, g->nvec, s)))
            return rc;
        items = groups << shift;
    }
    PullBufs pb{};
    pb.vals[0] = const_cast<void *>(d_prev);
    pb.vals[1] = d_nxt;
    pb.fbits[0] = pb.fbits[1] = d_out_words;
    pb.fvert[0] = ws.fvert[0];
    pb.fvert[1] = ws.fvert[1];
    pb.fpref[0] = ws.fpref[0];
    pb.fpref[1] = ws.fpref[1];
    pb.tstart[0] = ws.tstart[0];
    pb.tstart[1] = ws.tstart[1];
    pb.glist = ws.glist;
    pb.bcount = ws.bcount;
    pb.ticket = ws.ticket;
    pb.n = g->n;
    WG_CUDA(cudaMemsetAsync(ws.ticket, 0, sizeof(unsigned), s));
    if ((rc = launch_pull(c, g, pb, val_type, shift, k, items, s))) return rc;
    wg_iter_rec h[2];
    WG_CUDA(cudaMemcpyAsync(h, ws.recs, sizeof(h), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    if (h[1].overflow) {
        set_error("uint32 value overflow: a candidate reached 0xFFFFFFFF");
        return WG_EOVERFLOW;
    }
    *h_touched = h[1].vectors_touched;
    return WG_OK;
}

int wg_pull_full(const wg_graph *g, int val_type, const void *d_prev, void *d_nxt,
                 uint32_t *d_out_words, const wg_minplus *k, void *d_ws, size_t ws_bytes,
                 uint64_t *h_touched, void *stream) {
    return pull_common(g, nullptr, 0, val_type, d_prev, d_nxt, d_out_words, k, d_ws, ws_bytes,
                       h_touched, stream);
}

int wg_pull_wedge(const wg_graph *g, const uint32_t *d_wedge_words, int shift, int val_type,
                  const void *d_prev, void *d_nxt, uint32_t *d_out_words, const wg_minplus *k,
                  void *d_ws, size_t ws_bytes, uint64_t *h_touched, void *stream) {
    if (!d_wedge_words) {
        set_error("null wedge words");
        return WG_EINVAL;
    }
    return pull_common(g, d_wedge_words, shift, val_type, d_prev, d_nxt, d_out_words, k, d_ws,
                       ws_bytes, h_touched, stream);
}

int wg_covered_groups(const uint32_t *d_wedge_words, uint64_t group_count, uint32_t *d_groups,
                      void *d_ws, size_t ws_bytes, uint64_t *h_count, void *stream) {
    WG_REQUIRE(h_count, "null argument");
    *h_count = 0;
    if (group_count == 0) return WG_OK;
    WG_REQUIRE(d_wedge_words && d_groups, "null argument");
    cudaStream_t s = as_stream(stream);
    Carve cv{(char *)d_ws, 0, ws_bytes};
    wg_iter_rec *recs = cv.take<wg_iter_rec>(2);
    uint64_t *bcount = cv.take<uint64_t>(cb_blocks(group_count));
    if (!recs || !bcount) {
        set_error("workspace too small");
        return WG_ENOSPACE;
    }
    WG_CUDA(cudaMemsetAsync(recs, 0, 2 * sizeof(wg_iter_rec), s));
    LoopCtx c = forced_ctx(recs, MODE_WEDGE, 1);
    int rc = launch_group_compaction(c, const_cast<uint32_t *>(d_wedge_words), group_count, bcount,
                                     d_groups, 0, 0, group_count, s);
    if (rc) return rc;
    wg_iter_rec h[2];
    WG_CUDA(cudaMemcpyAsync(h, recs, sizeof(h), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    *h_count = h[1].groups;
    return WG_OK;
}

// ------------------------------------------------------------ run loop ---
int wg_run_buffer_sizes(const wg_graph *g, int shift, uint64_t *h_sizes4) {  /* 5 entries */
    int rc = check_graph(g);
    if (rc) return rc;
    WG_REQUIRE(h_sizes4, "null argument");
    uint64_t groups = groups_of(g, shift);
    h_sizes4[0] = ((uint64_t)g->n + 31) >> 5;
    h_sizes4[1] = groups;
    h_sizes4[2] = (groups + 31) >> 5;
    h_sizes4[3] = bcount_entries(g, shift);
    h_sizes4[4] = tstart_entries(g);
    return WG_OK;
}

}  // extern "C"

namespace {
// Advance the device iteration counter and decide whether the WHILE body runs
// again: stop once the iteration did not run or produced a frontier without
// out-edges (engine.py:356-386), or at the launch's iteration limit.
__global__ void loop_step_kernel(cudaGraphConditionalHandle h, uint64_t *ctrl, const wg_iter_rec *recs,
                                 uint32_t ring) {
    const uint64_t it = ctrl[0] + 1;
    WG_KTS(it, KTS_STEP);
    if (it > ctrl[1]) {  // the persistent sparse loop already reached the launch limit
        cudaGraphSetConditional(h, 0u);
        return;
    }
    ctrl[0] = it;
    const wg_iter_rec &r = recs[it % ring];
    const bool stop = r.mode == 0 || r.out_edge_sum == 0 || it >= ctrl[1];
    cudaGraphSetConditional(h, stop ? 0u : 1u);
}
__global__ void set_limit_kernel(uint64_t *ctrl, uint64_t limit) { ctrl[1] = limit; }

// After the top-level attempt of the persistent loop: enter the WHILE body
// unless the run is already over (the last iteration it ran produced a
// frontier without out-edges, or the launch limit was reached).  Nothing ran
// yet (ctrl[0] == 0): the body takes iteration 1.
__global__ void loop_enter_kernel(cudaGraphConditionalHandle h, const uint64_t *ctrl, const wg_iter_rec *recs,
                                  uint32_t ring) {
    const uint64_t done = ctrl[0];
    WG_KTS(done + 1, KTS_STEP);
    bool stop = false;
    if (done > 0) stop = recs[done % ring].out_edge_sum == 0 || done >= ctrl[1];
    cudaGraphSetConditional(h, stop ? 0u : 1u);
}

// Gate of the persistent sparse loop (its cooperative launch costs several
// microseconds even when it returns at once, so it sits behind an IF node).
// It also takes destination-major dense iterations (dense_ok: unweighted
// run with a work list) -- sparse_loop_kernel runs those as phases too.
__global__ void sparse_gate_kernel(LoopCtx c, cudaGraphConditionalHandle h, uint64_t ngroups, uint32_t dense_ok,
                                   uint64_t n, int bottom_up) {
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_SPARSE_GATE);
    const bool dense = dense_ok && ctx_mode(c, it) == MODE_FULL && dst_major_active(c, it, n, 1u, bottom_up != 0);
    cudaGraphSetConditional(h, (dense || sparse_wedge(c, it, ngroups)) ? 1u : 0u);
}

// Device-side gate of the graph body: FullScan, Wedge through the ordered
// group list, or Wedge through the sparse (append) path when the transform
// work is small against the group bitmap (no bitmap scans are worth it).
__global__ void decide_kernel(LoopCtx c, cudaGraphConditionalHandle hf, cudaGraphConditionalHandle hs,
                              cudaGraphConditionalHandle hp, uint64_t ngroups, int has_entries) {
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_DECIDE);
    const int mode = ctx_mode(c, it);
    int variant = 0;
    if (mode == MODE_FULL) {
        variant = 1;
    } else if (mode == MODE_WEDGE) {
        const uint64_t entries = ctx_in(c, it)->nz_packed & 0xffffffffull;
        variant = (has_entries && entries * SPARSE_ENTRY_RATIO < ngroups) ? 3 : 2;
    }
    ctx_out(c, it)->reserved[0] = (uint64_t)variant;
    cudaGraphSetConditional(hf, variant == 1 ? 1u : 0u);
    cudaGraphSetConditional(hs, variant == 2 ? 1u : 0u);
    cudaGraphSetConditional(hp, variant == 3 ? 1u : 0u);
}
}  // namespace

extern "C" {

static LoopCtx loop_ctx(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                        const uint64_t *ctrl, uint64_t it) {
    LoopCtx c{};
    c.recs = b->recs;
    c.ring = b->ring;
    c.forced_mode = 0;
    c.ctrl = ctrl;
    c.it_arg = it;
    c.wedge_limit = p->wedge_limit;
    c.gate_local = (p->flags & WG_RUN_LOCAL_GATE) ? 1 : 0;
    c.edges = c.gate_local ? g->entries : g->edges;  // the local gate compares against local entries
    c.keep_lists = (p->flags & WG_RUN_KEEP_LISTS) ? 1 : 0;
    return c;
}


static PullBufs pull_bufs(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p) {
    PullBufs pb{};
    for (int i = 0; i < 2; ++i) {
        pb.vals[i] = b->vals[i];
        pb.fbits[i] = b->fbits[i];
        pb.fvert[i] = b->fvert[i];
        pb.fpref[i] = b->fpref[i];
        pb.tstart[i] = b->tstart[i];
    }
    pb.glist = b->glist;
    pb.gbits2 = b->gbits_alt;  // both set: fused persistent loop
    pb.glist2 = b->glist_alt;
    pb.bcount = b->bcount;
    pb.ticket = bcount_ticket(g, p->shift, b->bcount);
    pb.n = g->n;
    pb.first_hit = (p->flags & WG_RUN_FIRST_HIT) && p->kern.filter_unvisited && !p->kern.use_weight ? 1u : 0u;
    pb.level_base = p->level_base;
    pb.ident = (p->flags & WG_RUN_IDENTITY_INIT) ? 1u : 0u;
    pb.floor_skip = (p->flags & WG_RUN_FLOOR_SKIP) && p->val_type == WG_VAL_U32 && !p->kern.filter_unvisited ? 1u : 0u;
    {
        const char *e = getenv("WG_FLOOR_KERNELS");
        // floor skipping (CC) and bottom-up BFS both switch to a plain kernel
        pb.floor_kernels = (pb.floor_skip || pb.first_hit) && !p->kern.use_weight && !(e && e[0] == '0') ? 1u : 0u;
        const char *f = getenv("WG_FLOOR_FROM");
        pb.floor_from = f ? (uint32_t)atoi(f) : (uint32_t)FLOOR_KERNELS_FROM;
        if (pb.floor_from < 2) pb.floor_from = 2;  // iteration 1 is pull_ident_kernel's
        // the plain kernels exist for unweighted floor-skipping and bottom-up
        // (first-hit, filtered) pulls only
        const bool plain = pb.floor_kernels && ((pb.floor_skip && !p->kern.filter_unvisited) || pb.first_hit);
        pb.pipeline_until = plain ? pb.floor_from : ~0ull;
    }
    // destination-major dense pulls: CC-like floor runs and level-synchronous
    // BFS, unweighted, when the graph carries voff and the run a work list
    pb.work = b->work;
    pb.dst_major = g->voff && b->work && !p->kern.use_weight &&
                           ((pb.floor_skip && !p->kern.filter_unvisited) || (pb.first_hit && p->kern.filter_unvisited))
                       ? 1u : 0u;
    {
        // destination-major dense iterations run as phases of the persistent loop
        // (no launches, counts and member list in the same kernel); WG_LOOP_DENSE=0:
        // as kernels of their own.  (Before the lane redistribution of
        // dense_dst_phase the bottom-up kind of large graphs was faster on its own:
        // BFS s26 1.31 vs 1.76 ms per iteration; now the loop wins, 4.1 vs 4.7 ms TTS.)
        const char *e = getenv("WG_LOOP_DENSE");
        const bool want = e ? e[0] != '0' : true;
        pb.loop_dense = pb.dst_major && want ? 1u : 0u;
    }
    {
        const char *e = getenv("WG_DST_LIGHT");
        pb.dst_light = e ? (uint32_t)atoi(e) : DST_LIGHT;
    }
    return pb;
}

static int check_run(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p) {
    int rc = check_graph(g);
    if (rc) return rc;
    WG_REQUIRE(b && p, "null argument");
    WG_REQUIRE(p->val_type == WG_VAL_U32 || p->val_type == WG_VAL_I64, "bad value type");
    WG_REQUIRE(p->shift >= 0 && p->shift <= 4, "shift must be in [0, 4]");
    WG_REQUIRE(b->ring >= 4, "record ring must hold >= 4 records");
    WG_REQUIRE(b->vals[0] && b->vals[1] && b->fbits[0] && b->fbits[1] && b->fvert[0] && b->fvert[1] &&
                   b->fpref[0] && b->fpref[1] && b->tstart[0] && b->tstart[1] && b->gbits && b->glist &&
                   b->bcount && b->recs &&
                   b->ctrl,
               "null run buffer");
    WG_REQUIRE(!p->kern.use_weight || g->vw, "weighted kernel on an unweighted layout");
    return WG_OK;
}

}  // extern "C" (reopened below)

namespace {
// One launch for the whole run initialisation: zero ranges (uint32 words),
// the control words, and both value buffers from the initial values.
struct InitRanges {
    uint32_t *ptr[8];
    uint64_t words[8];
    int count;
    uint64_t *ctrl;
    const void *init;  // [n] values of val_type, or null
    void *vals[2];
    uint64_t n, vbytes;
    int keep_limit;  // seeded loop graph: ctrl[1] was set by the launch (wg_run_loop_launch_seeded)
};

// frontier 0 = every vertex: its counts are the graph's own totals
__global__ void seed_all_record_kernel(wg_iter_rec *rec, uint64_t nz, uint64_t ent, uint64_t z, uint64_t es) {
    rec->nz_packed = (nz << 32) | ent;
    rec->z_count = z;
    rec->frontier_out = nz + z;
    rec->out_edge_sum = es;
    rec->reserved[2] = 1;  // no member list: the caller checked that iteration 1 is dense
}

__global__ void run_init_kernel(InitRanges r) {
    WG_KTS(0, KTS_SEED);
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    if (tid == 0) {
        r.ctrl[0] = 0;
        if (!r.keep_limit) r.ctrl[1] = ~0ull;  // no iteration limit
        r.ctrl[2] = 0;
        r.ctrl[3] = 0;
    }
    for (int k = 0; k < r.count; ++k)
        for (uint64_t i = tid; i < r.words[k]; i += nth) r.ptr[k][i] = 0u;
    if (r.init) {
        if (r.vbytes == 4) {
            const uint32_t *src = (const uint32_t *)r.init;
            for (uint64_t i = tid; i < r.n; i += nth) {
                const uint32_t v = src[i];
                ((uint32_t *)r.vals[0])[i] = v;
                ((uint32_t *)r.vals[1])[i] = v;
            }
        } else {
            const uint64_t *src = (const uint64_t *)r.init;
            for (uint64_t i = tid; i < r.n; i += nth) {
                const uint64_t v = src[i];
                ((uint64_t *)r.vals[0])[i] = v;
                ((uint64_t *)r.vals[1])[i] = v;
            }
        }
    }
}
}  // namespace

extern "C" {

static int seed_launches(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, const void *d_init_values,
                         const uint32_t *d_init_words, const uint64_t *h_all_counts4, cudaStream_t s,
                         int keep_limit = 0) {
    WG_REQUIRE(d_init_words || h_all_counts4, "null initial frontier");
    const uint64_t words = ((uint64_t)g->n + 31) >> 5;
    const uint64_t gwords = (groups_of(g, p->shift) + 31) >> 5;
    InitRanges r{};
    auto add = [&](void *ptr, uint64_t w) {
        if (ptr && w) {
            r.ptr[r.count] = (uint32_t *)ptr;
            r.words[r.count] = w;
            ++r.count;
        }
    };
    add(b->recs, sizeof(wg_iter_rec) * b->ring / 4);
    add(b->fbits[0], words);
    add(b->fbits[1], words);
    add(b->gbits, gwords);
    add(b->gbits_alt, gwords);
    // the destination-major pulls' per-chunk frontier counters (zeroed again by each pull's last block)
    add(b->work, 8 * fb_blocks(g->n ? g->n : 1));
    if (g->n) add(bcount_ticket(g, p->shift, b->bcount), 1);
    r.ctrl = b->ctrl;
    r.init = d_init_values;
    r.vals[0] = b->vals[0];
    r.vals[1] = b->vals[1];
    r.n = g->n;
    r.vbytes = p->val_type == WG_VAL_U32 ? 4 : 8;
    r.keep_limit = keep_limit;
    run_init_kernel<<<grid_for(words * 32 + 1, 256 * 4, 4), 256, 0, s>>>(r);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("run_init");
    if (g->n == 0) return WG_OK;
    if (h_all_counts4) {
        // every vertex in frontier 0 with a dense first iteration (the caller's
        // check): the counts are the graph's totals, no compaction pass
        const uint64_t es = h_all_counts4[3];
        WG_REQUIRE(!(p->flags & WG_RUN_KEEP_LISTS) && !(g->edges > 0 && es < p->wedge_limit),
                   "all-vertices seed needs a dense first iteration without member lists");
        seed_all_record_kernel<<<1, 1, 0, s>>>(&b->recs[0], h_all_counts4[0], h_all_counts4[1], h_all_counts4[2],
                                               es);
        ::wg::count_launch();
        WG_CHECK_LAUNCH("seed record");
        return WG_OK;
    }
    return launch_frontier_compaction(g, d_init_words, b->bcount, bcount_ticket(g, p->shift, b->bcount),
                                      b->fvert[0], b->fpref[0], b->tstart[0],
                                      &b->recs[0], s, (p->flags & WG_RUN_KEEP_LISTS) ? 1 : 0, p->wedge_limit);
}

int wg_run_seed(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, const void *d_init_values,
                const uint32_t *d_init_words, const uint64_t *h_all_counts4, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    return seed_launches(g, b, p, d_init_values, d_init_words, h_all_counts4, as_stream(stream));
}

int wg_run_init(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                const uint32_t *d_init_words, void *stream) {
    return wg_run_seed(g, b, p, nullptr, d_init_words, nullptr, stream);
}

static int enqueue_one(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                       const LoopCtx &c, cudaStream_t s) {
    int rc;
    uint64_t groups = groups_of(g, p->shift);
    uint32_t *fv[2] = {b->fvert[0], b->fvert[1]};
    uint32_t *fp[2] = {b->fpref[0], b->fpref[1]};
    uint32_t *ts[2] = {b->tstart[0], b->tstart[1]};
    int slot = timer_begin(p->timer, 1, (int64_t)c.it_arg, s);
    if (g->entries) {
        if ((rc = launch_transform(c, g, fv, fp, ts, p->shift, b->gbits, s))) return rc;
    }
    if (groups) {
        if ((rc = launch_group_compaction(c, b->gbits, groups, b->bcount, b->glist, 1, p->shift,
                                          g->nvec, s)))
            return rc;
    }
    timer_end(p->timer, slot, s);
    PullBufs pb = pull_bufs(g, b, p);
    slot = timer_begin(p->timer, 2, (int64_t)c.it_arg, s);
    if (g->nvec) {
        if ((rc = launch_pull(c, g, pb, p->val_type, p->shift, &p->kern, g->nvec, s, 0, p->timer, &slot)))
            return rc;
    }
    timer_end(p->timer, slot, s);
    unsigned grid = (unsigned)sm_count() * 2;
    slot = timer_begin(p->timer, 3, (int64_t)c.it_arg, s);
    if (p->val_type == WG_VAL_U32)
        finalize_kernel<uint32_t><<<grid, 256, 0, s>>>(c, pb);
    else
        finalize_kernel<int64_t><<<grid, 256, 0, s>>>(c, pb);
    ::wg::count_launch();
    timer_end(p->timer, slot, s);
    WG_CHECK_LAUNCH("finalize");
    return WG_OK;
}

int wg_run_enqueue(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                   uint64_t it_begin, uint32_t count, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    WG_REQUIRE(it_begin >= 1, "iterations are 1-based");
    WG_REQUIRE(count + 1 < b->ring, "batch of %u iterations needs a ring > %u", count, count + 1);
    cudaStream_t s = as_stream(stream);
    for (uint32_t i = 0; i < count; ++i) {
        LoopCtx c = loop_ctx(g, b, p, nullptr, it_begin + i);
        if ((rc = enqueue_one(g, b, p, c, s))) return rc;
    }
    return WG_OK;
}

int wg_run_enqueue_counter(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                           uint32_t count, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    WG_REQUIRE(count + 1 < b->ring, "batch of %u iterations needs a ring > %u", count, count + 1);
    cudaStream_t s = as_stream(stream);
    for (uint32_t i = 0; i < count; ++i) {
        LoopCtx c = loop_ctx(g, b, p, b->ctrl, 1 + i);
        if ((rc = enqueue_one(g, b, p, c, s))) return rc;
    }
    bump_counter_kernel<<<1, 1, 0, s>>>(b->ctrl, count); ::wg::count_launch();
    WG_CHECK_LAUNCH("bump");
    return WG_OK;
}

// ---------------------------------------------------------- CUDA graph --
void *wg_run_graph_create(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                          uint32_t count, void *stream) {
    if (check_run(g, b, p)) return nullptr;
    (void)stream;
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
        set_error("cudaStreamCreate failed");
        return nullptr;
    }
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } guard{s};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        set_error("cudaStreamBeginCapture failed");
        return nullptr;
    }
    int rc = wg_run_enqueue_counter(g, b, p, count, (void *)s);
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (rc != WG_OK || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        if (rc == WG_OK) cuda_fail(e, "cudaStreamEndCapture");
        return nullptr;
    }
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaGraphInstantiate");
        return nullptr;
    }
    return (void *)exec;
}

int wg_run_graph_launch(void *graph, void *stream) {
    WG_REQUIRE(graph, "null graph");
    WG_CUDA(cudaGraphLaunch((cudaGraphExec_t)graph, as_stream(stream)));
    return WG_OK;
}

void wg_run_graph_destroy(void *graph) {
    if (graph) cudaGraphExecDestroy((cudaGraphExec_t)graph);
}

// Append a conditional IF node to the graph being captured on `s` (after
// everything captured so far) and return its body graph.
static cudaError_t capture_if_node(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraph_t *inner) {
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t ndeps = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &ndeps);
    if (e != cudaSuccess) return e;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, g, deps, ndeps, &cp);
    if (e != cudaSuccess) return e;
    e = cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
    *inner = cp.conditional.phGraph_out[0];
    return e;
}

struct SeedSpec {
    const void *vals;
    const uint32_t *words;
    const uint64_t *counts;  // host, 4 words, or null
};

static void *create_loop_graph(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                               const SeedSpec *seed);

void *wg_run_loop_graph_create(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                               void *stream) {
    (void)stream;
    return create_loop_graph(g, b, p, nullptr);
}

void *wg_run_loop_graph_create_seeded(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                                      const void *d_seed_values, const uint32_t *d_seed_words,
                                      const uint64_t *h_all_counts4, void *stream) {
    (void)stream;
    SeedSpec sp{d_seed_values, d_seed_words, h_all_counts4};
    return create_loop_graph(g, b, p, &sp);
}

int wg_run_loop_launch_seeded(void *graph, const wg_run_bufs *b, uint64_t max_iteration, const void *d_init_values,
                              void *d_seed_values, size_t value_bytes, const uint32_t *d_init_words,
                              uint32_t *d_seed_words, size_t word_bytes, void *stream) {
    WG_REQUIRE(graph && b && b->ctrl, "null argument");
    cudaStream_t s = as_stream(stream);
    // the caller's initial state into the buffers the graph reads
    if (d_init_values && d_init_values != d_seed_values && value_bytes)
        WG_CUDA(cudaMemcpyAsync(d_seed_values, d_init_values, value_bytes, cudaMemcpyDeviceToDevice, s));
    if (d_init_words && d_init_words != d_seed_words && word_bytes)
        WG_CUDA(cudaMemcpyAsync(d_seed_words, d_init_words, word_bytes, cudaMemcpyDeviceToDevice, s));
    set_limit_kernel<<<1, 1, 0, s>>>(b->ctrl, max_iteration);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("set_limit");
    WG_CUDA(cudaGraphLaunch((cudaGraphExec_t)graph, s));
    return WG_OK;
}

static void *create_loop_graph(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                               const SeedSpec *seed) {
    if (check_run(g, b, p)) return nullptr;
    // capture on private streams (the legacy default stream cannot capture)
    cudaStream_t s = nullptr, s2 = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) != cudaSuccess) {
        set_error("cudaStreamCreate failed");
        return nullptr;
    }
    struct StreamGuard {
        cudaStream_t a, b;
        ~StreamGuard() {
            if (a) cudaStreamDestroy(a);
            if (b) cudaStreamDestroy(b);
        }
    } guard{s, s2};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    if (cudaGraphCreate(&graph, 0) != cudaSuccess) {
        set_error("cudaGraphCreate failed");
        return nullptr;
    }
    // optional prologue: the run's seed (wg_run_seed) as the graph's first nodes
    std::vector<cudaGraphNode_t> pro;
    cudaError_t e = cudaSuccess;
    if (seed) {
        e = cudaStreamBeginCaptureToGraph(s, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        int rc = e == cudaSuccess ? seed_launches(g, b, p, seed->vals, seed->words, seed->counts, s, 1) : WG_OK;
        if (e == cudaSuccess) {
            cudaStreamCaptureStatus st;
            const cudaGraphNode_t *deps = nullptr;
            size_t nd = 0;
            e = cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd);
            if (e == cudaSuccess) pro.assign(deps, deps + nd);
            cudaGraph_t gout = nullptr;
            cudaError_t e2 = cudaStreamEndCapture(s, &gout);
            if (e == cudaSuccess) e = e2;
        }
        if (rc != WG_OK || e != cudaSuccess) {
            cudaGraphDestroy(graph);
            if (rc == WG_OK) cuda_fail(e, "seed prologue capture");
            return nullptr;
        }
    }
    cudaGraphConditionalHandle hw;
    e = cudaGraphConditionalHandleCreate(&hw, graph, 1, cudaGraphCondAssignDefault);
    // Before the WHILE node: one attempt of the persistent loop on the top
    // level, then a kernel that decides whether the WHILE body runs at all.
    // Runs the persistent kernel finishes on its own (CC s22, BFS s16, the
    // grid: every iteration is one of its phases) end right there instead of
    // walking the body's gate / IF nodes / finalize / step once more.
    if (e == cudaSuccess && g_sparse_loop && g->entries && g->nvec) {
        wg_run_params q0 = *p;
        q0.timer = nullptr;
        LoopCtx c0 = loop_ctx(g, b, &q0, b->ctrl, 1);
        PullBufs pb0 = pull_bufs(g, b, &q0);
        const uint64_t groups0 = groups_of(g, q0.shift);
        e = cudaStreamBeginCaptureToGraph(s, graph, pro.empty() ? nullptr : pro.data(), nullptr, pro.size(),
                                          cudaStreamCaptureModeThreadLocal);
        int rc0 = WG_OK;
        if (e == cudaSuccess) {
            // no gate / IF node here: the kernel itself returns at once when the
            // iteration about to run is not one of its kinds (its launch costs a
            // few microseconds, which only matter to the runs it does take)
            rc0 = launch_sparse_loop(c0, g, pb0, q0.val_type, q0.shift, &q0.kern, b->gbits, groups0, s);
            if (e == cudaSuccess && rc0 == WG_OK) {
                loop_enter_kernel<<<1, 1, 0, s>>>(hw, b->ctrl, b->recs, b->ring);
                ::wg::count_launch();
            }
            cudaStreamCaptureStatus st;
            const cudaGraphNode_t *deps = nullptr;
            size_t nd = 0;
            cudaError_t e1 = cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd);
            if (e1 == cudaSuccess) pro.assign(deps, deps + nd);
            cudaGraph_t gout = nullptr;
            cudaError_t e2 = cudaStreamEndCapture(s, &gout);
            if (e == cudaSuccess) e = e1 != cudaSuccess ? e1 : e2;
        }
        if (rc0 != WG_OK || e != cudaSuccess) {
            cudaGraphDestroy(graph);
            if (rc0 == WG_OK) cuda_fail(e, "pre-loop capture");
            return nullptr;
        }
    }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hw;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, graph, pro.empty() ? nullptr : pro.data(), pro.size(), &cp);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        cuda_fail(e, "conditional node");
        return nullptr;
    }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphConditionalHandle hf, hs, hp, hl;
    e = cudaGraphConditionalHandleCreate(&hf, body, 0, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hl, body, 0, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hs, body, 0, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hp, body, 0, cudaGraphCondAssignDefault);
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        cuda_fail(e, "loop body capture");
        return nullptr;
    }
    wg_run_params q = *p;
    q.timer = nullptr;
    LoopCtx c = loop_ctx(g, b, &q, b->ctrl, 1);
    const uint64_t groups = groups_of(g, q.shift);
    uint32_t *fv[2] = {b->fvert[0], b->fvert[1]};
    uint32_t *fp[2] = {b->fpref[0], b->fpref[1]};
    uint32_t *ts[2] = {b->tstart[0], b->tstart[1]};
    PullBufs pb = pull_bufs(g, b, &q);
    int rc = WG_OK;
    cudaGraph_t inner;
    // 0. as many consecutive sparse Wedge iterations as possible, persistently
    //    (IF the iteration about to run is one)
    if (g_sparse_loop && g->entries && g->nvec) {
        sparse_gate_kernel<<<1, 1, 0, s>>>(c, hl, groups, pb.loop_dense && !q.kern.use_weight ? 1u : 0u, g->n,
                                           q.kern.filter_unvisited ? 1 : 0);
        ::wg::count_launch();
        if ((e = capture_if_node(s, hl, &inner)) == cudaSuccess &&
            (e = cudaStreamBeginCaptureToGraph(s2, inner, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) ==
                cudaSuccess) {
            rc = launch_sparse_loop(c, g, pb, q.val_type, q.shift, &q.kern, b->gbits, groups, s2);
            e = cudaStreamEndCapture(s2, &inner);
        }
    }
    // 1. device-side gate: which of the three bodies runs this iteration
    if (rc == WG_OK && e == cudaSuccess) {
        decide_kernel<<<1, 1, 0, s>>>(c, hf, hs, hp, groups, g->entries > 0 ? 1 : 0);
        ::wg::count_launch();
    }
    // 2. IF FullScan: dense pull
    if (rc == WG_OK && e == cudaSuccess && (e = capture_if_node(s, hf, &inner)) == cudaSuccess &&
        (e = cudaStreamBeginCaptureToGraph(s2, inner, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) ==
            cudaSuccess) {
        if (g->nvec) rc = launch_pull(c, g, pb, q.val_type, q.shift, &q.kern, g->nvec, s2, MODE_FULL);
        e = cudaStreamEndCapture(s2, &inner);
    }
    // 3. IF Wedge (large frontier): transform -> ordered group list -> pull
    if (rc == WG_OK && e == cudaSuccess && (e = capture_if_node(s, hs, &inner)) == cudaSuccess &&
        (e = cudaStreamBeginCaptureToGraph(s2, inner, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) ==
            cudaSuccess) {
        if (g->entries) rc = launch_transform(c, g, fv, fp, ts, q.shift, b->gbits, s2);
        if (rc == WG_OK && groups)
            rc = launch_group_compaction(c, b->gbits, groups, b->bcount, b->glist, 1, q.shift, g->nvec, s2);
        if (rc == WG_OK && g->nvec) rc = launch_pull(c, g, pb, q.val_type, q.shift, &q.kern, g->nvec, s2, MODE_WEDGE);
        e = cudaStreamEndCapture(s2, &inner);
    }
    // 4. IF Wedge (sparse frontier): transform appends groups -> unsorted pull
    if (rc == WG_OK && e == cudaSuccess && (e = capture_if_node(s, hp, &inner)) == cudaSuccess &&
        (e = cudaStreamBeginCaptureToGraph(s2, inner, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) ==
            cudaSuccess) {
        if (g->entries) rc = launch_transform(c, g, fv, fp, ts, q.shift, b->gbits, s2, 1, b->glist, groups);
        if (rc == WG_OK && g->nvec) rc = launch_pull_sparse(c, g, pb, q.val_type, q.shift, &q.kern, b->gbits, groups, s2);
        e = cudaStreamEndCapture(s2, &inner);
    }
    // 5. end of iteration + loop control
    if (rc == WG_OK && e == cudaSuccess) {
        unsigned grid = (unsigned)sm_count() * 2;
        if (q.val_type == WG_VAL_U32)
            finalize_kernel<uint32_t><<<grid, 256, 0, s>>>(c, pb);
        else
            finalize_kernel<int64_t><<<grid, 256, 0, s>>>(c, pb);
        ::wg::count_launch();
        loop_step_kernel<<<1, 1, 0, s>>>(hw, b->ctrl, b->recs, b->ring);
        ::wg::count_launch();
    }
    cudaError_t e2 = cudaStreamEndCapture(s, &body);
    if (rc != WG_OK || e != cudaSuccess || e2 != cudaSuccess) {
        cudaGraphDestroy(graph);
        if (rc == WG_OK) cuda_fail(e != cudaSuccess ? e : e2, "loop body capture");
        return nullptr;
    }
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaGraphInstantiate");
        return nullptr;
    }
    return (void *)exec;
}

// Debug: phase timestamps of the persistent loop into a device buffer.
int wg_debug_kernel_timeline(uint64_t *d_buf, uint64_t iterations) {
    WG_CUDA(cudaMemcpyToSymbol(g_kts, &d_buf, sizeof(d_buf)));
    WG_CUDA(cudaMemcpyToSymbol(g_kts_cap, &iterations, sizeof(iterations)));
    return WG_OK;
}

uint32_t wg_debug_kernel_ids(void) { return (uint32_t)KTS_IDS; }

int wg_debug_phase_buffer(uint64_t *d_buf, uint64_t iterations) {
    WG_CUDA(cudaMemcpyToSymbol(g_phase_ts, &d_buf, sizeof(d_buf)));
    WG_CUDA(cudaMemcpyToSymbol(g_phase_cap, &iterations, sizeof(iterations)));
    return WG_OK;
}

int wg_run_persistent(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                      uint64_t max_iteration, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    set_limit_kernel<<<1, 1, 0, s>>>(b->ctrl, max_iteration);
    ::wg::count_launch();
    LoopCtx c = loop_ctx(g, b, p, b->ctrl, 1);
    PullBufs pb = pull_bufs(g, b, p);
    if (!g->entries || !g->nvec) return WG_OK;
    return launch_sparse_loop(c, g, pb, p->val_type, p->shift, &p->kern, b->gbits, groups_of(g, p->shift), s);
}

int wg_run_loop_launch(void *graph, const wg_run_bufs *b, uint64_t max_iteration, void *stream) {
    WG_REQUIRE(graph && b && b->ctrl, "null argument");
    cudaStream_t s = as_stream(stream);
    set_limit_kernel<<<1, 1, 0, s>>>(b->ctrl, max_iteration);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("set_limit");
    WG_CUDA(cudaGraphLaunch((cudaGraphExec_t)graph, s));
    return WG_OK;
}

// ------------------------------------------------------- exchange (K10) --
}  // extern "C"

namespace {

template <typename T>
__global__ void exchange_pack_kernel(const uint32_t *list, uint64_t nz, uint64_t z, uint32_t n,
                                     const T *vals, uint32_t *verts, T *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nz + z;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = i < nz ? list[i] : list[n - 1 - (i - nz)];
        verts[i] = v;
        out[i] = vals[v];
    }
}

template <typename T>
__global__ void exchange_apply_kernel(const uint32_t *verts, const T *in, uint64_t count, T *v0, T *v1,
                                      uint32_t *bits) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = verts[i];
        T x = in[i];
        v0[v] = x;
        v1[v] = x;
        atomicOr(&bits[v >> 5], 1u << (v & 31));
    }
}

// Packed exchange: a rank's buffer is a 16-byte header (u64 entry count)
// followed by (vertex, value) entries, 8 bytes (u32 values) or 16 bytes
// (int64 values); any prefix of it is a valid, truncated message.
template <typename T>
struct XEntry {
    uint32_t v;
    uint32_t pad;
    T x;
};
template <>
struct XEntry<uint32_t> {
    uint32_t v;
    uint32_t x;
};

template <typename T>
__global__ void exchange_pack_all_kernel(const wg_iter_rec *rec, const uint32_t *list, uint32_t n, const T *vals,
                                         unsigned char *buf, uint64_t capacity) {
    const uint64_t nz = rec->nz_packed >> 32, z = rec->z_count;
    const uint64_t cnt = nz + z;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        reinterpret_cast<uint64_t *>(buf)[0] = cnt;
        reinterpret_cast<uint64_t *>(buf)[1] = rec->overflow;  // every rank learns of an overflow
    }
    XEntry<T> *e = reinterpret_cast<XEntry<T> *>(buf + 16);
    const uint64_t m = cnt < capacity ? cnt : capacity;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = i < nz ? list[i] : list[n - 1 - (i - nz)];
        XEntry<T> t{};
        t.v = v;
        t.x = vals[v];
        e[i] = t;
    }
}

// Applies the first min(count, cap) entries of every rank's part; status[0]
// receives the largest count (> cap: the gather was truncated, redo it).
template <typename T>
__global__ void exchange_apply_all_kernel(const unsigned char *parts, uint32_t world, uint64_t cap,
                                          uint64_t stride, T *v0, T *v1, uint32_t *bits, uint64_t *status) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint32_t r = 0; r < world; ++r) {
        const unsigned char *pr = parts + (uint64_t)r * stride;
        const uint64_t cnt = *reinterpret_cast<const uint64_t *>(pr);
        if (tid == 0) {
            atomicMax((unsigned long long *)status, (unsigned long long)cnt);
            if (reinterpret_cast<const uint64_t *>(pr)[1]) status[1] = 1;
        }
        const uint64_t m = cnt < cap ? cnt : cap;
        const XEntry<T> *e = reinterpret_cast<const XEntry<T> *>(pr + 16);
        for (uint64_t i = tid; i < m; i += nth) {
            const XEntry<T> t = e[i];
            v0[t.v] = t.x;
            v1[t.v] = t.x;
            atomicOr(&bits[t.v >> 5], 1u << (t.v & 31));
        }
    }
}

// Dense-iteration form: every rank's owned value slice (S values each, rank r
// owning [bounds[r], bounds[r+1])).  A destination of another rank changed
// iff its new value is below the replicated previous one (values never
// increase; this rank's end of iteration synced only its own members), so
// those frontier bits come from the values; this rank's own bits are its
// pull's.  A thread per bitmap word.
template <typename T>
__global__ void exchange_slices_kernel(const T *slices, const uint32_t *bounds, uint32_t world, uint32_t self,
                                       uint64_t S, uint32_t n, const T *prev, T *v0, T *v1, uint32_t *bits) {
    const uint64_t words = ((uint64_t)n + 31) >> 5;
    const uint64_t lo = bounds[self], hi = bounds[self + 1];
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t own = bits[w];
        uint32_t word = 0, r = 0;
        for (uint32_t j = 0; j < 32; ++j) {
            const uint64_t d = (w << 5) + j;
            if (d >= n) break;
            while (r + 1 < world && d >= bounds[r + 1]) ++r;
            const T x = slices[(uint64_t)r * S + (d - bounds[r])];
            if (d >= lo && d < hi) word |= own & (1u << j);
            else if (x < prev[d]) word |= 1u << j;
            v0[d] = x;
            v1[d] = x;
        }
        bits[w] = word;
    }
}

}  // namespace

extern "C" {

int wg_exchange_slice_pack(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                           uint32_t lo, uint32_t hi, void *d_slice, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    WG_REQUIRE(d_slice || hi == lo, "null argument");
    WG_REQUIRE(lo <= hi && hi <= g->n, "bad owned range");
    const size_t vb = p->val_type == WG_VAL_U32 ? 4 : 8;
    if (hi > lo)
        WG_CUDA(cudaMemcpyAsync(d_slice, (const char *)b->vals[it & 1] + lo * vb, (size_t)(hi - lo) * vb,
                                cudaMemcpyDeviceToDevice, as_stream(stream)));
    return WG_OK;
}

int wg_exchange_apply_slices(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                             const void *d_slices, const uint32_t *d_bounds, uint32_t world, uint32_t self,
                             uint64_t S, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    WG_REQUIRE(d_slices && d_bounds && world >= 1 && self < world, "bad argument");
    cudaStream_t s = as_stream(stream);
    uint32_t *bits = b->fbits[it & 1];
    const uint64_t words = ((uint64_t)g->n + 31) >> 5;
    const unsigned grid = grid_for(words ? words : 1, 256, 8);
    if (p->val_type == WG_VAL_U32)
        exchange_slices_kernel<uint32_t><<<grid, 256, 0, s>>>(
            (const uint32_t *)d_slices, d_bounds, world, self, S, g->n, (const uint32_t *)b->vals[(it - 1) & 1],
            (uint32_t *)b->vals[0], (uint32_t *)b->vals[1], bits);
    else
        exchange_slices_kernel<int64_t><<<grid, 256, 0, s>>>(
            (const int64_t *)d_slices, d_bounds, world, self, S, g->n, (const int64_t *)b->vals[(it - 1) & 1],
            (int64_t *)b->vals[0], (int64_t *)b->vals[1], bits);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("exchange_apply_slices");
    return launch_frontier_compaction(g, bits, b->bcount, bcount_ticket(g, p->shift, b->bcount),
                                      b->fvert[it & 1], b->fpref[it & 1], b->tstart[it & 1],
                                      &b->recs[it % b->ring], s);
}

uint64_t wg_exchange_bytes(uint64_t entries, int val_type) {
    return 16 + entries * (val_type == WG_VAL_U32 ? sizeof(XEntry<uint32_t>) : sizeof(XEntry<int64_t>));
}

int wg_exchange_pack_all(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                         void *d_buf, uint64_t capacity, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    WG_REQUIRE(d_buf, "null argument");
    cudaStream_t s = as_stream(stream);
    unsigned grid = grid_for(capacity ? capacity : 1, 256 * 4, 8);
    const uint32_t *list = b->fvert[it & 1];
    const wg_iter_rec *rec = &b->recs[it % b->ring];
    if (p->val_type == WG_VAL_U32)
        exchange_pack_all_kernel<uint32_t><<<grid, 256, 0, s>>>(rec, list, g->n, (const uint32_t *)b->vals[it & 1],
                                                                (unsigned char *)d_buf, capacity);
    else
        exchange_pack_all_kernel<int64_t><<<grid, 256, 0, s>>>(rec, list, g->n, (const int64_t *)b->vals[it & 1],
                                                               (unsigned char *)d_buf, capacity);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("exchange_pack_all");
    return WG_OK;
}

int wg_exchange_apply_all(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                          const void *d_parts, uint32_t world, uint64_t cap, uint64_t *d_status,
                          void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    WG_REQUIRE(d_parts && d_status && world >= 1, "null argument");
    cudaStream_t s = as_stream(stream);
    uint32_t *bits = b->fbits[it & 1];
    const uint64_t stride = wg_exchange_bytes(cap, p->val_type);
    WG_CUDA(cudaMemsetAsync(d_status, 0, 2 * sizeof(uint64_t), s));
    unsigned grid = grid_for(cap ? cap : 1, 256 * 4, 8);
    if (p->val_type == WG_VAL_U32)
        exchange_apply_all_kernel<uint32_t><<<grid, 256, 0, s>>>((const unsigned char *)d_parts, world, cap, stride,
                                                                 (uint32_t *)b->vals[0], (uint32_t *)b->vals[1],
                                                                 bits, d_status);
    else
        exchange_apply_all_kernel<int64_t><<<grid, 256, 0, s>>>((const unsigned char *)d_parts, world, cap, stride,
                                                                (int64_t *)b->vals[0], (int64_t *)b->vals[1],
                                                                bits, d_status);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("exchange_apply_all");
    return launch_frontier_compaction(g, bits, b->bcount, bcount_ticket(g, p->shift, b->bcount),
                                      b->fvert[it & 1], b->fpref[it & 1], b->tstart[it & 1],
                                      &b->recs[it % b->ring], s);
}

int wg_exchange_pack(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                     uint32_t *d_verts, void *d_vals, uint64_t capacity, uint64_t *h_count,
                     void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    WG_REQUIRE(d_verts && d_vals && h_count, "null argument");
    cudaStream_t s = as_stream(stream);
    wg_iter_rec h;
    WG_CUDA(cudaMemcpyAsync(&h, &b->recs[it % b->ring], sizeof(h), cudaMemcpyDeviceToHost, s));
    WG_CUDA(cudaStreamSynchronize(s));
    uint64_t nz = h.nz_packed >> 32, z = h.z_count;
    *h_count = nz + z;
    if (nz + z > capacity) {
        set_error("exchange capacity %llu < %llu", (unsigned long long)capacity,
                  (unsigned long long)(nz + z));
        return WG_ENOSPACE;
    }
    if (nz + z == 0) return WG_OK;
    unsigned grid = grid_for(nz + z, 256 * 4, 8);
    const uint32_t *list = b->fvert[it & 1];
    if (p->val_type == WG_VAL_U32)
        exchange_pack_kernel<uint32_t><<<grid, 256, 0, s>>>(list, nz, z, g->n,
                                                            (const uint32_t *)b->vals[it & 1], d_verts,
                                                            (uint32_t *)d_vals);
    else
        exchange_pack_kernel<int64_t><<<grid, 256, 0, s>>>(list, nz, z, g->n,
                                                           (const int64_t *)b->vals[it & 1], d_verts,
                                                           (int64_t *)d_vals);
    ::wg::count_launch();
    WG_CHECK_LAUNCH("exchange_pack");
    return WG_OK;
}

int wg_exchange_apply(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                      const uint32_t *d_verts, const void *d_vals, uint64_t count, void *stream) {
    int rc = check_run(g, b, p);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    uint32_t *bits = b->fbits[it & 1];
    if (count) {
        WG_REQUIRE(d_verts && d_vals, "null argument");
        unsigned grid = grid_for(count, 256 * 4, 8);
        if (p->val_type == WG_VAL_U32)
            exchange_apply_kernel<uint32_t><<<grid, 256, 0, s>>>(
                d_verts, (const uint32_t *)d_vals, count, (uint32_t *)b->vals[0], (uint32_t *)b->vals[1], bits);
        else
            exchange_apply_kernel<int64_t><<<grid, 256, 0, s>>>(
                d_verts, (const int64_t *)d_vals, count, (int64_t *)b->vals[0], (int64_t *)b->vals[1], bits);
        ::wg::count_launch();
        WG_CHECK_LAUNCH("exchange_apply");
    }
    // the global frontier of `it`: ordered list, index prefixes, counts and
    // the global out-degree sum (the next gate's input) from the bitmap
    return launch_frontier_compaction(g, bits, b->bcount, bcount_ticket(g, p->shift, b->bcount),
                                      b->fvert[it & 1], b->fpref[it & 1],
                                      b->tstart[it & 1], &b->recs[it % b->ring], s);
}

}  // extern "C"
