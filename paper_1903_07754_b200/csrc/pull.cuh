// pull.cuh — the atomic-free, warp-segmented min-plus pull (K5 wedge / K6 dense).
//
// Reference semantics (engine.py:251-327; _kernels.pyx:65-95, 113-173):
// per destination d, agg = min over processed in-lanes of prev[src] (+ weight);
// cand = agg + inc; d is updated (nxt[d] = cand) and activated (next-frontier
// bit) iff cand < prev[d].  BFS skips destinations already visited and does
// not count their vectors as touched.
//
// B200 mapping: a warp consumes a tile of 32 work items, one vector per lane
// (dense mode: consecutive vectors; wedge mode: vectors of the selected groups,
// ascending).  Each lane streams its vector's W lanes with one vector load,
// gathers prev[src], and reduces locally; a 5-step segmented min-scan keyed by
// destination combines the lanes of equal destinations.  The tail lane of each
// segment applies.  Only a segment that touches the tile's first or last lane
// AND continues in the neighbouring work item can be shared with another warp;
// those (at most two per tile) use atomicMin, every other destination is a
// plain store.  The next-frontier bitmap, the produced member list (with the
// edge-index prefix the next transform balances on), the out-degree sum (next
// gate input) and the work counters are all emitted in the same kernel.
#pragma once
#include "loop.cuh"

namespace wg {

template <typename T>
struct ValTraits;
template <>
struct ValTraits<uint32_t> {
    static constexpr bool U32 = true;
    __device__ static uint32_t inf(int64_t) { return 0xffffffffu; }
};
template <>
struct ValTraits<int64_t> {
    static constexpr bool U32 = false;
    __device__ static int64_t inf(int64_t sentinel) { return sentinel; }
};

struct PullBufs {
    void *vals[2];
    uint32_t *fbits[2];
    uint32_t *fvert[2];
    uint32_t *fpref[2];
    const uint32_t *glist;
    uint32_t n;
};

__device__ __forceinline__ uint64_t min_u64(uint64_t a, uint64_t b) { return a < b ? a : b; }

template <typename T>
__device__ __forceinline__ T shfl_up_t(T v, int off) {
    if constexpr (sizeof(T) == 8) {
        return (T)__shfl_up_sync(FULL, (unsigned long long)v, off);
    } else {
        return (T)__shfl_up_sync(FULL, (unsigned)v, off);
    }
}

// Map work item k to a vector position (or ~0 when out of range).
__device__ __forceinline__ uint64_t item_pos(uint64_t k, uint64_t nitems, bool wedge,
                                             const uint32_t *glist, int shift, uint64_t nvec) {
    if (k >= nitems) return ~0ull;
    if (!wedge) return k;
    uint64_t p = ((uint64_t)glist[k >> shift] << shift) | (k & ((1ull << shift) - 1));
    return p < nvec ? p : ~0ull;
}

template <typename T, int W, bool WEIGHT, bool FILTER>
__global__ void __launch_bounds__(256) pull_kernel(LoopCtx c, wg_graph g, PullBufs b, int shift,
                                                   int64_t inc, int64_t sentinel) {
    using VT = ValTraits<T>;
    const uint64_t it = ctx_iter(c);
    const int mode = ctx_mode(c, it);
    if (mode == MODE_NONE) return;
    const bool wedge = (mode == MODE_WEDGE);
    wg_iter_rec *out = ctx_out(c, it);
    const T *__restrict__ prev = (const T *)b.vals[(it - 1) & 1];
    T *__restrict__ nxt = (T *)b.vals[it & 1];
    uint32_t *__restrict__ obits = b.fbits[it & 1];
    uint32_t *__restrict__ overt = b.fvert[it & 1];
    uint32_t *__restrict__ opref = b.fpref[it & 1];
    const uint64_t nitems = wedge ? (out->groups << shift) : g.nvec;
    const T INF = VT::inf(sentinel);
    const unsigned lane = lane_id();
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t ntiles = (nitems + 31) >> 5;
    uint64_t touched = 0;
    uint32_t ovf = 0;

    for (uint64_t tile = gwarp; tile < ntiles; tile += nwarps) {
        const uint64_t k = (tile << 5) + lane;
        const uint64_t p = item_pos(k, nitems, wedge, b.glist, shift, g.nvec);
        const bool valid = p != ~0ull;
        const uint32_t d = valid ? g.vdst[p] : 0xffffffffu;
        T pd = INF;
        if (FILTER && valid) pd = prev[d];
        const bool active = valid && !(FILTER && pd != INF);
        T agg = INF;
        if (active) {
            uint32_t src[W];
            load_lanes<W>(g.vsrc, p, src);
            uint32_t wt[W];
            if (WEIGHT) load_lanes<W>(g.vw, p, wt);
#pragma unroll
            for (int l = 0; l < W; ++l) {
                if (src[l] == WG_NO_LANE) continue;
                T ps = prev[src[l]];
                if constexpr (VT::U32) {
                    if (ps == INF) continue;
                    uint64_t m = (uint64_t)ps + (WEIGHT ? wt[l] : 0u);
                    if (m >= 0xffffffffull) { ovf = 1; continue; }
                    agg = (T)min_u64(agg, m);
                } else {
                    T m = ps + (WEIGHT ? (T)wt[l] : (T)0);
                    agg = m < agg ? m : agg;
                }
            }
        }
        touched += __popc(__ballot_sync(FULL, active));

        // segmented inclusive min-scan keyed by destination
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            T o = shfl_up_t(agg, off);
            uint32_t od = __shfl_up_sync(FULL, d, off);
            if ((int)lane >= off && od == d && o < agg) agg = o;
        }
        const uint32_t dn = __shfl_down_sync(FULL, d, 1);
        const uint32_t dp = __shfl_up_sync(FULL, d, 1);
        const bool head = lane == 0 || dp != d;
        const bool tail = lane == 31 || dn != d;
        const unsigned heads = __ballot_sync(FULL, head);
        const unsigned head_lane = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));

        bool newly = false;
        if (tail && active) {
            // complete iff no neighbouring work item (outside the tile) has d
            bool complete = true;
            if (head_lane == 0 && (tile << 5) > 0) {
                uint64_t q = item_pos((tile << 5) - 1, nitems, wedge, b.glist, shift, g.nvec);
                if (q != ~0ull && g.vdst[q] == d) complete = false;
            }
            if (lane == 31) {
                uint64_t q = item_pos((tile << 5) + 32, nitems, wedge, b.glist, shift, g.nvec);
                if (q != ~0ull && g.vdst[q] == d) complete = false;
            }
            if (!FILTER) pd = prev[d];
            bool upd;
            T cand;
            if constexpr (VT::U32) {
                upd = false;
                if (agg != INF) {
                    uint64_t cc = (uint64_t)agg + (uint64_t)inc;
                    if (cc >= 0xffffffffull) {
                        ovf = 1;
                    } else {
                        cand = (T)cc;
                        upd = cand < pd;
                    }
                }
            } else {
                cand = agg + (T)inc;
                upd = cand < pd;
            }
            if (upd) {
                if (complete) {
                    nxt[d] = cand;
                } else {
                    if constexpr (VT::U32) atomicMin((unsigned *)&nxt[d], (unsigned)cand);
                    else atomicMin((long long *)&nxt[d], (long long)cand);
                }
                const uint32_t bit = 1u << (d & 31);
                newly = !(atomicOr(&obits[d >> 5], bit) & bit);
            }
        }

        // warp-aggregated append of newly activated destinations
        const unsigned nm = __ballot_sync(FULL, newly);
        if (nm) {
            uint32_t len = 0, od = 0;
            if (newly) {
                len = (uint32_t)(g.idx_off[d + 1] - g.idx_off[d]);
                od = g.outdeg[d];
            }
            const bool nz = newly && len > 0;
            const unsigned nzm = __ballot_sync(FULL, nz);
            const unsigned zm = nm & ~nzm;
            const uint32_t incl = warp_inclusive_sum(nz ? len : 0u);
            const uint32_t tot = __shfl_sync(FULL, incl, 31);
            const uint64_t osum = warp_sum((uint64_t)od);
            unsigned long long base = 0, zbase = 0;
            if (lane == 0) {
                if (nzm)
                    base = atomicAdd((unsigned long long *)&out->nz_packed,
                                     ((unsigned long long)__popc(nzm) << 32) | tot);
                if (zm) zbase = atomicAdd((unsigned long long *)&out->z_count,
                                          (unsigned long long)__popc(zm));
                atomicAdd((unsigned long long *)&out->out_edge_sum, (unsigned long long)osum);
            }
            base = __shfl_sync(FULL, base, 0);
            zbase = __shfl_sync(FULL, zbase, 0);
            if (nz) {
                uint64_t pos = (base >> 32) + __popc(nzm & lanemask_lt());
                overt[pos] = d;
                opref[pos] = (uint32_t)(base & 0xffffffffull) + (incl - len);
            } else if (newly) {
                uint64_t zpos = zbase + __popc(zm & lanemask_lt());
                overt[b.n - 1 - zpos] = d;
            }
        }
    }
    touched = warp_sum(touched) / 32;  // every lane counted the same ballots
    ovf = __any_sync(FULL, ovf);
    if (lane == 0) {
        if (touched) atomicAdd((unsigned long long *)&out->vectors_touched, (unsigned long long)touched);
        if (ovf) out->overflow = 1;
    }
}

// ---------------- K7: end of iteration -------------------------------------
// Keeps the strict double buffer coherent in O(|F|) instead of the
// reference's O(V) copy-forward (engine.py:198-202, 264, 300): the two value
// buffers differ exactly at the vertices updated this iteration, so those are
// copied into the buffer the next iteration writes.  Also clears the output
// bitmap of iteration it-1 (reused by it+1), finalises the record and zeroes
// the record the next iteration will fill.
template <typename T>
__global__ void __launch_bounds__(256) finalize_kernel(LoopCtx c, PullBufs b) {
    const uint64_t it = ctx_iter(c);
    const int mode = ctx_mode(c, it);
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    if (mode != MODE_NONE) {
        const wg_iter_rec *out = ctx_out(c, it);
        const wg_iter_rec *in = ctx_in(c, it);
        const T *src = (const T *)b.vals[it & 1];
        T *dst = (T *)b.vals[(it - 1) & 1];
        const uint32_t *list = b.fvert[it & 1];
        uint64_t nz = out->nz_packed >> 32, z = out->z_count;
        for (uint64_t i = tid; i < nz + z; i += nthreads) {
            uint32_t v = i < nz ? list[i] : list[b.n - 1 - (i - nz)];
            dst[v] = src[v];
        }
        // clear bits of the frontier produced by it-1 (its bitmap is reused by it+1)
        uint32_t *obits = b.fbits[(it - 1) & 1];
        const uint32_t *plist = b.fvert[(it - 1) & 1];
        uint64_t pnz = in->nz_packed >> 32, pz = in->z_count;
        uint64_t words = ((uint64_t)b.n + 31) >> 5;
        if (pnz + pz > words) {
            for (uint64_t w = tid; w < words; w += nthreads) obits[w] = 0;
        } else {
            for (uint64_t i = tid; i < pnz + pz; i += nthreads) {
                uint32_t v = i < pnz ? plist[i] : plist[b.n - 1 - (i - pnz)];
                obits[v >> 5] = 0;
            }
        }
    }
    if (tid == 0) {
        wg_iter_rec *out = ctx_out(c, it);
        if (mode != MODE_NONE) {
            out->mode = (uint64_t)mode;
            out->frontier_out = (out->nz_packed >> 32) + out->z_count;
            out->active_edges = ctx_in(c, it)->out_edge_sum;
        }
        wg_iter_rec *nx = &c.recs[(it + 1) % c.ring];
        uint64_t *q = (uint64_t *)nx;
#pragma unroll
        for (int i = 0; i < 16; ++i) q[i] = 0;
    }
}

__global__ void bump_counter_kernel(uint64_t *ctrl, uint64_t by) { ctrl[0] += by; }

}  // namespace wg
