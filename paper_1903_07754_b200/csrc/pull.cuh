// pull.cuh — the warp-segmented min-plus pull (K5 wedge / K6 dense).
//
// Reference semantics (engine.py:251-327; _kernels.pyx:65-95, 113-173):
// per destination d, agg = min over processed in-lanes of prev[src] (+ weight);
// cand = agg + inc; d is updated (nxt[d] = cand) and activated (next-frontier
// bit) iff cand < prev[d].  BFS skips destinations already visited and does
// not count their vectors as touched.
//
// B200 mapping.  Every warp owns a contiguous range of 32-item tiles (dense:
// consecutive vectors; wedge: the vectors of the selected groups) and walks it
// in order, one vector per lane.  Lanes gather prev[src] for their W lanes and
// fold them; equal destinations are combined with a shuffle min-scan limited
// to the longest segment of the tile (a REDUX with per-segment lane masks
// serialises per mask).  The segment touching lane 31 is CARRIED into the next
// tile, so a destination is applied once, by one lane, with a plain store --
// atomicMin only for a run shared with a neighbouring warp's range.  Sparse /
// Wedge pulls also produce the next-frontier member list (staged per warp in
// shared memory, one atomic per 32 members), its out-degree sum (the next
// gate's input) and the work counter in the same kernel; dense pulls set
// bitmap bits only and the list is built afterwards when a Wedge iteration
// will consume it.
//
// Dense pulls stream the edge layout with TMA bulk copies (cp.async.bulk +
// mbarrier, a per-warp ring in shared memory, tma.cuh) and software-pipeline
// the gathers across chunks; Wedge pulls load their vectors directly.  The
// persistent sparse loop runs consecutive sparse Wedge iterations in one
// cooperative launch (grid barriers between phases).
#pragma once
#include <cooperative_groups.h>

#include "frontier.cuh"
#include "loop.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

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
    uint32_t *tstart[2];
    uint64_t *bcount;  // compaction scratch (dense-pull frontier build)
    unsigned *ticket;  // its completion ticket
    const uint32_t *glist;
    uint32_t *gbits2, *glist2;  // second group bitmap / list (fused persistent loop) or null
    uint32_t n;
    uint32_t first_hit;  // WG_RUN_FIRST_HIT (filtered pulls only)
    uint32_t ident;      // WG_RUN_IDENTITY_INIT
    uint32_t floor_skip; // WG_RUN_FLOOR_SKIP: dense pulls skip destinations already at 0
    uint32_t floor_kernels;  // ... and from iteration floor_from on run floor_pull_kernel
    uint32_t floor_from;
    uint64_t pipeline_until = ~0ull;  // dense iterations >= this one skip the TMA pipeline (plain kernels)
    int64_t level_base;  // its frontier-0 value
    uint32_t *work;      // wg_run_bufs.work: destination list of the destination-major dense pulls
    uint32_t dst_major;  // dense iterations run dense_dst_kernel (DSTK_FLOOR / DSTK_BOTTOM_UP)
    uint32_t loop_dense; // ... and the persistent loop runs them as phases (WG_LOOP_DENSE=0: off)
    uint32_t dst_light;  // destination-major pulls: in-lists up to this many vectors are walked by one lane
};


#ifndef SPARSE_MINB
#define SPARSE_MINB 3
#endif
#ifndef SPARSE_U
#define SPARSE_U 2
#endif
// a Wedge iteration is "sparse" when its index entries * this < groups
constexpr uint64_t SPARSE_ENTRY_RATIO = 8;
constexpr uint64_t PERSIST_MAX_ENTRIES = 1ull << 24;
constexpr uint32_t NONE = 0xffffffffu;

template <typename T>
__device__ __forceinline__ T shfl_t(T v, int src) {
    if constexpr (sizeof(T) == 8) return (T)__shfl_sync(FULL, (unsigned long long)v, src);
    else return (T)__shfl_sync(FULL, (unsigned)v, src);
}
template <typename T>
__device__ __forceinline__ T warp_min_t(T v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        T o;
        if constexpr (sizeof(T) == 8) o = (T)__shfl_xor_sync(FULL, (unsigned long long)v, off);
        else o = (T)__shfl_xor_sync(FULL, (unsigned)v, off);
        v = o < v ? o : v;
    }
    return v;
}
template <typename T>
__device__ __forceinline__ T shfl_up_t(T v, int off) {
    if constexpr (sizeof(T) == 8) return (T)__shfl_up_sync(FULL, (unsigned long long)v, off);
    else return (T)__shfl_up_sync(FULL, (unsigned)v, off);
}


// Map work item k to a vector position (or ~0 when out of range).
__device__ __forceinline__ uint64_t item_pos(uint64_t k, uint64_t nitems, bool wedge,
                                             const uint32_t *glist, int shift, uint64_t nvec) {
    if (k >= nitems) return ~0ull;
    if (!wedge) return k;
    uint64_t p = ((uint64_t)glist[k >> shift] << shift) | (k & ((1ull << shift) - 1));
    return p < nvec ? p : ~0ull;
}

// ---------------------------------------------------------------------------
// Per-warp output: counters in registers, frontier list staged in smem.
struct PullOut {
    uint32_t *stage;
    uint32_t staged;    // warp-uniform
    uint64_t edge_sum;  // per lane
    uint64_t touched;   // lane 0
    uint32_t ovf;
};

// Fused transform of the NEXT iteration (persistent sparse loop): the warp
// that adds vertices to the produced frontier also maps their edge-index
// entries to Wedge groups (frontier.py:174-209), into the other group
// bitmap / list buffer, so iteration it+1 needs no transform phase.
constexpr uint32_t FUSED_MAX_LEN = 256;  // longer index lists: transform phase next iteration

struct FusedT {
    uint32_t *gbits;          // group bitmap of iteration it+1 (zero on entry)
    uint32_t *glist;          // its appended group list
    wg_iter_rec *rec;         // its record: groups, clipped-last-group flag
    const uint32_t *idx_pos;
    int shift;
    uint64_t ngroups;
};

// The 32 staged vertices of one flush round own entry ranges [excl, excl+len)
// of a warp-local prefix; lanes walk the concatenation 32 entries at a time
// (owner found by a shuffle binary search), so a hub's entries are spread
// over the warp.
__device__ __forceinline__ void fused_append(const FusedT &fx, uint64_t off0, uint32_t excl, uint32_t tot) {
    constexpr int R = 4;  // rounds of 32 entries whose loads / atomics are in flight together
    const unsigned lane = lane_id();
    for (uint32_t k0 = 0; k0 < tot; k0 += 32 * R) {
        uint32_t gid[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t k = k0 + r * 32 + lane;
            int own = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const int cand = own + step;
                const uint32_t e = __shfl_sync(FULL, excl, cand & 31);
                if (cand < 32 && e <= k) own = cand;
            }
            const uint64_t base = __shfl_sync(FULL, off0, own);
            const uint32_t pre = __shfl_sync(FULL, excl, own);
            gid[r] = k < tot ? fx.idx_pos[base + (k - pre)] >> fx.shift : NONE;
        }
        bool fresh[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            // a source's positions ascend: equal groups are adjacent
            const uint32_t gprev = __shfl_up_sync(FULL, gid[r], 1);
            fresh[r] = false;
            if (gid[r] != NONE && !(lane > 0 && gprev == gid[r])) {
                const uint32_t bit = 1u << (gid[r] & 31);
                fresh[r] = !(atomicOr(&fx.gbits[gid[r] >> 5], bit) & bit);
            }
        }
        unsigned fm[R], cnt = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            fm[r] = __ballot_sync(FULL, fresh[r]);
            cnt += __popc(fm[r]);
        }
        if (cnt) {
            unsigned long long at = 0;
            if (lane == 0) at = atomicAdd((unsigned long long *)&fx.rec->groups, (unsigned long long)cnt);
            at = __shfl_sync(FULL, at, 0);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (fresh[r]) {
                    fx.glist[at + __popc(fm[r] & lanemask_lt())] = gid[r];
                    if (gid[r] == fx.ngroups - 1) fx.rec->reserved[1] = 1;  // the clipped last group
                }
                at += __popc(fm[r]);
            }
        }
    }
}

__device__ __forceinline__ void flush_stage(PullOut &o, const wg_graph &g, wg_iter_rec *out,
                                            uint32_t *overt, uint32_t *opref, uint32_t *otstart,
                                            uint32_t n, const FusedT *fx = nullptr) {
    const unsigned lane = lane_id();
    for (uint32_t base = 0; base < o.staged; base += 32) {
        const bool have = base + lane < o.staged;
        const uint32_t d = have ? o.stage[base + lane] : 0u;
        uint32_t len = 0;
        uint64_t off0 = 0;
        if (have) {
            off0 = g.idx_off[d];
            len = (uint32_t)(g.idx_off[d + 1] - off0);
            o.edge_sum += g.outdeg[d];
        }
        const bool nz = have && len > 0;
        const unsigned nzm = __ballot_sync(FULL, nz);
        const unsigned zm = __ballot_sync(FULL, have) & ~nzm;
        const uint32_t incl = warp_inclusive_sum(nz ? len : 0u);
        const uint32_t tot = __shfl_sync(FULL, incl, 31);
        unsigned long long nzb = 0, zb = 0;
        if (lane == 0) {
            if (nzm)
                nzb = atomicAdd((unsigned long long *)&out->nz_packed,
                                ((unsigned long long)__popc(nzm) << 32) | tot);
            if (zm) zb = atomicAdd((unsigned long long *)&out->z_count, (unsigned long long)__popc(zm));
        }
        nzb = __shfl_sync(FULL, nzb, 0);
        zb = __shfl_sync(FULL, zb, 0);
        if (nz) {
            const uint64_t pos = (nzb >> 32) + __popc(nzm & lanemask_lt());
            const uint32_t pref = (uint32_t)(nzb & 0xffffffffull) + (incl - len);
            overt[pos] = d;
            opref[pos] = pref;
            if (otstart) mark_tile_starts(otstart, pref, len, (uint32_t)pos);
        } else if (have) {
            overt[n - 1 - (zb + __popc(zm & lanemask_lt()))] = d;
        }
        if (fx) {
            // vertices with long index lists are left to a regular transform
            // phase of the next iteration (one warp would serialise them)
            const bool big = nz && len > FUSED_MAX_LEN;
            if (__any_sync(FULL, big) && lane == 0) fx->rec->reserved[3] = 1;
            const uint32_t flen = (nz && !big) ? len : 0u;
            const uint32_t fincl = warp_inclusive_sum(flen);
            fused_append(*fx, off0, fincl - flen, __shfl_sync(FULL, fincl, 31));
        }
    }
    __syncwarp();
    o.staged = 0;
}

// Collective apply, one segment per flagged lane (the min-plus update rule,
// _kernels.pyx:91-94): plain store when the segment is complete, atomicMin
// when another warp may hold part of it; one atomicOr per run of updating
// lanes sharing a bitmap word; newly set destinations are staged.
template <typename T>
__device__ __forceinline__ void apply_segments(bool app, uint32_t d, T agg, T pd, bool complete,
                                               T INF, int64_t inc, T *nxt, uint32_t *obits,
                                               PullOut &o) {
    using VT = ValTraits<T>;
    const unsigned lane = lane_id();
    bool upd = false;
    T cand = agg;
    if (app) {
        if constexpr (VT::U32) {
            if (agg != INF) {
                uint64_t cc = (uint64_t)agg + (uint64_t)inc;
                if (cc >= 0xffffffffull) o.ovf = 1;
                else {
                    cand = (T)cc;
                    upd = cand < pd;
                }
            }
        } else {
            cand = agg + (T)inc;
            upd = cand < pd;
        }
    }
    if (__ballot_sync(FULL, upd) == 0) return;
    bool newly = false;
    if (upd) {
        const uint32_t bit = 1u << (d & 31);
        if (complete) {
            // the only writer of d this iteration: the bit is new (the bitmap
            // was cleared by the previous end-of-iteration kernel)
            nxt[d] = cand;
            atomicOr(&obits[d >> 5], bit);
            newly = true;
        } else {
            if constexpr (VT::U32) atomicMin((unsigned *)&nxt[d], (unsigned)cand);
            else atomicMin((long long *)&nxt[d], (long long)cand);
            newly = !(atomicOr(&obits[d >> 5], bit) & bit);
        }
    }
    const unsigned nm = __ballot_sync(FULL, newly);
    if (newly) o.stage[o.staged + __popc(nm & lanemask_lt())] = d;
    __syncwarp();
    o.staged += __popc(nm);
}

// Dense-mode apply: values and next-frontier bits only; the member list, its
// index-length prefixes and the out-degree sum are produced afterwards by the
// ordered bitmap compaction (frontier_count/list kernels), which is cheaper
// than staging ~V appends inside the pull.
// The dense pull writes EVERY destination it covers (min(prev[d], cand)), so
// after a dense iteration nxt holds the full value vector and no buffer sync
// is needed when the next iteration is dense too (end_of_iteration).  Shared
// (incomplete) segments use atomicMin, which is exact because values never
// increase: the stale nxt[d] (two iterations old) is >= prev[d].
// The value part of a dense apply; returns the next-frontier bit to set (0 if
// d did not improve).
template <typename T>
__device__ __forceinline__ uint32_t apply_dense_value(bool app, uint32_t d, T agg, T pd, bool complete, T INF,
                                                      int64_t inc, T *nxt, uint32_t &ovf) {
    using VT = ValTraits<T>;
    if (!app) return 0u;
    T cand = INF;
    if constexpr (VT::U32) {
        if (agg != INF) {
            const uint64_t cc = (uint64_t)agg + (uint64_t)inc;
            if (cc >= 0xffffffffull) {
                ovf = 1;
                return 0u;
            }
            cand = (T)cc;
        }
    } else {
        cand = agg + (T)inc;
    }
    const bool upd = cand < pd;
    const T v = upd ? cand : pd;
    if (complete) nxt[d] = v;
    else if constexpr (VT::U32) atomicMin((unsigned *)&nxt[d], (unsigned)v);
    else atomicMin((long long *)&nxt[d], (long long)v);
    return upd ? 1u << (d & 31) : 0u;
}

template <typename T>
__device__ __forceinline__ void apply_dense(bool app, uint32_t d, T agg, T pd, bool complete, T INF,
                                            int64_t inc, T *nxt, uint32_t *obits, uint32_t &ovf) {
    const uint32_t bit = apply_dense_value<T>(app, d, agg, pd, complete, INF, inc, nxt, ovf);
    if (bit) atomicOr(&obits[d >> 5], bit);
}



// Fold one vector's lanes into a minimum (messages prev[src] (+ weight)).
template <typename T, int W, bool WEIGHT>
__device__ __forceinline__ T fold_lanes(const uint32_t (&src)[W], const uint32_t (&wt)[W],
                                        const T *prev, T INF, uint32_t &ovf) {
    using VT = ValTraits<T>;
    T ps[W];
#pragma unroll
    for (int l = 0; l < W; ++l) ps[l] = src[l] != WG_NO_LANE ? prev[src[l]] : INF;
    T agg = INF;
#pragma unroll
    for (int l = 0; l < W; ++l) {
        if constexpr (VT::U32) {
            if (WEIGHT) {
                if (ps[l] != INF) {
                    uint64_t m = (uint64_t)ps[l] + wt[l];
                    if (m >= 0xffffffffull) ovf = 1;
                    else agg = (T)m < agg ? (T)m : agg;
                }
            } else {
                agg = ps[l] < agg ? ps[l] : agg;  // INF never wins; no overflow without weights
            }
        } else {
            if (src[l] != WG_NO_LANE) {
                T m = ps[l] + (WEIGHT ? (T)wt[l] : (T)0);
                agg = m < agg ? m : agg;
            }
        }
    }
    return agg;
}

// Warp-uniform carry of the open segment across tiles of a warp's range.
template <typename T>
struct Carry {
    uint32_t d = NONE;
    T agg, pd;
    bool act = false, left = true;
};

// Reduce + apply one tile (32 lanes, lane order = item order).  The segment
// min is a shuffle scan limited to each lane's distance from its segment head
// (one SHFL + one predicated min per step, and only as many steps as the
// longest segment in the tile needs).
template <typename T>
__device__ __forceinline__ void finish_tile(uint32_t d, T agg, T pd, bool act, bool first_tile,
                                            bool last_tile, uint32_t dleft, uint32_t dright,
                                            Carry<T> &cy, T INF, int64_t inc, T *nxt,
                                            uint32_t *obits, PullOut &o, const wg_graph &g,
                                            wg_iter_rec *out, uint32_t *overt, uint32_t *opref,
                                            uint32_t *otstart, uint32_t n) {
    const unsigned lane = lane_id();
    const unsigned am = __ballot_sync(FULL, act);
    o.touched += __popc(am);
    const uint32_t d0 = __shfl_sync(FULL, d, 0);
    bool left0;
    if (cy.d == NONE) {
        left0 = first_tile ? (dleft != d0) : true;
    } else if (d0 == cy.d) {
        if (lane == 0 && cy.act) agg = cy.agg < agg ? cy.agg : agg;
        left0 = cy.left;
    } else {
        // the carried segment ended exactly at the previous tile's end
        apply_segments<T>(lane == 0 && cy.act, cy.d, cy.agg, cy.pd, cy.left, INF, inc, nxt, obits, o);
        left0 = true;
    }
    const uint32_t dp = __shfl_up_sync(FULL, d, 1);
    const unsigned heads = __ballot_sync(FULL, lane == 0 || dp != d);
    const unsigned h = 31u - __clz(heads & (0xffffffffu >> (31 - lane)));
    const unsigned dist = lane - h;
    const unsigned maxdist = __reduce_max_sync(FULL, dist);
    for (unsigned off = 1; off <= maxdist; off <<= 1) {
        const T ov = shfl_up_t(agg, (int)off);
        if (off <= dist && ov < agg) agg = ov;
    }
    const bool tail = ((heads >> 1) | 0x80000000u) >> lane & 1u;
    const bool left = h > 0 || left0;
    const uint32_t d31 = __shfl_sync(FULL, d, 31);
    const bool carry = !last_tile && d31 != NONE;
    if (carry) {
        cy.d = d31;
        cy.agg = shfl_t(agg, 31);
        cy.pd = shfl_t(pd, 31);
        cy.act = (am >> 31) & 1u;
        cy.left = (31u - __clz(heads)) > 0 || left0;
    } else {
        cy.d = NONE;
    }
    const bool right = !(lane == 31 && last_tile && dright == d);
    const bool app = tail && act && !(carry && lane == 31);
    apply_segments<T>(app, d, agg, pd, left && right, INF, inc, nxt, obits, o);
    if (o.staged > STAGE - 34) flush_stage(o, g, out, overt, opref, otstart, n);
}

template <typename T>
__device__ __forceinline__ void end_of_pull(PullOut &o, wg_iter_rec *out) {
    const uint64_t es = warp_sum(o.edge_sum);
    const uint32_t ovf = __any_sync(FULL, o.ovf);
    if (lane_id() == 0) {
        if (o.touched) atomicAdd((unsigned long long *)&out->vectors_touched, (unsigned long long)o.touched);
        if (es) atomicAdd((unsigned long long *)&out->out_edge_sum, (unsigned long long)es);
        if (ovf) out->overflow = 1;
    }
}

// ---------------------------------------------------------------------------
// Direct-load pull: wedge mode, filtered (BFS) dense mode, and any width.
template <typename T, int W, bool WEIGHT, bool FILTER, int U>
__global__ void __launch_bounds__(PULL_THREADS) pull_kernel(LoopCtx c, wg_graph g, PullBufs b,
                                                            int shift, int64_t inc, int64_t sentinel,
                                                            int handles) {
    using VT = ValTraits<T>;
    __shared__ uint32_t s_stage[PULL_WARPS][STAGE];
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_PULL_WEDGE);
    const int mode = ctx_mode(c, it);
    if (mode == MODE_NONE || !((handles >> mode) & 1)) return;
    const bool wedge = (mode == MODE_WEDGE);
    wg_iter_rec *out = ctx_out(c, it);
    const T *__restrict__ prev = (const T *)(((it - 1) & 1) ? b.vals[1] : b.vals[0]);
    T *__restrict__ nxt = (T *)((it & 1) ? b.vals[1] : b.vals[0]);
    uint32_t *__restrict__ obits = ((it & 1) ? b.fbits[1] : b.fbits[0]);
    uint32_t *__restrict__ overt = ((it & 1) ? b.fvert[1] : b.fvert[0]);
    uint32_t *__restrict__ opref = ((it & 1) ? b.fpref[1] : b.fpref[0]);
    uint32_t *otstart = ((it & 1) ? b.tstart[1] : b.tstart[0]);
    const uint64_t nitems = wedge ? (out->groups << shift) : g.nvec;
    const T INF = VT::inf(sentinel);
    const unsigned lane = lane_id();
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    PullOut o{s_stage[threadIdx.x >> 5], 0u, 0ull, 0ull, 0u};

    uint64_t t0, t1;
    warp_range((nitems + 31) >> 5, gwarp, nwarps, t0, t1);
    if (t0 < t1) {
        uint32_t dleft = NONE, dright = NONE;
        if (lane == 0 && t0 > 0) {
            uint64_t q = item_pos((t0 << 5) - 1, nitems, wedge, b.glist, shift, g.nvec);
            if (q != ~0ull) dleft = g.vdst[q];
        }
        if (lane == 1) {
            uint64_t q = item_pos(t1 << 5, nitems, wedge, b.glist, shift, g.nvec);
            if (q != ~0ull) dright = g.vdst[q];
        }
        dleft = __shfl_sync(FULL, dleft, 0);
        dright = __shfl_sync(FULL, dright, 1);
        Carry<T> cy;
        for (uint64_t tile = t0; tile < t1; tile += U) {
            uint32_t d[U];
            T pd[U], agg[U];
            bool act[U];
            // first-hit programs: the destination carried into this step
            // already has its (only possible) minimum; skip its gathers
            const uint32_t hit_d = (FILTER && b.first_hit && cy.d != NONE && cy.act && cy.agg != INF) ? cy.d : NONE;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t p = (tile + u < t1)
                                       ? item_pos(((tile + u) << 5) + lane, nitems, wedge, b.glist, shift, g.nvec)
                                       : ~0ull;
                d[u] = p != ~0ull ? g.vdst[p] : NONE;
                pd[u] = INF;
                agg[u] = INF;
                if (FILTER && d[u] != NONE) pd[u] = prev[d[u]];
                act[u] = d[u] != NONE && !(FILTER && pd[u] != INF);
                if (act[u] && d[u] != hit_d) {
                    uint32_t src[W], wt[W];
                    load_lanes<W>(g.vsrc, p, src);
                    if (WEIGHT) load_lanes<W>(g.vw, p, wt);
                    if (!FILTER) pd[u] = prev[d[u]];
                    agg[u] = fold_lanes<T, W, WEIGHT>(src, wt, prev, INF, o.ovf);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (tile + u < t1)
                    finish_tile<T>(d[u], agg[u], pd[u], act[u], tile + u == t0, tile + u == t1 - 1, dleft,
                               dright, cy, INF, inc, nxt, obits, o, g, out, overt, opref, otstart, b.n);
            }
        }
        if (o.staged) flush_stage(o, g, out, overt, opref, otstart, b.n);
    }
    end_of_pull<T>(o, out);
}


// First dense pull of a run whose initial values are the vertex ids
// (WG_RUN_IDENTITY_INIT, CC): every message is its source id and a
// destination's lanes ascend (graph.py:235), so its minimum message is lane 0
// of its first vector -- one load per destination instead of a pass over all
// lanes and gathers.  Full occupancy, K vectors per thread in flight; every
// vector still counts as touched (the reference's full scan).
template <typename T, int W>
__global__ void __launch_bounds__(256) pull_ident_kernel(LoopCtx c, wg_graph g, PullBufs b, int64_t inc,
                                                         int64_t sentinel) {
    using VT = ValTraits<T>;
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_IDENT);
    if (it != 1 || ctx_mode(c, it) != MODE_FULL) return;
    wg_iter_rec *out = ctx_out(c, it);
    const T *__restrict__ prev = (const T *)b.vals[0];
    T *__restrict__ nxt = (T *)b.vals[1];
    uint32_t *__restrict__ obits = b.fbits[1];
    const T INF = VT::inf(sentinel);
    const uint64_t nvec = g.nvec;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    uint32_t ovf = 0;
    constexpr int K = 4;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < nvec; base += K * nth) {
        uint32_t d[K], s0[K];
        bool head[K];
        T pd[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint64_t v = base + k * nth;
            d[k] = v < nvec ? g.vdst[v] : NONE;
            head[k] = v < nvec && (v == 0 || g.vdst[v - 1] != d[k]);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            s0[k] = head[k] ? g.vsrc[(base + k * nth) * W] : 0u;
            pd[k] = head[k] ? prev[d[k]] : INF;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) apply_dense<T>(head[k], d[k], (T)s0[k], pd[k], true, INF, inc, nxt, obits, ovf);
    }
    if (ovf) out->overflow = 1;
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd((unsigned long long *)&out->vectors_touched, (unsigned long long)nvec);
}

// Floor-skipping dense pull (WG_RUN_FLOOR_SKIP, iterations >= 3; CC): the
// same result as pull_dense_tma_kernel without streaming the layout through
// a pipeline -- after two iterations almost every in-edge belongs to a
// destination already at 0.  A thread per vector: the destination's first
// vector lowers nxt[d] to prev[d], a vector whose destination is not at 0
// gathers its lanes and lowers nxt[d] with an atomic min, setting d's
// frontier bit when its candidate beats prev[d].
// Every vector counts as touched (the reference's full scan).  Iteration 2,
// where a third of the in-edges still gather (CC s22), stays on the TMA
// pipeline (0.43 vs 0.52 ms); iteration 3 gathers for 0.2% (0.18 vs 0.38 ms).
constexpr uint64_t FLOOR_KERNELS_FROM = 3;

template <typename T, int W>
__global__ void __launch_bounds__(256) floor_pull_kernel(LoopCtx c, wg_graph g, PullBufs b, int64_t inc,
                                                         int64_t sentinel) {
    using VT = ValTraits<T>;
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_FLOOR);
    if (ctx_mode(c, it) != MODE_FULL || it < b.floor_from) return;
    wg_iter_rec *out = ctx_out(c, it);
    const T *__restrict__ prev = (const T *)(((it - 1) & 1) ? b.vals[1] : b.vals[0]);
    T *__restrict__ nxt = (T *)((it & 1) ? b.vals[1] : b.vals[0]);
    uint32_t *__restrict__ obits = ((it & 1) ? b.fbits[1] : b.fbits[0]);
    const T INF = VT::inf(sentinel);
    uint32_t ovf = 0;
    // K vectors per thread in flight: destinations, then prev[d], then the
    // lanes and gathers of those not at the floor, then the atomics
    constexpr int K = 4;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < g.nvec; base += K * nth) {
        uint32_t d[K];
        T pd[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint64_t v = base + k * nth;
            d[k] = v < g.nvec ? g.vdst[v] : NONE;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) pd[k] = d[k] != NONE ? prev[d[k]] : (T)0;  // 0: nothing to do
        // a destination's first vector lowers nxt[d] to prev[d]: the buffer holds
        // the values of two iterations ago, never below prev (values only
        // decrease), so every destination ends at min(prev[d], its candidates)
        // in any order of the atomics -- no separate init pass
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint64_t v = base + k * nth;
            if (d[k] != NONE && (v == 0 || g.vdst[v - 1] != d[k])) {
                if constexpr (VT::U32) atomicMin((unsigned *)&nxt[d[k]], (unsigned)pd[k]);
                else atomicMin((long long *)&nxt[d[k]], (long long)pd[k]);
            }
        }
        T agg[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            agg[k] = INF;
            if (pd[k] != (T)0) {  // at the floor nothing can lower it
                uint32_t src[W], wt[W];
                load_lanes<W>(g.vsrc, base + k * nth, src);
                agg[k] = fold_lanes<T, W, false>(src, wt, prev, INF, ovf);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (agg[k] == INF) continue;
            T cand;
            if constexpr (VT::U32) {
                const uint64_t cc = (uint64_t)agg[k] + (uint64_t)inc;
                if (cc >= 0xffffffffull) {
                    ovf = 1;
                    continue;
                }
                cand = (T)cc;
            } else {
                cand = agg[k] + (T)inc;
            }
            if (cand < pd[k]) {
                if constexpr (VT::U32) atomicMin((unsigned *)&nxt[d[k]], (unsigned)cand);
                else atomicMin((long long *)&nxt[d[k]], (long long)cand);
                atomicOr(&obits[d[k] >> 5], 1u << (d[k] & 31));
            }
        }
    }
    if (ovf) out->overflow = 1;
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd((unsigned long long *)&out->vectors_touched, (unsigned long long)g.nvec);
}

// Bottom-up BFS dense pull from iteration `floor_from` on (WG_RUN_FIRST_HIT,
// level-synchronous): a thread per vector; a visited destination only lowers
// nxt[d] to prev[d] from its first vector (the buffer holds older, never
// smaller values); a vector of an unvisited destination tests its sources'
// bits in the previous frontier and, on a hit, lowers nxt[d] to the new level.
// Counts the vectors of unvisited destinations as touched (pulls.pyx:77-80).
template <typename T, int W>
__global__ void __launch_bounds__(256) bottom_up_pull_kernel(LoopCtx c, wg_graph g, PullBufs b, int64_t inc,
                                                             int64_t sentinel) {
    using VT = ValTraits<T>;
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_BOTTOM_UP);
    if (ctx_mode(c, it) != MODE_FULL || it < b.floor_from || it < 2) return;
    if (dst_major_active(c, it, b.n, b.dst_major, true)) return;  // dense_dst_kernel's iteration
    wg_iter_rec *out = ctx_out(c, it);
    const T *__restrict__ prev = (const T *)(((it - 1) & 1) ? b.vals[1] : b.vals[0]);
    T *__restrict__ nxt = (T *)((it & 1) ? b.vals[1] : b.vals[0]);
    uint32_t *__restrict__ obits = ((it & 1) ? b.fbits[1] : b.fbits[0]);
    const uint32_t *__restrict__ inbits = (((it - 1) & 1) ? b.fbits[1] : b.fbits[0]);
    const T INF = VT::inf(sentinel);
    const T level = (T)(b.level_base + (int64_t)(it - 1) * inc);
    // a uint32 candidate that does not fit is an overflow only where it
    // would be applied (a hit), like the pipeline and floor kernels
    bool cand_ovf = false;
    uint32_t ovf = 0;
    T cand = INF;
    if constexpr (VT::U32) {
        const uint64_t cc = (uint64_t)level + (uint64_t)inc;
        if (cc >= 0xffffffffull) cand_ovf = true;
        else cand = (T)cc;
    } else {
        cand = level + (T)inc;
    }
    constexpr int K = 4;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    uint64_t touched = 0;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < g.nvec; base += K * nth) {
        uint32_t d[K];
        T pd[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint64_t v = base + k * nth;
            d[k] = v < g.nvec ? g.vdst[v] : NONE;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) pd[k] = d[k] != NONE ? prev[d[k]] : (T)0;
        bool hit[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint64_t v = base + k * nth;
            hit[k] = false;
            if (d[k] == NONE) continue;
            if (pd[k] != INF) {  // visited: only keep prev[d] in this buffer
                if (v == 0 || g.vdst[v - 1] != d[k]) {
                    if constexpr (VT::U32) atomicMin((unsigned *)&nxt[d[k]], (unsigned)pd[k]);
                    else atomicMin((long long *)&nxt[d[k]], (long long)pd[k]);
                }
                continue;
            }
            ++touched;
            uint32_t src[W];
            load_lanes<W>(g.vsrc, v, src);
#pragma unroll
            for (int l = 0; l < W; ++l)
                hit[k] |= src[l] != WG_NO_LANE && ((inbits[src[l] >> 5] >> (src[l] & 31)) & 1u);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (hit[k] && cand_ovf) ovf = 1;
            if (!hit[k] || cand == INF) continue;
            if constexpr (VT::U32) atomicMin((unsigned *)&nxt[d[k]], (unsigned)cand);
            else atomicMin((long long *)&nxt[d[k]], (long long)cand);
            atomicOr(&obits[d[k] >> 5], 1u << (d[k] & 31));
        }
    }
    if (ovf) out->overflow = 1;
    const uint64_t t = warp_sum(touched);
    if (lane_id() == 0 && t) atomicAdd((unsigned long long *)&out->vectors_touched, (unsigned long long)t);
}

// ---------------------------------------------------------------------------
// Destination-major dense pulls (g.voff present, PullBufs::dst_major).
//
// A thread per destination d walks d's own vectors [voff[d], voff[d+1]) --
// no per-vector vdst stream -- and stops as soon as d's result is decided:
//
//  * FLOOR (WG_RUN_FLOOR_SKIP, unweighted, uint32: CC-like min-label runs).
//    0 is the smallest uint32 value, so a destination already at 0 gathers
//    nothing and a destination whose running minimum reaches 0 stops
//    gathering.  The first lane probed is the destination's smallest source
//    (lanes ascend, graph.py:235), the likeliest to carry the smallest label;
//    with identity initial values at iteration 1 it IS the minimum message
//    (no gather at all).  CC s22, iteration 2: 2.23M destinations not at 0,
//    all but 0.34M decided by that probe.
//  * BOTTOM-UP (WG_RUN_FIRST_HIT, filtered, unweighted: level-synchronous
//    BFS).  Visited destinations keep prev[d] and count as untouched
//    (_kernels.pyx:77-80); an unvisited destination tests its sources'
//    membership in the previous frontier -- every finite in-neighbour of it
//    sits there -- and stops at the first hit (cand = level + inc).
//
// Destinations with more than DST_LIGHT vectors that are still undecided are
// finished by their whole warp (lanes strided over the vectors, early exit
// by vote).  Every destination's nxt[d] is written (prev[d] or its
// improvement), so no buffer sync is needed after a dense iteration
// (end_of_iteration); a warp owns 32 consecutive destinations = one
// next-frontier word.  The same pass counts the produced frontier per
// 8192-vertex chunk (members with / without out-edges, their index entries
// and out-degree sum: atomics of one warp each into b.work) and the last
// block turns those into the record and the list pass's prefixes
// (count_epilogue) -- no separate count pass over the bitmap.  Results and
// counters are those of the reference's full scan (every vector touched;
// bottom-up: the vectors of unvisited destinations).
static_assert(PULL_THREADS == FB_WORDS, "the persistent loop runs frontier_list_words with one word per thread");
constexpr uint32_t DST_LIGHT = 512;  // vectors walked by one lane (WG_DST_LIGHT).  8 -> 32: CC s22 it 2 63 -> 58 us,
                                     // BFS s16 it 2 23 -> 13 us; 32 -> 512: BFS s26 it 2 2.83 -> 1.88 ms (with the
                                     // early exit a lane rarely walks far; CC s22 unchanged).  Longer in-lists stay
                                     // with the whole warp: one lane scanning a hub's list would serialise it.
constexpr int DST_K = 4;           // destinations per thread in flight (one warp = DST_K words)
constexpr int DSTK_FLOOR = 0, DSTK_BOTTOM_UP = 1;

// One destination-major dense iteration over warps [warp0, warp0 + nwarps)
// of a grid-stride split; per-chunk frontier totals into b.work (the caller
// then runs count_tail / count_epilogue).
template <typename T, int W, int KIND>
__device__ __forceinline__ void dense_dst_phase(const LoopCtx &c, uint64_t it, const wg_graph &g, const PullBufs &b,
                                                int64_t inc, int64_t sentinel, uint64_t warp0, uint64_t nwarps) {
    using VT = ValTraits<T>;
    wg_iter_rec *out = ctx_out(c, it);
    const T *__restrict__ prev = (const T *)(((it - 1) & 1) ? b.vals[1] : b.vals[0]);
    T *__restrict__ nxt = (T *)((it & 1) ? b.vals[1] : b.vals[0]);
    uint32_t *__restrict__ obits = ((it & 1) ? b.fbits[1] : b.fbits[0]);
    const uint32_t *__restrict__ inbits = (((it - 1) & 1) ? b.fbits[1] : b.fbits[0]);
    const uint32_t *__restrict__ voff = g.voff;
    unsigned long long *totals = (unsigned long long *)b.work;  // 4 counters per 8192-vertex chunk
    const T INF = VT::inf(sentinel);
    const bool lens_deg = (g.flags & WG_GRAPH_LENS_ARE_DEGREES) != 0;
    // iteration 1 reads no bitmap (the initial frontier lives in the caller's
    // words): a level-synchronous run's finite vertices ARE that frontier
    const auto in_prev_frontier = [&](uint32_t v) -> bool {
        return it == 1 ? prev[v] != INF : ((inbits[v >> 5] >> (v & 31)) & 1u) != 0u;
    };
    const bool exact_first = KIND == DSTK_FLOOR && b.ident && it == 1;  // identity values: lane 0 is the min
    uint32_t ovf = 0;
    bool bu_ovf = false;  // flagged only where a hit would apply it
    T bu_cand = INF;  // bottom-up: the level after the previous frontier's
    if constexpr (KIND == DSTK_BOTTOM_UP) {
        const T level = (T)(b.level_base + (int64_t)(it - 1) * inc);
        if constexpr (VT::U32) {
            const uint64_t cc = (uint64_t)level + (uint64_t)inc;
            if (cc >= 0xffffffffull) bu_ovf = true;
            else bu_cand = (T)cc;
        } else {
            bu_cand = level + (T)inc;
        }
    }
    const unsigned lane = lane_id();
    uint64_t touched = 0, lanes_rd = 0, gath = 0;  // algorithmic work (the record's lanes_read / gathers)
    const uint64_t n = g.n;
    const uint64_t span = 32ull * DST_K;  // destinations per warp step, word-aligned
    for (uint64_t wb = warp0 * span; wb < n; wb += nwarps * span) {
        T p[DST_K], agg[DST_K];
        uint32_t v0[DST_K], v1[DST_K], s0[DST_K], deg[DST_K];
        bool need[DST_K];
        // (a) prev[d], d's vector range and (FLOOR) its smallest source, DST_K
        // destinations in flight
#pragma unroll
        for (int k = 0; k < DST_K; ++k) {
            const uint64_t d = wb + 32 * k + lane;
            const bool ok = d < n;
            p[k] = ok ? prev[d] : (T)0;
            v0[k] = ok ? voff[d] : 0u;
            v1[k] = ok ? voff[d + 1] : 0u;
            if constexpr (KIND == DSTK_FLOOR) s0[k] = ok && g.vfirst ? g.vfirst[d] : WG_NO_LANE;
            // out-degree for the frontier counts, in the same round trip (no
            // dependency on the values: 4 bytes per vertex)
            deg[k] = ok ? g.outdeg[d] : 0u;
        }
        // (b) FLOOR: the first lane of every destination not at the floor
#pragma unroll
        for (int k = 0; k < DST_K; ++k) {
            need[k] = v1[k] > v0[k] && (KIND == DSTK_FLOOR ? p[k] != (T)0 : p[k] == INF);
            agg[k] = INF;
        }
        if constexpr (KIND == DSTK_FLOOR) {
            if (!g.vfirst) {
#pragma unroll
                for (int k = 0; k < DST_K; ++k) s0[k] = need[k] ? g.vsrc[(uint64_t)v0[k] * W] : 0u;
            }
#pragma unroll
            for (int k = 0; k < DST_K; ++k)
                if (need[k]) {
                    agg[k] = exact_first ? (T)s0[k] : prev[s0[k]];
                    lanes_rd += 1;
                    gath += exact_first ? 0 : 1;
                }
        } else {
#pragma unroll
            for (int k = 0; k < DST_K; ++k) touched += need[k] ? v1[k] - v0[k] : 0u;
        }
        // (c) undecided destinations: short in-lists by their thread ...
        bool heavy[DST_K], und[DST_K], any_und = false;
#pragma unroll
        for (int k = 0; k < DST_K; ++k) {
            und[k] = need[k] && (KIND == DSTK_FLOOR ? (!exact_first && agg[k] != (T)0) : true);
            heavy[k] = und[k] && v1[k] - v0[k] > b.dst_light;
            any_und |= und[k];
        }
        // (warp-uniform skip: identity first iterations and late iterations
        // decide every destination of most steps from the probe alone)
        if (__any_sync(FULL, any_und)) {
        // The step's light items (destination, k) are spread over the warp's
        // lanes first: a thread that owns several undecided destinations would
        // walk them one after the other (each walk is a chain of dependent
        // round trips) while most lanes idle -- typically ~10 of a step's 128
        // destinations are undecided, so one round of 32 lanes takes them all.
        {
            unsigned lm[DST_K];
            uint32_t cum[DST_K + 1];
            cum[0] = 0;
#pragma unroll
            for (int k = 0; k < DST_K; ++k) {
                lm[k] = __ballot_sync(FULL, und[k] && !heavy[k]);
                cum[k + 1] = cum[k] + __popc(lm[k]);
            }
            const uint32_t nlight = cum[DST_K];
            const unsigned lt = lanemask_lt();
            for (uint32_t r0 = 0; r0 < nlight; r0 += 32) {
                const uint32_t i = r0 + lane;  // this lane's item of the round
                const bool have = i < nlight;
                int mk = -1;
                uint32_t sl = 0;
#pragma unroll
                for (int k = 0; k < DST_K; ++k)
                    if (have && i >= cum[k] && i < cum[k + 1]) {
                        mk = k;
                        sl = __fns(lm[k], 0, (int)(i - cum[k]) + 1);  // its owner lane
                    }
                uint32_t iv0 = 0, iv1 = 0;
                T ia = INF;
#pragma unroll
                for (int k = 0; k < DST_K; ++k) {
                    const uint32_t t0 = __shfl_sync(FULL, v0[k], sl), t1 = __shfl_sync(FULL, v1[k], sl);
                    const T ta = shfl_t(agg[k], (int)sl);
                    if (mk == k) {
                        iv0 = t0;
                        iv1 = t1;
                        ia = ta;
                    }
                }
                // two vectors per round trip (v + 1 < iv1 is checked)
                T res = INF;
                if constexpr (KIND == DSTK_FLOOR) {
                    T a = ia;
                    for (uint32_t v = iv0; v < iv1 && a != (T)0; v += 2) {
                        uint32_t src[W], src2[W], wt[W];
                        load_lanes<W>(g.vsrc, v, src);
                        const bool two = v + 1 < iv1;
                        lanes_rd += two ? 2 * W : W;
                        gath += two ? 2 * W : W;
                        if (two) load_lanes<W>(g.vsrc, v + 1, src2);
                        T m = fold_lanes<T, W, false>(src, wt, prev, INF, ovf);
                        if (two) {
                            const T m2 = fold_lanes<T, W, false>(src2, wt, prev, INF, ovf);
                            m = m2 < m ? m2 : m;
                        }
                        a = m < a ? m : a;
                    }
                    res = a;
                } else {
                    bool hit = false;
                    for (uint32_t v = iv0; v < iv1 && !hit; v += 2) {
                        uint32_t src[W], src2[W];
                        load_lanes<W>(g.vsrc, v, src);
                        const bool two = v + 1 < iv1;
                        lanes_rd += two ? 2 * W : W;
                        gath += two ? 2 * W : W;
                        if (two) load_lanes<W>(g.vsrc, v + 1, src2);
#pragma unroll
                        for (int l = 0; l < W; ++l) hit |= src[l] != WG_NO_LANE && in_prev_frontier(src[l]);
                        if (two) {
#pragma unroll
                            for (int l = 0; l < W; ++l) hit |= src2[l] != WG_NO_LANE && in_prev_frontier(src2[l]);
                        }
                    }
                    res = hit ? (T)0 : INF;  // hit marker
                }
                // results back to the owners: item j of this round sits in lane j - r0
#pragma unroll
                for (int k = 0; k < DST_K; ++k) {
                    const uint32_t j = cum[k] + __popc(lm[k] & lt);
                    const T t = shfl_t(res, (int)((j - r0) & 31u));
                    if (und[k] && !heavy[k] && j >= r0 && j < r0 + 32) agg[k] = t;
                }
            }
        }
        // ... long ones by the whole warp, one at a time (early exit by vote)
#pragma unroll
        for (int k = 0; k < DST_K; ++k) {
            for (unsigned hv = __ballot_sync(FULL, heavy[k]); hv; hv &= hv - 1) {
                const int j = __ffs(hv) - 1;
                const uint32_t h0 = __shfl_sync(FULL, v0[k], j), h1 = __shfl_sync(FULL, v1[k], j);
                T hagg = KIND == DSTK_FLOOR ? shfl_t(agg[k], j) : INF;  // FLOOR: the probe's value
                bool hit = false;
                for (uint32_t v = h0 + lane;; v += 32) {
                    if (v < h1) {
                        uint32_t src[W], wt[W];
                        load_lanes<W>(g.vsrc, v, src);
                        lanes_rd += W;
                        gath += W;
                        if constexpr (KIND == DSTK_FLOOR) {
                            const T m = fold_lanes<T, W, false>(src, wt, prev, INF, ovf);
                            hagg = m < hagg ? m : hagg;
                        } else {
#pragma unroll
                            for (int l = 0; l < W; ++l) hit |= src[l] != WG_NO_LANE && in_prev_frontier(src[l]);
                        }
                    }
                    const bool done = KIND == DSTK_FLOOR ? __any_sync(FULL, hagg == (T)0) : __any_sync(FULL, hit);
                    if (done || v - lane + 32 >= h1) break;
                }
                if constexpr (KIND == DSTK_FLOOR) hagg = warp_min_t(hagg);
                else hagg = __any_sync(FULL, hit) ? (T)0 : INF;
                if (lane == (unsigned)j) agg[k] = hagg;
            }
        }
        }  // any undecided
        // (d) apply: every destination's nxt[d]; bits one word per k; counts
        uint64_t ent = 0, es = 0;
        uint32_t nz = 0, z = 0;
        bool any = false;
#pragma unroll
        for (int k = 0; k < DST_K; ++k) {
            const uint64_t d = wb + 32 * k + lane;
            bool upd = false;
            T res = p[k];
            if (d < n && agg[k] != INF) {
                T cand = INF;
                if constexpr (KIND == DSTK_BOTTOM_UP) {
                    cand = bu_cand;
                    if (bu_ovf) ovf = 1;
                } else if constexpr (VT::U32) {
                    const uint64_t cc = (uint64_t)agg[k] + (uint64_t)inc;
                    if (cc >= 0xffffffffull) ovf = 1;
                    else cand = (T)cc;
                } else {
                    cand = agg[k] + (T)inc;
                }
                if (cand != INF && cand < p[k]) {
                    res = cand;
                    upd = true;
                }
            }
            if (d < n) nxt[d] = res;
            const unsigned word = __ballot_sync(FULL, upd);
            // the warp owns this word: a plain store, zeros included (the
            // bitmap need not be cleared before a destination-major pull)
            if (lane == 0 && d - lane < n) obits[(wb >> 5) + k] = word;
            if (word) {
                any = true;
                if (upd) {
                    const uint64_t len = lens_deg ? deg[k] : g.idx_off[d + 1] - g.idx_off[d];
                    nz += len != 0;
                    ent += len;
                    z += len == 0;
                    es += deg[k];
                }
            }
        }
        if (any) {  // warp-uniform: the produced frontier's counts of this 8192-vertex chunk
            // (REDUX sums; members with / without entries share one: each <= 32 * DST_K)
            const uint32_t nzz = __reduce_add_sync(FULL, nz | (z << 16));
            es = warp_sum_u64_redux(es);
            ent = lens_deg ? es : warp_sum_u64_redux(ent);  // index lengths = out-degrees
            if (lane == 0) {
                unsigned long long *t = totals + 4 * ((wb >> 5) / FB_WORDS);
                if (nzz & 0xffffu) atomicAdd(&t[0], (unsigned long long)(nzz & 0xffffu));
                if (ent) atomicAdd(&t[1], (unsigned long long)ent);
                if (nzz >> 16) atomicAdd(&t[2], (unsigned long long)(nzz >> 16));
                if (es) atomicAdd(&t[3], (unsigned long long)es);
            }
        }
    }
    if (ovf) out->overflow = 1;
    lanes_rd = warp_sum(lanes_rd);
    gath = warp_sum(gath);
    if (lane == 0 && lanes_rd) atomicAdd((unsigned long long *)&out->lanes_read, (unsigned long long)lanes_rd);
    if (lane == 0 && gath) atomicAdd((unsigned long long *)&out->gathers, (unsigned long long)gath);
    if constexpr (KIND == DSTK_FLOOR) {
        if (blockIdx.x == 0 && threadIdx.x == 0)
            atomicAdd((unsigned long long *)&out->vectors_touched, (unsigned long long)g.nvec);
    } else {
        const uint64_t t = warp_sum(touched);
        if (lane == 0 && t) atomicAdd((unsigned long long *)&out->vectors_touched, (unsigned long long)t);
    }
}

template <typename T, int W, int KIND>
__global__ void __launch_bounds__(256) dense_dst_kernel(LoopCtx c, wg_graph g, PullBufs b, int64_t inc,
                                                        int64_t sentinel) {
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_DENSE_DST);
    if (ctx_mode(c, it) != MODE_FULL) return;
    if (!dst_major_active(c, it, b.n, b.dst_major, KIND == DSTK_BOTTOM_UP)) return;
    dense_dst_phase<T, W, KIND>(c, it, g, b, inc, sentinel, ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                                ((uint64_t)gridDim.x * blockDim.x) >> 5);
    count_epilogue(fb_blocks(b.n ? b.n : 1), (uint64_t *)b.work, b.bcount, true, b.ticket, ctx_out(c, it),
                   c.keep_lists, c.edges, c.wedge_limit);
}

// One dense-pull chunk after its gathers were issued: destinations, segment
// heads, the raw gathered messages (INF for padding lanes) and prev[d] of
// segment tails.
template <typename T, int W, bool WEIGHT, int CH>
struct DenseChunk {
    uint32_t d[CH];
    unsigned heads[CH];
    bool valid[CH];
    T ps[CH][W];
    uint32_t src[CH][W];  // filtered pulls: between the prev[d] and the lane gathers
    uint32_t wt[CH][WEIGHT ? W : 1];
    T pd[CH];
};

// fold_lanes over already-gathered messages (a lane whose source value is INF
// never contributes: INF + w >= INF for both encodings)
template <typename T, int W, bool WEIGHT>
__device__ __forceinline__ T fold_gathered(const T (&ps)[W], const uint32_t (&wt)[WEIGHT ? W : 1], T INF,
                                           uint32_t &ovf) {
    using VT = ValTraits<T>;
    T agg = INF;
#pragma unroll
    for (int l = 0; l < W; ++l) {
        if constexpr (!WEIGHT) {
            agg = ps[l] < agg ? ps[l] : agg;
        } else if constexpr (VT::U32) {
            if (ps[l] != INF) {
                const uint64_t m = (uint64_t)ps[l] + wt[l];
                if (m >= 0xffffffffull) ovf = 1;
                else agg = (T)m < agg ? (T)m : agg;
            }
        } else {
            if (ps[l] != INF) {
                const T m = ps[l] + (T)wt[l];
                agg = m < agg ? m : agg;
            }
        }
    }
    return agg;
}

// Dense pull (every min-plus program): the warp streams its tile range with
// TMA and processes CH tiles per stage in four phases so that independent
// work overlaps:
//   1. destinations and lanes from shared memory; segment heads per tile
//      (ballot) -> only segment TAILS gather prev[d];
//   2. all gathers of the CH tiles in flight together; lane folds;
//   3. the CH segmented min-scans, interleaved (none depends on the carry:
//      the carried segment only ever joins a tile's HEAD segment, whose tail
//      lane takes the carried minimum in phase 4);
//   4. a warp-uniform carry chain across the CH tiles, then the applies.
// Chunks are software-pipelined across the warp's range: unfiltered programs
// gather chunk k+1 while chunk k reduces; filtered programs (BFS: only
// destinations with prev[d] == INF pull, pulls.pyx:77-80) read prev[d] of
// chunk k+2, gather chunk k+1 and reduce chunk k, so the dependent
// prev[d] -> prev[src] chain never stalls the warp.  With WG_RUN_FIRST_HIT a
// destination whose carried minimum is already finite gathers nothing more.
template <typename T, int W, bool WEIGHT, bool FILTER, int TMA_CH, int TMA_S, int MINB>
__global__ void __launch_bounds__(PULL_THREADS, MINB) pull_dense_tma_kernel(LoopCtx c, wg_graph g, PullBufs b,
                                                                      int shift, int64_t inc,
                                                                      int64_t sentinel) {
    using VT = ValTraits<T>;
    using SM = TmaSmem<W, WEIGHT, TMA_CH, TMA_S>;
    constexpr int CH = TMA_CH;
    extern __shared__ __align__(128) unsigned char s_raw[];
    const uint64_t it = ctx_iter(c);
    const int mode = ctx_mode(c, it);
    if (mode != MODE_FULL) return;  // wedge iterations use pull_kernel
    if (FILTER && b.dst_major && dst_major_active(c, it, b.n, 1u, !b.floor_skip)) return;  // dense_dst_kernel's
    wg_iter_rec *out = ctx_out(c, it);
    const T *__restrict__ prev = (const T *)(((it - 1) & 1) ? b.vals[1] : b.vals[0]);
    T *__restrict__ nxt = (T *)((it & 1) ? b.vals[1] : b.vals[0]);
    uint32_t *__restrict__ obits = ((it & 1) ? b.fbits[1] : b.fbits[0]);
    const uint32_t nvec = (uint32_t)g.nvec;
    const T INF = VT::inf(sentinel);
    const unsigned lane = lane_id();
    const unsigned wib = threadIdx.x >> 5;
    const bool w8 = WEIGHT && g.vw8 != nullptr;  // byte weights: a quarter of the weight stream
    // bottom-up BFS (level-synchronous runs, WG_RUN_FIRST_HIT): every finite
    // in-neighbour of an unvisited destination is in frontier(it-1) and holds
    // level = base + (it-1)*inc, so its frontier bit replaces the value gather.
    // Frontier 0 lives in the caller's initial words, hence it > 1.
    const bool bottom_up = FILTER && b.first_hit && it > 1;
    // unfiltered program run on the filtered pipeline: prev[d] of every
    // destination is read ahead and one already at 0 (the floor of any
    // min-plus candidate over uint32) gathers nothing -- CC from iteration 2
    // on, where the giant component's label 0 spreads over most vertices
    const bool floor = FILTER && b.floor_skip;
    // identity initial values: iteration 1 belongs to pull_ident_kernel
    const bool ident = (!FILTER || floor) && !WEIGHT && b.ident && it == 1;
    const uint32_t *__restrict__ inbits = (((it - 1) & 1) ? b.fbits[1] : b.fbits[0]);
    const T level = (T)(b.level_base + (int64_t)(it - 1) * inc);
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned le = 0xffffffffu >> (31 - lane);

    unsigned char *wbase = s_raw + (size_t)wib * SM::WARP_BYTES;
    uint32_t *ring = reinterpret_cast<uint32_t *>(wbase);
    uint64_t *bars = reinterpret_cast<uint64_t *>(wbase + (size_t)TMA_S * SM::STAGE_WORDS * 4);
    uint32_t *stage_buf = reinterpret_cast<uint32_t *>(bars + TMA_S);
    PullOut o{stage_buf, 0u, 0ull, 0ull, 0u};

    uint64_t t0w, t1w;
    warp_range(((uint64_t)nvec + 31) >> 5, gwarp, nwarps, t0w, t1w);
    if (ident) return;  // pull_ident_kernel did this iteration
    if (it >= b.pipeline_until) return;  // floor_pull_kernel / bottom_up_pull_kernel did
    if (t0w < t1w) {
        const uint32_t tfirst = (uint32_t)t0w, tend = (uint32_t)t1w;
        const uint32_t vend = (tend << 5) < nvec ? (tend << 5) : nvec;
        if (!FILTER || floor) o.touched = vend - (tfirst << 5);  // every vector of the range is processed
        const uint32_t nchunks = (tend - tfirst + CH - 1) / CH;
        if (lane == 0) {
            for (int s = 0; s < TMA_S; ++s) mbar_init(&bars[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        auto issue = [=](uint32_t ch) {
            const int s = (int)(ch % TMA_S);
            const uint32_t v0 = (tfirst + ch * CH) << 5;
            uint32_t v1 = (tfirst + (ch + 1) * CH) << 5;
            if (v1 > vend) v1 = vend;
            const uint32_t nv = v1 - v0;
            uint32_t *st = ring + (size_t)s * SM::STAGE_WORDS;
            const uint32_t b_src = pad16(nv * W * 4), b_dst = pad16(nv * 4);
            const uint32_t b_w = w8 ? pad16(nv * W) : b_src;
            mbar_expect_tx(&bars[s], b_src + b_dst + (WEIGHT ? b_w : 0));
            const uint64_t pol = l2_evict_first();
            tma_1d_stream(st, g.vsrc + (uint64_t)v0 * W, b_src, &bars[s], pol);
            tma_1d_stream(st + SM::SRC_WORDS, g.vdst + v0, b_dst, &bars[s], pol);
            if (WEIGHT) {
                if (w8) tma_1d_stream(st + SM::SRC_WORDS + SM::VEC, g.vw8 + (uint64_t)v0 * W, b_w, &bars[s], pol);
                else tma_1d_stream(st + SM::SRC_WORDS + SM::VEC, g.vw + (uint64_t)v0 * W, b_w, &bars[s], pol);
            }
        };
        if (lane == 0)
            for (uint32_t ch = 0; ch < nchunks && ch < (uint32_t)TMA_S; ++ch) issue(ch);
        uint32_t dleft = NONE, dright = NONE;
        if (lane == 0 && tfirst > 0) dleft = g.vdst[(tfirst << 5) - 1];
        if (lane == 1 && (tend << 5) < nvec) dright = g.vdst[tend << 5];
        dleft = __shfl_sync(FULL, dleft, 0);
        dright = __shfl_sync(FULL, dright, 1);
        Carry<T> cy;

        // software pipeline: chunk ch+1's gathers are in flight while chunk
        // ch is reduced (two register sets, loop unrolled by two so that no
        // copy touches a register with a load outstanding)
        using Chunk = DenseChunk<T, W, WEIGHT, CH>;
        // lane gathers of a chunk whose prev[d] are known (filtered) or not
        // needed first (unfiltered)
        auto gath = [&](Chunk &k) {
            uint32_t hit_d = NONE;
            if (FILTER && b.first_hit && cy.d != NONE && cy.agg != INF) hit_d = cy.d;
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                bool pull = true;
                if (FILTER && floor) {
                    pull = k.valid[u] && k.pd[u] != (T)0;
                } else if (FILTER) {
                    const bool unv = k.valid[u] && k.pd[u] == INF;  // only unvisited destinations
                    o.touched += __popc(__ballot_sync(FULL, unv));
                    pull = unv && k.d[u] != hit_d;
                }
#pragma unroll
                for (int l = 0; l < W; ++l) {
                    const bool take = pull && k.src[u][l] != WG_NO_LANE;
                    if (FILTER && bottom_up)  // the source's frontier word (8 MB at s26, L2-resident)
                        k.ps[u][l] = take ? (T)inbits[k.src[u][l] >> 5] : (T)0;
                    else
                        k.ps[u][l] = take ? prev[k.src[u][l]] : INF;
                }
            }
        };
        // destinations, lanes and segment heads of a chunk from shared memory;
        // refills the stage; issues prev[d] (all lanes if filtered, else the
        // segment tails) and, unfiltered, the gathers
        auto load = [&](uint32_t ch, Chunk &k) {
            const int s = (int)(ch % TMA_S);
            mbar_wait(&bars[s], (ch / TMA_S) & 1u);
            const uint32_t *st = ring + (size_t)s * SM::STAGE_WORDS;
            const uint32_t tbase = tfirst + ch * CH;
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const uint32_t tile = tbase + u;
                const int j = u * 32 + lane;
                k.valid[u] = tile < tend && (tile << 5) + lane < nvec;
                k.d[u] = k.valid[u] ? st[SM::SRC_WORDS + j] : NONE;
                if constexpr (W == 4) {
                    const uint4 v = *reinterpret_cast<const uint4 *>(st + j * 4);
                    k.src[u][0] = v.x; k.src[u][1] = v.y; k.src[u][2] = v.z; k.src[u][3] = v.w;
                } else {
#pragma unroll
                    for (int l = 0; l < W; ++l) k.src[u][l] = st[j * W + l];
                }
#pragma unroll
                for (int l = 0; l < W; ++l) {
                    if (!k.valid[u]) k.src[u][l] = WG_NO_LANE;
                    if constexpr (WEIGHT)
                        k.wt[u][l] = w8 ? (uint32_t)reinterpret_cast<const uint8_t *>(st + SM::SRC_WORDS + SM::VEC)[j * W + l]
                                        : st[SM::SRC_WORDS + SM::VEC + j * W + l];
                }
            }
            // all lanes' generic-proxy reads of this stage precede the async-proxy
            // (TMA) refill that overwrites it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0 && ch + TMA_S < nchunks) issue(ch + TMA_S);
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const uint32_t dp = __shfl_up_sync(FULL, k.d[u], 1);
                k.heads[u] = __ballot_sync(FULL, lane == 0 || dp != k.d[u]);
            }
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const bool tail = (((k.heads[u] >> 1) | 0x80000000u) >> lane) & 1u;
                k.pd[u] = (k.valid[u] && (FILTER || tail)) ? prev[k.d[u]] : INF;
            }
            if (!FILTER) gath(k);
        };
        auto reduce = [&](uint32_t ch, Chunk &k) {
            const uint32_t tbase = tfirst + ch * CH;
            T agg[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                if (FILTER && bottom_up) {
                    // a source in the previous frontier holds exactly `level`
                    bool any = false;
#pragma unroll
                    for (int l = 0; l < W; ++l)
                        any |= k.src[u][l] != WG_NO_LANE && ((uint32_t)k.ps[u][l] >> (k.src[u][l] & 31)) & 1u;
                    agg[u] = any ? level : INF;
                } else {
                    agg[u] = fold_gathered<T, W, WEIGHT>(k.ps[u], k.wt[u], INF, o.ovf);
                }
            }
            // segmented min-scans, interleaved across tiles (none depends on
            // the carry: the carried segment only ever joins a tile's HEAD
            // segment, whose tail lane takes the carried minimum below)
            unsigned dist[CH], maxd = 0;
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                dist[u] = lane - (31u - __clz(k.heads[u] & le));
                maxd = dist[u] > maxd ? dist[u] : maxd;
            }
            maxd = __reduce_max_sync(FULL, maxd);
            for (unsigned off = 1; off <= maxd; off <<= 1) {
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const T ov = shfl_up_t(agg[u], (int)off);
                    if (off <= dist[u] && ov < agg[u]) agg[u] = ov;
                }
            }
            // warp-uniform carry chain across the CH tiles, then the applies
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const uint32_t tile = tbase + u;
                if (tile >= tend) continue;
                const bool last_tile = tile == tend - 1;
                const uint32_t d0 = __shfl_sync(FULL, k.d[u], 0);
                const uint32_t d31 = __shfl_sync(FULL, k.d[u], 31);
                const T a31 = shfl_t(agg[u], 31);
                const T p31 = shfl_t(k.pd[u], 31);
                const unsigned first_tail = __ffs((k.heads[u] >> 1) | 0x80000000u) - 1;
                bool left0;
                bool merge = false;
                T cin = INF;
                if (cy.d == NONE) {
                    left0 = tile == tfirst ? (dleft != d0) : true;
                } else if (d0 == cy.d) {
                    merge = true;
                    cin = cy.agg;
                    left0 = cy.left;
                } else {
                    apply_dense<T>(lane == 0, cy.d, cy.agg, cy.pd, cy.left, INF, inc, nxt, obits, o.ovf);
                    left0 = true;
                }
                if (merge && lane == first_tail && cin < agg[u]) agg[u] = cin;
                const bool whole = k.heads[u] == 1u;  // one segment spans the tile
                const bool carry = !last_tile && d31 != NONE;
                if (carry) {
                    cy.d = d31;
                    cy.agg = (merge && whole && cin < a31) ? cin : a31;
                    cy.pd = p31;
                    cy.left = (k.heads[u] >> 1) ? true : left0;  // a head after lane 0 precedes lane 31
                } else {
                    cy.d = NONE;
                }
                const bool tail = (((k.heads[u] >> 1) | 0x80000000u) >> lane) & 1u;
                const bool left = (k.heads[u] & le & ~1u) ? true : left0;
                const bool right = !(lane == 31 && last_tile && dright == k.d[u]);
                const bool app = tail && k.valid[u] && !(carry && lane == 31);
                apply_dense<T>(app, k.d[u], agg[u], k.pd[u], left && right, INF, inc, nxt, obits, o.ovf);
            }
        };
        if constexpr (!FILTER) {
            Chunk ka, kb;
            load(0, ka);
            for (uint32_t ch = 0; ch < nchunks; ch += 2) {
                if (ch + 1 < nchunks) load(ch + 1, kb);
                reduce(ch, ka);
                if (ch + 1 >= nchunks) break;
                if (ch + 2 < nchunks) load(ch + 2, ka);
                reduce(ch + 1, kb);
            }
        } else {
            // three register sets: A gathers in flight, B prev[d] in flight
            Chunk ka, kb, kc;
            load(0, ka);
            if (1 < nchunks) load(1, kb);
            gath(ka);
            for (uint32_t ch = 0; ch < nchunks; ch += 3) {
                if (ch + 2 < nchunks) load(ch + 2, kc);
                if (ch + 1 < nchunks) gath(kb);
                reduce(ch, ka);
                if (ch + 1 >= nchunks) break;
                if (ch + 3 < nchunks) load(ch + 3, ka);
                if (ch + 2 < nchunks) gath(kc);
                reduce(ch + 1, kb);
                if (ch + 2 >= nchunks) break;
                if (ch + 4 < nchunks) load(ch + 4, kb);
                if (ch + 3 < nchunks) gath(ka);
                reduce(ch + 2, kc);
            }
        }
    }
    end_of_pull<T>(o, out);
}

// ---------------------------------------------------------------------------
// Sparse Wedge pull: the selected groups come UNSORTED from the transform's
// append list (no bitmap scans).  A warp tile holds 32/vpg groups, one
// vector per lane; segments never cross a group, so a segment is complete
// unless it touches its group's first / last vector AND the neighbouring
// vector outside the group has the same destination (then atomicMin; the
// minimum is order-independent, so the unsorted list gives the reference's
// values, frontier and counters exactly).  Clears the group bits it consumed.
template <typename T, int W, bool WEIGHT, bool FILTER>
__device__ __forceinline__ void sparse_pull_phase(const LoopCtx &c, uint64_t it, const wg_graph &g,
                                                  const PullBufs &b, int shift, int64_t inc,
                                                  int64_t sentinel, uint32_t *gbits, uint64_t ngroups_all,
                                                  uint32_t *stage, uint64_t gwarp, uint64_t nwarps,
                                                  const uint32_t *glist, const FusedT *fx) {
    using VT = ValTraits<T>;
    constexpr int U = SPARSE_U;  // tiles per warp step: independent load chains in flight
    wg_iter_rec *out = ctx_out(c, it);
    // no read-only-cache loads of values here: the persistent loop rewrites them
    const T *prev = (const T *)(((it - 1) & 1) ? b.vals[1] : b.vals[0]);
    T *nxt = (T *)((it & 1) ? b.vals[1] : b.vals[0]);
    uint32_t *obits = ((it & 1) ? b.fbits[1] : b.fbits[0]);
    uint32_t *overt = ((it & 1) ? b.fvert[1] : b.fvert[0]);
    uint32_t *opref = ((it & 1) ? b.fpref[1] : b.fpref[0]);
    uint32_t *otstart = ((it & 1) ? b.tstart[1] : b.tstart[0]);
    const T INF = VT::inf(sentinel);
    const unsigned lane = lane_id();
    const unsigned le = 0xffffffffu >> (31 - lane);
    const uint64_t nsel = *(volatile const uint64_t *)&out->groups;
    const uint32_t vpg = 1u << shift, jmask = vpg - 1, gpt = 32u >> shift;
    const uint32_t j = lane & jmask;
    const uint64_t ntiles = (nsel + gpt - 1) / gpt;
    PullOut o{stage, 0u, 0ull, 0ull, 0u};
    if (gwarp == 0 && lane == 0) {
        uint64_t cov = nsel * vpg;
        if (*(volatile const uint64_t *)&out->reserved[1]) cov -= ngroups_all * vpg - g.nvec;
        out->covered_vectors = cov;
    }
    for (uint64_t t0 = gwarp * U; t0 < ntiles; t0 += nwarps * U) {
        uint64_t grp[U], p[U];
        uint32_t d[U];
        bool gvalid[U], valid[U], act[U];
        T pd[U], agg[U];
        unsigned heads[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t gi = (t0 + u) * gpt + (lane >> shift);
            gvalid[u] = gi < nsel;
            grp[u] = gvalid[u] ? ((volatile const uint32_t *)glist)[gi] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            p[u] = (grp[u] << shift) + j;
            valid[u] = gvalid[u] && p[u] < g.nvec;
            d[u] = valid[u] ? g.vdst[p[u]] : NONE;
            if (gvalid[u] && j == 0) gbits[grp[u] >> 5] = 0;  // all its bits were set this iteration
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pd[u] = INF;
            agg[u] = INF;
            if (FILTER && valid[u]) pd[u] = prev[d[u]];
            act[u] = valid[u] && !(FILTER && pd[u] != INF);
            const uint32_t dp = __shfl_up_sync(FULL, d[u], 1);
            heads[u] = __ballot_sync(FULL, j == 0 || dp != d[u]);
            if (act[u]) {
                uint32_t src[W], wt[W];
                load_lanes<W>(g.vsrc, p[u], src);
                if (WEIGHT) load_lanes<W>(g.vw, p[u], wt);
                agg[u] = fold_lanes<T, W, WEIGHT>(src, wt, prev, INF, o.ovf);
                const bool tail = (((heads[u] >> 1) | 0x80000000u) >> lane) & 1u;
                if (!FILTER && tail) pd[u] = prev[d[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (t0 + u >= ntiles) continue;
            o.touched += __popc(__ballot_sync(FULL, act[u]));
            const unsigned hl = 31u - __clz(heads[u] & le);
            const unsigned dist = lane - hl;
            const unsigned maxd = __reduce_max_sync(FULL, dist);
            for (unsigned off = 1; off <= maxd; off <<= 1) {
                const T ov = shfl_up_t(agg[u], (int)off);
                if (off <= dist && ov < agg[u]) agg[u] = ov;
            }
            const bool tail = (((heads[u] >> 1) | 0x80000000u) >> lane) & 1u;
            const bool app = tail && act[u];
            bool complete = true;
            if (app) {
                const uint64_t g0 = grp[u] << shift;
                // left: the segment starts at the group's first vector -> look before it
                if ((hl & jmask) == 0 && g0 > 0 && g.vdst[g0 - 1] == d[u]) complete = false;
                // right: the segment ends at the group's last vector -> look after it
                if (j == jmask && p[u] + 1 < g.nvec && g.vdst[p[u] + 1] == d[u]) complete = false;
            }
            apply_segments<T>(app, d[u], agg[u], pd[u], complete, INF, inc, nxt, obits, o);
            if (o.staged > STAGE - 34) flush_stage(o, g, out, overt, opref, otstart, b.n, fx);
        }
    }
    if (o.staged) flush_stage(o, g, out, overt, opref, otstart, b.n, fx);
    end_of_pull<T>(o, out);
}

template <typename T, int W, bool WEIGHT, bool FILTER>
__global__ void __launch_bounds__(PULL_THREADS) pull_sparse_kernel(LoopCtx c, wg_graph g, PullBufs b,
                                                                   int shift, int64_t inc, int64_t sentinel,
                                                                   uint32_t *gbits, uint64_t ngroups_all) {
    __shared__ uint32_t s_stage[PULL_WARPS][STAGE];
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_PULL_SPARSE);
    if (ctx_mode(c, it) != MODE_WEDGE) return;
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    sparse_pull_phase<T, W, WEIGHT, FILTER>(c, it, g, b, shift, inc, sentinel, gbits, ngroups_all,
                                            s_stage[threadIdx.x >> 5], gwarp, nwarps, b.glist, nullptr);
}

// ---------------- K7: end of iteration -------------------------------------
// Keeps the strict double buffer coherent in O(|F|) instead of the
// reference's O(V) copy-forward (engine.py:198-202, 264, 300): the two value
// buffers differ exactly at the vertices updated this iteration, so those are
// copied into the buffer the next iteration writes.  Also clears the output
// bitmap of iteration it-1 (reused by it+1), finalises the record and zeroes
// the record the next iteration will fill.
// records_only: the next iteration is a destination-major dense pull, which
// writes every value and every bitmap word it produces -- neither the buffer
// sync nor the bitmap clear is needed, only the record.
template <typename T>
__device__ __forceinline__ void end_of_iteration(const LoopCtx &c, uint64_t it, int mode, const PullBufs &b,
                                                 uint64_t tid, uint64_t nthreads, int zero_ahead,
                                                 bool records_only = false) {
    if (mode != MODE_NONE && !records_only) {
        const wg_iter_rec *out = ctx_out(c, it);
        const wg_iter_rec *in = ctx_in(c, it);
        const T *src = (const T *)((it & 1) ? b.vals[1] : b.vals[0]);
        T *dst = (T *)(((it - 1) & 1) ? b.vals[1] : b.vals[0]);
        const uint32_t *list = ((it & 1) ? b.fvert[1] : b.fvert[0]);
        const uint64_t nz = *(volatile const uint64_t *)&out->nz_packed >> 32;
        const uint64_t z = *(volatile const uint64_t *)&out->z_count;
        if (*(volatile const uint64_t *)&out->reserved[2]) {
            // no member list: the next iteration is a dense pull, which writes
            // every destination (apply_dense), so nothing needs syncing
        } else {
            for (uint64_t i = tid; i < nz + z; i += nthreads) {
                const uint32_t v = i < nz ? list[i] : list[b.n - 1 - (i - nz)];
                dst[v] = *(volatile const T *)&src[v];
            }
        }
        // clear bits of the frontier produced by it-1 (its bitmap is reused by it+1)
        uint32_t *obits = (((it - 1) & 1) ? b.fbits[1] : b.fbits[0]);
        const uint32_t *plist = (((it - 1) & 1) ? b.fvert[1] : b.fvert[0]);
        const uint64_t pnz = *(volatile const uint64_t *)&in->nz_packed >> 32;
        const uint64_t pz = *(volatile const uint64_t *)&in->z_count;
        const uint64_t words = ((uint64_t)b.n + 31) >> 5;
        if (pnz + pz > words || *(volatile const uint64_t *)&in->reserved[2]) {
            for (uint64_t w = tid; w < words; w += nthreads) obits[w] = 0;
        } else {
            for (uint64_t i = tid; i < pnz + pz; i += nthreads) {
                const uint32_t v = i < pnz ? plist[i] : plist[b.n - 1 - (i - pnz)];
                obits[v >> 5] = 0;
            }
        }
    }
    if (tid == 0) {
        wg_iter_rec *out = ctx_out(c, it);
        if (mode != MODE_NONE) {
            out->mode = (uint64_t)mode;
            out->frontier_out = (*(volatile uint64_t *)&out->nz_packed >> 32) + *(volatile uint64_t *)&out->z_count;
            out->active_edges = *(volatile const uint64_t *)&ctx_in(c, it)->out_edge_sum;
            // members of the initial and every produced frontier so far (dst_major_active)
            const wg_iter_rec *pin = ctx_in(c, it);
            out->reserved[4] = (it == 1 ? *(volatile const uint64_t *)&pin->frontier_out
                                        : *(volatile const uint64_t *)&pin->reserved[4]) + out->frontier_out;
        }
        uint64_t *q = (uint64_t *)&c.recs[(it + zero_ahead) % c.ring];
#pragma unroll
        for (int i = 0; i < (int)(sizeof(wg_iter_rec) / 8); ++i) q[i] = 0;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) finalize_kernel(LoopCtx c, PullBufs b) {
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_FINALIZE);
    const int mode = ctx_mode(c, it);
    end_of_iteration<T>(c, it, mode, b, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
                        (uint64_t)gridDim.x * blockDim.x, 1);
}

// ---------------- persistent sparse loop ----------------------------------
// Runs consecutive SPARSE Wedge iterations (transform with group append ->
// unsorted-group pull -> end of iteration) inside one cooperative launch,
// separated by grid-wide barriers, and advances the device iteration counter
// ctrl[0].  It returns as soon as the next iteration is not a sparse Wedge
// iteration (dense, large frontier, converged or past the launch limit
// ctrl[1]); the regular kernels of the loop graph take it from there.  This is
// what keeps high-diameter runs (the 4096^2 grid: ~8.6K thin wavefronts) from
// paying several kernel launches per iteration.
// Optional phase timestamps of the persistent loop (tools/prof_persistent.py):
// 4 x uint64 %globaltimer per iteration.
// The persistent loop takes a Wedge iteration when its transform is small
// in absolute terms (a few index entries per thread of the grid) or sparse
// relative to the group space (decide_kernel's sparse variant); very large
// Wedge frontiers (SSSP s26 iteration 6: 126M entries) run faster through the
// sorted transform + group compaction path of the graph body.
__device__ __forceinline__ bool sparse_wedge(const LoopCtx &c, uint64_t it, uint64_t ngroups) {
    if (ctx_mode(c, it) != MODE_WEDGE) return false;
    const uint64_t entries = *(volatile const uint64_t *)&ctx_in(c, it)->nz_packed & 0xffffffffull;
    return entries < PERSIST_MAX_ENTRIES || entries * SPARSE_ENTRY_RATIO < ngroups;
}

__device__ uint64_t *g_phase_ts = nullptr;
__device__ uint64_t g_phase_cap = 0;

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void phase_stamp(uint64_t it, int k) {
    uint64_t *buf = g_phase_ts;
    if (buf && it < g_phase_cap && blockIdx.x == 0 && threadIdx.x == 0) buf[it * 4 + k] = globaltimer();
}

template <typename T, int W, bool WEIGHT, bool FILTER>
__global__ void __launch_bounds__(PULL_THREADS, SPARSE_MINB) sparse_loop_kernel(LoopCtx c, wg_graph g, PullBufs b,
                                                                   int shift, int64_t inc, int64_t sentinel,
                                                                   uint32_t *gbits, uint64_t ngroups) {
    __shared__ TransformSmem tsm;
    __shared__ uint32_t s_stage[PULL_WARPS][STAGE];
    cg::grid_group grid = cg::this_grid();
    const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    uint64_t *ctrl = const_cast<uint64_t *>(c.ctrl);
    const uint64_t first = *(volatile uint64_t *)&ctrl[0] + 1;
    WG_KTS(first, KTS_PERSIST);
    uint64_t it = first;
    if (g.entries == 0) return;
    const bool fused = b.gbits2 != nullptr && b.glist2 != nullptr;
    // iteration `first`'s record was zeroed by whoever finished first-1; the
    // end-of-iteration work below zeroes records further ahead
    if (tid == 0) {
        for (int a = 1; a <= (fused ? 2 : 1); ++a) {
            uint64_t *q = (uint64_t *)&c.recs[(first + a) % c.ring];
            for (int i = 0; i < (int)(sizeof(wg_iter_rec) / 8); ++i) q[i] = 0;
        }
    }
    grid.sync();
    if (!fused) {
        // destination-major dense iterations run here too (unweighted, dst_major):
        // pull -> barrier -> one block's count scan -> barrier -> the ordered
        // member list when a Wedge iteration follows
        constexpr int KIND = FILTER ? DSTK_BOTTOM_UP : DSTK_FLOOR;
        const uint64_t nchunks = fb_blocks(b.n ? b.n : 1);
        int prev_mode = MODE_NONE;
        while (true) {
            const bool dense = !WEIGHT && b.dst_major && b.loop_dense && ctx_mode(c, it) == MODE_FULL &&
                               dst_major_active(c, it, b.n, 1u, FILTER);
            if (!dense && !sparse_wedge(c, it, ngroups)) break;
            if (dense) {
                phase_stamp(it, 0);
                if (it > first) end_of_iteration<T>(c, it - 1, prev_mode, b, tid, nthreads, 2, true);
                dense_dst_phase<T, W, KIND>(c, it, g, b, inc, sentinel, gwarp, nwarps);
                // the last block to finish scans the per-chunk counts (ticket)
                count_epilogue(nchunks, (uint64_t *)b.work, b.bcount, true, b.ticket, ctx_out(c, it), c.keep_lists,
                               c.edges, c.wedge_limit);
                grid.sync();
                phase_stamp(it, 1);
                phase_stamp(it, 2);
                if (!*(volatile const uint64_t *)&ctx_out(c, it)->reserved[2]) {  // a Wedge iteration follows
                    const int k = (int)(it & 1);
                    const uint64_t *off = (g.flags & WG_GRAPH_LENS_ARE_DEGREES) ? nullptr : g.idx_off;
                    for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
                        frontier_list_words(b.fbits[k], b.n, off, g.outdeg, b.bcount, b.fvert[k], b.fpref[k],
                                            b.tstart[k], ctx_out(c, it), ch);
                        __syncthreads();
                    }
                    grid.sync();
                }
                phase_stamp(it, 3);
                prev_mode = MODE_FULL;
                ++it;
                continue;
            }
            phase_stamp(it, 0);
            if (tid == 0) ctx_out(c, it)->reserved[0] = 3;
            // phase A: transform(it)  ||  end of iteration it-1 (buffer sync, bitmap
            // clear, record) -- independent: it-1's end writes vals[it&1] and
            // fbits[it&1], which only the pull of `it` touches, after the barrier
            transform_phase(c, it, b.fvert[0], b.fvert[1], b.fpref[0], b.fpref[1], b.tstart[0], b.tstart[1],
                            g.idx_off, g.idx_pos, shift, gbits, 1, const_cast<uint32_t *>(b.glist), ngroups,
                            tsm, blockIdx.x, gridDim.x);
            if (it > first) end_of_iteration<T>(c, it - 1, prev_mode, b, tid, nthreads, 2);
            grid.sync();
            phase_stamp(it, 1);
            // phase B: pull(it)
            sparse_pull_phase<T, W, WEIGHT, FILTER>(c, it, g, b, shift, inc, sentinel, gbits, ngroups,
                                                    s_stage[threadIdx.x >> 5], gwarp, nwarps, b.glist, nullptr);
            grid.sync();
            phase_stamp(it, 2);
            phase_stamp(it, 3);
            prev_mode = MODE_WEDGE;
            ++it;
        }
        // the last iteration run here still needs its end-of-iteration work
        if (it > first) {
            end_of_iteration<T>(c, it - 1, prev_mode, b, tid, nthreads, 1);
            if (tid == 0) *(volatile uint64_t *)&ctrl[0] = it - 1;
        }
        return;
    }
    // Fused schedule: ONE phase and one barrier per iteration.  The pull of
    // `it` reads the groups of `it` (slot it) and appends the groups of it+1
    // into the other slot; the end of iteration it-1 runs in the same phase:
    // its value sync into vals[it&1] uses atomicMin (a concurrent update by
    // pull(it) is smaller: values never increase), and it clears the bitmap
    // of frontier(it-1), which pull(it+1) reuses.  Slot of iteration k:
    // (k - first) & 1, slot 0 = the run's regular buffers.
    auto slot_bits = [&](uint64_t k) { return ((k - first) & 1) ? b.gbits2 : gbits; };
    auto slot_list = [&](uint64_t k) { return ((k - first) & 1) ? b.glist2 : const_cast<uint32_t *>(b.glist); };
    if (sparse_wedge(c, it, ngroups)) {
        transform_phase(c, it, b.fvert[0], b.fvert[1], b.fpref[0], b.fpref[1], b.tstart[0], b.tstart[1],
                        g.idx_off, g.idx_pos, shift, gbits, 1, const_cast<uint32_t *>(b.glist), ngroups, tsm,
                        blockIdx.x, gridDim.x);
        grid.sync();
    }
    while (sparse_wedge(c, it, ngroups)) {
        phase_stamp(it, 0);
        if (tid == 0) {
            ctx_out(c, it)->reserved[0] = 3;
            if (it > first)  // the fused transform's entry count (frontier.py:205)
                ctx_out(c, it)->transform_entries =
                    *(volatile const uint64_t *)&ctx_in(c, it)->nz_packed & 0xffffffffull;
        }
        // end of iteration it-1
        {
            const uint64_t ip = it - 1;
            const wg_iter_rec *pr = ctx_out(c, ip);
            const uint32_t *list = (ip & 1) ? b.fvert[1] : b.fvert[0];
            const uint64_t nz = *(volatile const uint64_t *)&pr->nz_packed >> 32;
            const uint64_t z = *(volatile const uint64_t *)&pr->z_count;
            const bool nolist = *(volatile const uint64_t *)&pr->reserved[2] != 0;
            if (it > first && !nolist) {
                const T *src = (const T *)((ip & 1) ? b.vals[1] : b.vals[0]);
                T *dst = (T *)((it & 1) ? b.vals[1] : b.vals[0]);
                for (uint64_t i = tid; i < nz + z; i += nthreads) {
                    const uint32_t v = i < nz ? list[i] : list[b.n - 1 - (i - nz)];
                    const T x = *(volatile const T *)&src[v];
                    if constexpr (ValTraits<T>::U32) atomicMin((unsigned *)&dst[v], (unsigned)x);
                    else atomicMin((long long *)&dst[v], (long long)x);
                }
            }
            uint32_t *pbits = (ip & 1) ? b.fbits[1] : b.fbits[0];
            const uint64_t words = ((uint64_t)b.n + 31) >> 5;
            if (nz + z > words || nolist) {
                for (uint64_t w = tid; w < words; w += nthreads) pbits[w] = 0;
            } else {
                for (uint64_t i = tid; i < nz + z; i += nthreads) {
                    const uint32_t v = i < nz ? list[i] : list[b.n - 1 - (i - nz)];
                    pbits[v >> 5] = 0;
                }
            }
            if (tid == 0) {
                if (it > first) {
                    wg_iter_rec *po = ctx_out(c, ip);
                    po->mode = MODE_WEDGE;
                    po->frontier_out = nz + z;
                    po->active_edges = *(volatile const uint64_t *)&ctx_in(c, ip)->out_edge_sum;
                }
                uint64_t *q = (uint64_t *)&c.recs[(it + 2) % c.ring];
                for (int i = 0; i < (int)(sizeof(wg_iter_rec) / 8); ++i) q[i] = 0;
            }
        }
        // a vertex with a long index list joined frontier(it-1): the groups of
        // `it` still need the regular (load-balanced) transform
        if (it > first && *(volatile const uint64_t *)&ctx_out(c, it)->reserved[3]) {
            transform_phase(c, it, b.fvert[0], b.fvert[1], b.fpref[0], b.fpref[1], b.tstart[0], b.tstart[1],
                            g.idx_off, g.idx_pos, shift, slot_bits(it), 1, slot_list(it), ngroups, tsm,
                            blockIdx.x, gridDim.x);
            grid.sync();
        }
        phase_stamp(it, 1);
        FusedT fx{slot_bits(it + 1), slot_list(it + 1), ctx_out(c, it + 1), g.idx_pos, shift, ngroups};
        sparse_pull_phase<T, W, WEIGHT, FILTER>(c, it, g, b, shift, inc, sentinel, slot_bits(it), ngroups,
                                                s_stage[threadIdx.x >> 5], gwarp, nwarps, slot_list(it), &fx);
        grid.sync();
        phase_stamp(it, 2);
        phase_stamp(it, 3);
        ++it;
    }
    // `it` did not run: drop the groups appended for it, then the end of the
    // last iteration that ran
    const uint64_t napp = *(volatile const uint64_t *)&ctx_out(c, it)->groups;
    grid.sync();
    if (it > first) {
        uint32_t *lb = slot_bits(it);
        const uint32_t *ll = slot_list(it);
        for (uint64_t i = tid; i < napp; i += nthreads) lb[ll[i] >> 5] = 0;
        end_of_iteration<T>(c, it - 1, MODE_WEDGE, b, tid, nthreads, 1);
        if (tid == 0) *(volatile uint64_t *)&ctrl[0] = it - 1;
    }
}

__global__ void bump_counter_kernel(uint64_t *ctrl, uint64_t by) { ctrl[0] += by; }

}  // namespace wg
