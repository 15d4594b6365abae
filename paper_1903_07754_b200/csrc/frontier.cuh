// frontier.cuh — frontier compaction (K2), Wedge transform (K3) and group
// compaction (K4).
//
// Reference: VertexFrontier / WedgeFrontier / transform_frontier
// (frontier.py:65-209) and the native transform loop (_kernels.pyx:35-52).
//
// Bitmaps are uint32 little-endian words: the same memory image as the
// reference's uint64 words (bitmask.py:15-32), so a reference Bitmask buffer
// is consumed and produced without conversion.
#pragma once
#include "loop.cuh"

namespace wg {

// Ordered bitmap compaction: one block owns CB_WORDS consecutive words; the
// first pass writes per-block totals, the second pass sums the totals of the
// preceding blocks (no separate scan launch) and writes ids in ascending order.
constexpr int CB_THREADS = 256;
constexpr int CB_WPT = 4;                       // words per thread
constexpr int CB_WORDS = CB_THREADS * CB_WPT;   // words per block

constexpr int TR_THREADS = 256;
constexpr int TR_EPT = 8;
constexpr int TR_TILE = TR_THREADS * TR_EPT;
static_assert(TR_TILE == WG_TRANSFORM_TILE, "transform tile");

// A list member covering entries [pref, pref+len) at list position pos owns
// the tile starts of every transform tile whose first entry it covers.
__device__ __forceinline__ void mark_tile_starts(uint32_t *tstart, uint64_t pref, uint64_t len,
                                                 uint32_t pos) {
    const uint64_t k0 = (pref + TR_TILE - 1) / TR_TILE, k1 = (pref + len - 1) / TR_TILE;
    for (uint64_t k = k0; k <= k1; ++k) tstart[k] = pos;
}

__host__ __device__ inline uint64_t cb_blocks(uint64_t nbits) {
    uint64_t words = (nbits + 31) >> 5;
    return (words + CB_WORDS - 1) / CB_WORDS;
}

__device__ __forceinline__ uint32_t masked_word(const uint32_t *words, uint64_t w, uint64_t nbits) {
    uint64_t nwords = (nbits + 31) >> 5;
    if (w >= nwords) return 0;
    uint32_t x = words[w];
    uint64_t hi = (w + 1) << 5;
    if (hi > nbits) x &= (1u << (nbits & 31)) - 1u;
    return x;
}

// Sum of `stride`-strided per-block totals of blocks [0, upto) (block-wide).
__device__ __forceinline__ uint64_t prior_blocks_sum(const uint64_t *bcount, uint64_t upto,
                                                     int stride, int field, uint64_t *smem) {
    uint64_t s = 0;
    for (uint64_t b = threadIdx.x; b < upto; b += blockDim.x) s += bcount[b * stride + field];
    return block_sum(s, smem);
}

// ---------------- K4: group bitmap -> ascending group list ----------------
__global__ void __launch_bounds__(CB_THREADS) group_count_kernel(LoopCtx c, const uint32_t *words,
                                                                 uint64_t nbits, uint64_t *bcount) {
    if (ctx_mode(c, ctx_iter(c)) != MODE_WEDGE) return;
    __shared__ uint64_t sm[33];
    uint64_t w0 = (uint64_t)blockIdx.x * CB_WORDS + threadIdx.x * CB_WPT;
    uint64_t cnt = 0;
#pragma unroll
    for (int i = 0; i < CB_WPT; ++i) cnt += __popc(masked_word(words, w0 + i, nbits));
    uint64_t tot = block_sum(cnt, sm);
    if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

// Writes glist, the record's `groups` and `covered_vectors`
// (frontier.py:143-150), and optionally clears the words for reuse.
__global__ void __launch_bounds__(CB_THREADS) group_list_kernel(LoopCtx c, uint32_t *words,
                                                                uint64_t nbits,
                                                                const uint64_t *bcount,
                                                                uint32_t *glist, int clear,
                                                                int shift, uint64_t nvec) {
    uint64_t it = ctx_iter(c);
    if (ctx_mode(c, it) != MODE_WEDGE) return;
    __shared__ uint64_t sm[33];
    uint64_t base = prior_blocks_sum(bcount, blockIdx.x, 1, 0, sm);
    uint64_t w0 = (uint64_t)blockIdx.x * CB_WORDS + threadIdx.x * CB_WPT;
    uint32_t x[CB_WPT];
    uint64_t cnt = 0;
#pragma unroll
    for (int i = 0; i < CB_WPT; ++i) {
        x[i] = masked_word(words, w0 + i, nbits);
        cnt += __popc(x[i]);
    }
    uint64_t tot;
    uint64_t pos = base + block_exclusive_sum(cnt, sm, &tot);
    __shared__ int s_last;
    if (threadIdx.x == 0) s_last = 0;
    __syncthreads();
    const uint64_t last_word = (nbits - 1) >> 5;
#pragma unroll
    for (int i = 0; i < CB_WPT; ++i) {
        uint32_t v = x[i];
        if (w0 + i == last_word && ((v >> ((nbits - 1) & 31)) & 1u)) s_last = 1;
        if (v && clear) words[w0 + i] = 0;
        while (v) {
            int b = __ffs(v) - 1;
            v &= v - 1;
            glist[pos++] = (uint32_t)(((w0 + i) << 5) + b);
        }
    }
    __syncthreads();
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        uint64_t groups = base + tot;
        wg_iter_rec *r = ctx_out(c, it);
        r->groups = groups;
        // covered vectors: set bits * vpg minus the overhang of a clipped last group
        uint64_t vpg = 1ull << shift;
        uint64_t cov = groups * vpg;
        if (s_last) cov -= nbits * vpg - nvec;
        r->covered_vectors = cov;
    }
}

// ---------------- K2: frontier bitmap -> member list ----------------------
// Members with out-edges go to the front of the list in ascending order,
// each with the exclusive prefix of their edge-index lengths (the Wedge
// transform's load-balancing key); members without out-edges go to the back.
// bcount holds 4 counters per block: nz members, their entries, zero-degree
// members, out-degree sum.
__device__ __forceinline__ void frontier_count_body(const uint32_t *words, uint64_t nbits,
                                                    const uint64_t *idx_off, const uint32_t *outdeg,
                                                    uint64_t *bcount) {
    __shared__ uint64_t sm[33];
    uint64_t w0 = (uint64_t)blockIdx.x * CB_WORDS + threadIdx.x * CB_WPT;
    uint64_t nz = 0, ent = 0, z = 0, es = 0;
#pragma unroll
    for (int i = 0; i < CB_WPT; ++i) {
        uint32_t v = masked_word(words, w0 + i, nbits);
        while (v) {
            int b = __ffs(v) - 1;
            v &= v - 1;
            uint64_t u = ((w0 + i) << 5) + b;
            uint64_t len = idx_off[u + 1] - idx_off[u];
            if (len) { ++nz; ent += len; } else { ++z; }
            es += outdeg[u];
        }
    }
    nz = block_sum(nz, sm);
    ent = block_sum(ent, sm);
    z = block_sum(z, sm);
    es = block_sum(es, sm);
    if (threadIdx.x == 0) {
        uint64_t *o = bcount + 4ull * blockIdx.x;
        o[0] = nz; o[1] = ent; o[2] = z; o[3] = es;
    }
}

__device__ __forceinline__ void frontier_list_body(const uint32_t *words, uint64_t nbits,
                                                   const uint64_t *idx_off, const uint64_t *bcount,
                                                   uint32_t *fvert, uint32_t *fpref, uint32_t *tstart,
                                                   wg_iter_rec *rec) {
    __shared__ uint64_t sm[33];
    uint64_t nz_base = prior_blocks_sum(bcount, blockIdx.x, 4, 0, sm);
    uint64_t ent_base = prior_blocks_sum(bcount, blockIdx.x, 4, 1, sm);
    uint64_t z_base = prior_blocks_sum(bcount, blockIdx.x, 4, 2, sm);
    uint64_t w0 = (uint64_t)blockIdx.x * CB_WORDS + threadIdx.x * CB_WPT;
    uint32_t x[CB_WPT];
    uint64_t nz = 0, ent = 0, z = 0;
#pragma unroll
    for (int i = 0; i < CB_WPT; ++i) {
        x[i] = masked_word(words, w0 + i, nbits);
        uint32_t v = x[i];
        while (v) {
            int b = __ffs(v) - 1;
            v &= v - 1;
            uint64_t u = ((w0 + i) << 5) + b;
            uint64_t len = idx_off[u + 1] - idx_off[u];
            if (len) { ++nz; ent += len; } else { ++z; }
        }
    }
    uint64_t nz_tot, ent_tot, z_tot;
    uint64_t nzp = nz_base + block_exclusive_sum(nz, sm, &nz_tot);
    uint64_t entp = ent_base + block_exclusive_sum(ent, sm, &ent_tot);
    uint64_t zp = z_base + block_exclusive_sum(z, sm, &z_tot);
#pragma unroll
    for (int i = 0; i < CB_WPT; ++i) {
        uint32_t v = x[i];
        while (v) {
            int b = __ffs(v) - 1;
            v &= v - 1;
            uint64_t u = ((w0 + i) << 5) + b;
            uint64_t len = idx_off[u + 1] - idx_off[u];
            if (len) {
                fvert[nzp] = (uint32_t)u;
                fpref[nzp] = (uint32_t)entp;
                if (tstart) mark_tile_starts(tstart, entp, len, (uint32_t)nzp);
                ++nzp;
                entp += len;
            } else {
                fvert[nbits - 1 - zp] = (uint32_t)u;
                ++zp;
            }
        }
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        uint64_t nz_all = nz_base + nz_tot, ent_all = ent_base + ent_tot, z_all = z_base + z_tot;
        uint64_t es = 0;
        for (uint64_t b = 0; b < gridDim.x; ++b) es += bcount[4 * b + 3];
        rec->nz_packed = (nz_all << 32) | ent_all;
        rec->z_count = z_all;
        rec->frontier_out = nz_all + z_all;
        rec->out_edge_sum = es;
    }
}

__global__ void __launch_bounds__(CB_THREADS) frontier_count_kernel(const uint32_t *words, uint64_t nbits,
                                                                    const uint64_t *idx_off,
                                                                    const uint32_t *outdeg, uint64_t *bcount) {
    frontier_count_body(words, nbits, idx_off, outdeg, bcount);
}

__global__ void __launch_bounds__(CB_THREADS) frontier_list_kernel(const uint32_t *words, uint64_t nbits,
                                                                   const uint64_t *idx_off, const uint64_t *bcount,
                                                                   uint32_t *fvert, uint32_t *fpref,
                                                                   uint32_t *tstart, wg_iter_rec *rec) {
    frontier_list_body(words, nbits, idx_off, bcount, fvert, fpref, tstart, rec);
}

// The same two passes inside the device loop after a dense pull, which only
// sets next-frontier bits: build iteration it's member list, tile starts,
// counts and out-degree sum from its bitmap (gated on the device mode).
struct FrontierBufs {
    uint32_t *fbits[2], *fvert[2], *fpref[2], *tstart[2];
};

__global__ void __launch_bounds__(CB_THREADS) loop_frontier_count_kernel(LoopCtx c, FrontierBufs f, uint64_t n,
                                                                         const uint64_t *idx_off,
                                                                         const uint32_t *outdeg,
                                                                         uint64_t *bcount) {
    const uint64_t it = ctx_iter(c);
    if (ctx_mode(c, it) != MODE_FULL) return;
    frontier_count_body((it & 1) ? f.fbits[1] : f.fbits[0], n, idx_off, outdeg, bcount);
}

__global__ void __launch_bounds__(CB_THREADS) loop_frontier_list_kernel(LoopCtx c, FrontierBufs f, uint64_t n,
                                                                        const uint64_t *idx_off,
                                                                        const uint64_t *bcount) {
    const uint64_t it = ctx_iter(c);
    if (ctx_mode(c, it) != MODE_FULL) return;
    const int k = (int)(it & 1);
    frontier_list_body(k ? f.fbits[1] : f.fbits[0], n, idx_off, bcount, k ? f.fvert[1] : f.fvert[0],
                       k ? f.fpref[1] : f.fpref[0], k ? f.tstart[1] : f.tstart[0], ctx_out(c, it));
}

// ---------------- K3: Wedge transform --------------------------------------
// Load-balanced over index ENTRIES (not vertices), so hub sources with huge
// out-lists do not serialise a thread (the CPU transform lost up to 89% of its
// time to imbalance).  A block takes tiles of TR_TILE entries;
// the list items overlapping the tile are staged in shared memory; each thread
// then walks TR_EPT consecutive entries, OR-ing group bits pos >> shift and
// skipping repeats (a source's positions ascend, so equal groups are adjacent).


// Last index i in [lo, hi) with pref[i] <= e (block-cooperative k-ary search;
// pref ascending, pref[lo] <= e).  All threads return the same value.
__device__ __forceinline__ uint64_t block_search(const uint32_t *pref, uint64_t lo, uint64_t hi,
                                                 uint64_t e, uint64_t *sh) {
    while (hi - lo > 1) {
        uint64_t span = hi - lo;
        uint64_t step = (span + blockDim.x - 1) / blockDim.x;
        uint64_t probe = lo + threadIdx.x * step;
        bool ok = probe < hi && pref[probe] <= e;
        // the largest ok probe
        unsigned b = __ballot_sync(FULL, ok);
        if (threadIdx.x == 0) sh[0] = 0;
        __syncthreads();
        if ((threadIdx.x & 31) == 0 && b) atomicMax((unsigned long long *)&sh[0],
                                                    (unsigned long long)(threadIdx.x + 31 - __clz(b)));
        __syncthreads();
        uint64_t best = sh[0];
        __syncthreads();
        uint64_t nlo = lo + best * step;
        uint64_t nhi = nlo + step < hi ? nlo + step : hi;
        lo = nlo;
        hi = nhi;
        if (step == 1) break;
    }
    return lo;
}

struct TransformSmem {
    uint32_t pref[TR_TILE + 1];
    uint64_t base[TR_TILE + 1];
    uint64_t tmp[2];
    uint32_t app[TR_TILE];  // groups newly selected by this block in this tile (append mode)
    uint32_t napp;
};

// Append mode (unsorted Wedge path): newly selected groups are staged in
// shared memory and appended to the group list with one global atomic per
// block tile.
__device__ __forceinline__ void flush_appended(TransformSmem &sm, uint32_t *glist, wg_iter_rec *out,
                                               uint64_t ngroups) {
    __syncthreads();
    const uint32_t k = sm.napp;
    if (k) {
        if (threadIdx.x == 0)
            sm.tmp[1] = atomicAdd((unsigned long long *)&out->groups, (unsigned long long)k);
        __syncthreads();
        const uint64_t base = sm.tmp[1];
        for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
            const uint32_t gid = sm.app[i];
            glist[base + i] = gid;
            if (gid == ngroups - 1) out->reserved[1] = 1;  // the clipped last group is selected
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) sm.napp = 0;
    __syncthreads();
}

// Transform of iteration `it` by `nblocks` cooperating blocks (block index
// `block`).  Also used inside the persistent sparse-loop kernel, hence no
// read-only-cache loads of the (rewritten) frontier lists.
__device__ __forceinline__ void transform_phase(const LoopCtx &c, uint64_t it, const uint32_t *fvert0,
                                                const uint32_t *fvert1, const uint32_t *fpref0,
                                                const uint32_t *fpref1, const uint32_t *tstart0,
                                                const uint32_t *tstart1, const uint64_t *idx_off,
                                                const uint32_t *idx_pos, int shift, uint32_t *gbits,
                                                int append, uint32_t *glist, uint64_t ngroups,
                                                TransformSmem &sm, uint64_t block, uint64_t nblocks) {
    const wg_iter_rec *in = ctx_in(c, it);
    const uint64_t packed = *(volatile const uint64_t *)&in->nz_packed;
    const uint64_t count = packed >> 32, total = packed & 0xffffffffull;
    if (block == 0 && threadIdx.x == 0) ctx_out(c, it)->transform_entries = total;
    if (total == 0) return;
    const uint32_t *fvert = ((it - 1) & 1) ? fvert1 : fvert0;
    const uint32_t *fpref = ((it - 1) & 1) ? fpref1 : fpref0;
    const uint32_t *tstart = ((it - 1) & 1) ? tstart1 : tstart0;
    const uint64_t ntiles = (total + TR_TILE - 1) / TR_TILE;
    if (threadIdx.x == 0) sm.napp = 0;
    __syncthreads();
    for (uint64_t tile = block; tile < ntiles; tile += nblocks) {
        const uint64_t e0 = tile * TR_TILE;
        const uint64_t e1 = e0 + TR_TILE < total ? e0 + TR_TILE : total;
        // members covering this tile: from the one holding entry e0 to the one
        // holding the next tile's first entry (recorded by the list producer)
        const uint64_t i0 = tstart[tile];
        const uint64_t ilast = tile + 1 < ntiles ? tstart[tile + 1] : count - 1;
        const uint64_t nitems = ilast - i0 + 1;
        for (uint64_t k = threadIdx.x; k < nitems; k += blockDim.x) {
            const uint32_t v = fvert[i0 + k];
            const uint32_t p = fpref[i0 + k];
            sm.pref[k] = p;
            sm.base[k] = idx_off[v] - p;
        }
        __syncthreads();
        uint64_t e = e0 + (uint64_t)threadIdx.x * TR_EPT;
        if (e < e1) {
            uint32_t lo = 0, hi = (uint32_t)nitems;  // last k with pref[k] <= e
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (sm.pref[mid] <= e) lo = mid; else hi = mid;
            }
            uint32_t k = lo;
            uint64_t next = (k + 1 < nitems) ? sm.pref[k + 1] : ~0ull;
            // all loads of this thread's entries first, then all atomics, so
            // neither the index reads nor the bit sets wait on one another
            uint32_t gid[TR_EPT];
#pragma unroll
            for (int i = 0; i < TR_EPT; ++i) {
                const uint64_t ee = e + i;
                gid[i] = 0xffffffffu;
                if (ee < e1) {
                    while (ee >= next) {
                        ++k;
                        next = (k + 1 < nitems) ? sm.pref[k + 1] : ~0ull;
                    }
                    gid[i] = idx_pos[sm.base[k] + ee] >> shift;
                }
            }
            uint32_t old[TR_EPT];
#pragma unroll
            for (int i = 0; i < TR_EPT; ++i) {
                old[i] = 0xffffffffu;
                // a source's positions ascend: equal groups are adjacent
                const bool fresh_gid = gid[i] != 0xffffffffu && (i == 0 || gid[i] != gid[i - 1]);
                if (fresh_gid) {
                    const uint32_t bit = 1u << (gid[i] & 31);
                    if (append) old[i] = atomicOr(&gbits[gid[i] >> 5], bit);
                    else atomicOr(&gbits[gid[i] >> 5], bit);
                }
            }
            if (append) {
#pragma unroll
                for (int i = 0; i < TR_EPT; ++i) {
                    if (old[i] != 0xffffffffu && !((old[i] >> (gid[i] & 31)) & 1u))
                        sm.app[atomicAdd(&sm.napp, 1u)] = gid[i];
                }
            }
        }
        if (append) flush_appended(sm, glist, ctx_out(c, it), ngroups);
        else __syncthreads();
    }
}

__global__ void __launch_bounds__(TR_THREADS) transform_kernel(
    LoopCtx c, const uint32_t *fvert0, const uint32_t *fvert1, const uint32_t *fpref0,
    const uint32_t *fpref1, const uint32_t *tstart0, const uint32_t *tstart1, const uint64_t *idx_off,
    const uint32_t *idx_pos, int shift, uint32_t *gbits, int append, uint32_t *glist, uint64_t ngroups) {
    const uint64_t it = ctx_iter(c);
    if (ctx_mode(c, it) != MODE_WEDGE) return;
    __shared__ TransformSmem sm;
    transform_phase(c, it, fvert0, fvert1, fpref0, fpref1, tstart0, tstart1, idx_off, idx_pos, shift, gbits,
                    append, glist, ngroups, sm, blockIdx.x, gridDim.x);
}

}  // namespace wg
