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
    WG_KTS(ctx_iter(c), KTS_GROUP_COUNT);
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
    WG_KTS(it, KTS_GROUP_LIST);
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
// Lane-per-vertex traversal: each warp owns one 32-word chunk (1024
// vertices) and for each word the 32 lanes look at its 32 vertices, so the
// index offsets / out-degrees of set bits are read with coalesced loads
// whatever the frontier density; empty chunks cost one ballot.  Pass 1
// writes per-block totals; the LAST block to finish (atomic ticket) turns
// them into exclusive prefixes, writes the record's counts and decides
// whether the ordered list is needed at all: after a dense pull whose output
// frontier gates the next iteration to FullScan again, nothing consumes the
// list (the next pull is dense, end-of-iteration syncs all values, the
// bitmap is cleared whole), so pass 2 is skipped (record reserved[2] = 1).
constexpr int FB_WORDS = CB_THREADS;  // words per block (one chunk per warp)

__host__ __device__ inline uint64_t fb_blocks(uint64_t nbits) {
    uint64_t words = (nbits + 31) >> 5;
    return (words + FB_WORDS - 1) / FB_WORDS;
}

struct VertexInfo {
    bool set;
    uint32_t len;    // edge-index entries (0: member without out-edges)
    uint32_t deg;    // out-degree
};

// idx_off == nullptr: the layout has one index entry per edge (entries ==
// edges, a de-duplicated graph), so a vertex's index length is its
// out-degree and only the 4-byte degrees are read.
__device__ __forceinline__ VertexInfo vertex_info(uint32_t x, uint64_t wi, unsigned lane,
                                                  const uint64_t *idx_off, const uint32_t *outdeg) {
    VertexInfo r{((x >> lane) & 1u) != 0, 0u, 0u};
    if (r.set) {
        const uint64_t u = (wi << 5) + lane;
        r.deg = outdeg[u];
        r.len = idx_off ? (uint32_t)(idx_off[u + 1] - idx_off[u]) : r.deg;
    }
    return r;
}

// Warp totals of the warp's 32-word chunk starting at word wbase.
__device__ __forceinline__ void chunk_counts(const uint32_t *words, uint64_t nbits, uint64_t wbase,
                                            const uint64_t *idx_off, const uint32_t *outdeg, uint64_t &nz,
                                            uint64_t &ent, uint64_t &z, uint64_t &es) {
    const unsigned lane = lane_id();
    nz = ent = z = es = 0;
    const uint32_t myw = masked_word(words, wbase + lane, nbits);
    if (__ballot_sync(FULL, myw != 0) == 0) return;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
        const uint32_t x = __shfl_sync(FULL, myw, j);
        const VertexInfo vi = vertex_info(x, wbase + j, lane, idx_off, outdeg);
        if (vi.set) {
            if (vi.len) { ++nz; ent += vi.len; } else { ++z; }
            es += vi.deg;
        }
    }
    nz = warp_sum(nz);
    ent = warp_sum(ent);
    z = warp_sum(z);
    es = warp_sum(es);
}

// End of a count pass (every block calls it): the LAST block to arrive
// (atomic ticket) turns the per-chunk totals -- 4 counters per chunk: nz
// members, their index entries, zero-degree members, out-degree sum -- into
// exclusive prefixes in `prefix` (the list pass's starting points), writes
// the record's counts and decides whether the ordered list is needed at all:
// after a dense pull whose output frontier gates the next iteration to
// FullScan again, nothing consumes it (record reserved[2] = 1).  totals may
// alias prefix; zero_totals clears them after reading (atomic accumulators).
// The scan of a count pass, by ONE block: per-chunk totals -> exclusive
// prefixes (see count_epilogue).
__device__ __forceinline__ void count_tail(uint64_t B, uint64_t *totals, uint64_t *prefix, bool zero_totals,
                                           wg_iter_rec *rec, int keep_list, uint64_t edges, uint64_t wedge_limit) {
    __shared__ uint64_t sm[33];
    const uint64_t per = (B + blockDim.x - 1) / blockDim.x;
    const uint64_t b0 = threadIdx.x * per, b1 = b0 + per < B ? b0 + per : B;
    uint64_t loc[3] = {0, 0, 0}, les = 0;
    for (uint64_t b = b0; b < b1; ++b) {
        const volatile uint64_t *q = totals + 4 * b;
        loc[0] += q[0]; loc[1] += q[1]; loc[2] += q[2]; les += q[3];
    }
    uint64_t base[3], tot[3];
    for (int f = 0; f < 3; ++f) base[f] = block_exclusive_sum(loc[f], sm, &tot[f]);
    const uint64_t es_all = block_sum(les, sm);
    for (uint64_t b = b0; b < b1; ++b) {
        volatile uint64_t *q = totals + 4 * b;
        volatile uint64_t *o = prefix + 4 * b;
        for (int f = 0; f < 3; ++f) {
            const uint64_t v = q[f];
            o[f] = base[f];
            base[f] += v;
        }
        if (zero_totals) {
            q[0] = 0; q[1] = 0; q[2] = 0; q[3] = 0;
        }
    }
    if (threadIdx.x == 0) {
        rec->nz_packed = (tot[0] << 32) | tot[1];
        rec->z_count = tot[2];
        rec->frontier_out = tot[0] + tot[2];
        rec->out_edge_sum = es_all;
        // the list is consumed only by a Wedge iteration (or the caller)
        const bool wedge_next = es_all > 0 && edges > 0 && es_all < wedge_limit;
        rec->reserved[2] = (keep_list || wedge_next) ? 0 : 1;
    }
}

// End of a count pass (every block calls it): the LAST block to arrive
// (atomic ticket) turns the per-chunk totals -- 4 counters per chunk: nz
// members, their index entries, zero-degree members, out-degree sum -- into
// exclusive prefixes in `prefix` (the list pass's starting points), writes
// the record's counts and decides whether the ordered list is needed at all:
// after a dense pull whose output frontier gates the next iteration to
// FullScan again, nothing consumes it (record reserved[2] = 1).  totals may
// alias prefix; zero_totals clears them after reading (atomic accumulators).
__device__ __forceinline__ void count_epilogue(uint64_t B, uint64_t *totals, uint64_t *prefix, bool zero_totals,
                                               unsigned *counter, wg_iter_rec *rec, int keep_list, uint64_t edges,
                                               uint64_t wedge_limit) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    count_tail(B, totals, prefix, zero_totals, rec, keep_list, edges, wedge_limit);
    if (threadIdx.x == 0) *counter = 0;
}

// keep_list: 1 = always build the list; 0 = decide from the next gate
// (edges, wedge_limit as in ctx_mode).  counter: zero-initialised ticket,
// reset by the last block.
__device__ __forceinline__ void frontier_count_body(const uint32_t *words, uint64_t nbits,
                                                    const uint64_t *idx_off, const uint32_t *outdeg,
                                                    uint64_t *bcount, unsigned *counter, wg_iter_rec *rec,
                                                    int keep_list, uint64_t edges, uint64_t wedge_limit) {
    __shared__ uint64_t s_w[4][CB_THREADS / 32];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint64_t nz, ent, z, es;
    chunk_counts(words, nbits, (uint64_t)blockIdx.x * FB_WORDS + (uint64_t)warp * 32, idx_off, outdeg, nz, ent,
                 z, es);
    if (lane == 0) {
        s_w[0][warp] = nz; s_w[1][warp] = ent; s_w[2][warp] = z; s_w[3][warp] = es;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        uint64_t t = 0;
        for (int w = 0; w < CB_THREADS / 32; ++w) t += s_w[threadIdx.x][w];
        bcount[4ull * blockIdx.x + threadIdx.x] = t;
    }
    count_epilogue(gridDim.x, bcount, bcount, false, counter, rec, keep_list, edges, wedge_limit);
}

__device__ __forceinline__ void frontier_list_body(const uint32_t *words, uint64_t nbits,
                                                   const uint64_t *idx_off, const uint32_t *outdeg,
                                                   const uint64_t *bcount,
                                                   uint32_t *fvert, uint32_t *fpref, uint32_t *tstart,
                                                   const wg_iter_rec *rec, uint64_t chunk = ~0ull) {
    if (*(volatile const uint64_t *)&rec->reserved[2]) return;  // nobody consumes the list
    if (chunk == ~0ull) chunk = blockIdx.x;
    __shared__ uint64_t s_w[3][CB_THREADS / 32];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint64_t wbase = chunk * FB_WORDS + (uint64_t)warp * 32;
    uint64_t nz, ent, z, es;
    chunk_counts(words, nbits, wbase, idx_off, outdeg, nz, ent, z, es);
    if (lane == 0) {
        s_w[0][warp] = nz; s_w[1][warp] = ent; s_w[2][warp] = z;
    }
    __syncthreads();
    uint64_t nzp = bcount[4ull * chunk], entp = bcount[4ull * chunk + 1], zp = bcount[4ull * chunk + 2];
    for (unsigned w = 0; w < warp; ++w) {
        nzp += s_w[0][w];
        entp += s_w[1][w];
        zp += s_w[2][w];
    }
    const uint32_t myw = masked_word(words, wbase + lane, nbits);
    if (__ballot_sync(FULL, myw != 0) == 0) return;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
        const uint32_t x = __shfl_sync(FULL, myw, j);
        if (x == 0) continue;  // warp-uniform
        const uint64_t wi = wbase + j;
        const VertexInfo vi = vertex_info(x, wi, lane, idx_off, outdeg);
        const bool hasd = vi.set && vi.len != 0, zero = vi.set && vi.len == 0;
        const unsigned mnz = __ballot_sync(FULL, hasd), mz = __ballot_sync(FULL, zero);
        const uint64_t elen = hasd ? vi.len : 0u;
        const uint64_t incl = warp_inclusive_sum(elen);
        const uint64_t u = (wi << 5) + lane;
        if (hasd) {
            const uint64_t pos = nzp + __popc(mnz & lt);
            const uint64_t pref = entp + incl - elen;
            fvert[pos] = (uint32_t)u;
            fpref[pos] = (uint32_t)pref;
            if (tstart) mark_tile_starts(tstart, pref, elen, (uint32_t)pos);
        } else if (zero) {
            fvert[nbits - 1 - (zp + __popc(mz & lt))] = (uint32_t)u;
        }
        nzp += __popc(mnz);
        entp += __shfl_sync(FULL, incl, 31);
        zp += __popc(mz);
    }
}

// The same ordered list, one WORD per thread (block = FB_WORDS threads = one
// chunk): the thread counts its word's members (index lengths of its set
// bits only), the block scans the three counts once on top of the chunk's
// prefix (bcount, from the count pass) and each thread writes its members.
// Reads the bitmap once and the degrees of members only -- no recount of
// the whole chunk (frontier_list_body) -- so a sparse frontier costs little.
__device__ __forceinline__ void frontier_list_words(const uint32_t *words, uint64_t nbits,
                                                    const uint64_t *idx_off, const uint32_t *outdeg,
                                                    const uint64_t *bcount, uint32_t *fvert, uint32_t *fpref,
                                                    uint32_t *tstart, const wg_iter_rec *rec, uint64_t chunk) {
    __shared__ uint64_t sm[33];
    if (*(volatile const uint64_t *)&rec->reserved[2]) return;  // nobody consumes the list (block-uniform)
    const uint64_t w = chunk * FB_WORDS + threadIdx.x;
    const uint32_t x = masked_word(words, w, nbits);
    uint64_t nz = 0, ent = 0, z = 0;
    for (uint32_t m = x; m; m &= m - 1) {
        const uint64_t u = (w << 5) + __ffs(m) - 1;
        const uint64_t len = idx_off ? idx_off[u + 1] - idx_off[u] : outdeg[u];
        nz += len != 0;
        ent += len;
        z += len == 0;
    }
    uint64_t nzp = block_exclusive_sum(nz, sm, (uint64_t *)nullptr) + bcount[4 * chunk];
    uint64_t entp = block_exclusive_sum(ent, sm, (uint64_t *)nullptr) + bcount[4 * chunk + 1];
    uint64_t zp = block_exclusive_sum(z, sm, (uint64_t *)nullptr) + bcount[4 * chunk + 2];
    for (uint32_t m = x; m; m &= m - 1) {
        const uint64_t u = (w << 5) + __ffs(m) - 1;
        const uint64_t len = idx_off ? idx_off[u + 1] - idx_off[u] : outdeg[u];
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

__global__ void __launch_bounds__(CB_THREADS) frontier_count_kernel(const uint32_t *words, uint64_t nbits,
                                                                    const uint64_t *idx_off,
                                                                    const uint32_t *outdeg, uint64_t *bcount,
                                                                    unsigned *counter, wg_iter_rec *rec,
                                                                    int keep_list, uint64_t edges,
                                                                    uint64_t wedge_limit) {
    frontier_count_body(words, nbits, idx_off, outdeg, bcount, counter, rec, keep_list, edges, wedge_limit);
}

__global__ void __launch_bounds__(CB_THREADS) frontier_list_kernel(const uint32_t *words, uint64_t nbits,
                                                                   const uint64_t *idx_off, const uint32_t *outdeg,
                                                                   const uint64_t *bcount, uint32_t *fvert,
                                                                   uint32_t *fpref, uint32_t *tstart,
                                                                   const wg_iter_rec *rec) {
    frontier_list_body(words, nbits, idx_off, outdeg, bcount, fvert, fpref, tstart, rec);
}

// The same two passes inside the device loop after a dense pull, which only
// sets next-frontier bits: build iteration it's counts, out-degree sum and
// (when a Wedge iteration follows) member list and tile starts from its
// bitmap (gated on the device mode).
struct FrontierBufs {
    uint32_t *fbits[2], *fvert[2], *fpref[2], *tstart[2];
    uint32_t dst_major, dst_bottom_up;  // a destination-major pull may have counted the frontier already
};

__global__ void __launch_bounds__(CB_THREADS) loop_frontier_count_kernel(LoopCtx c, FrontierBufs f, uint64_t n,
                                                                         const uint64_t *idx_off,
                                                                         const uint32_t *outdeg,
                                                                         uint64_t *bcount, unsigned *counter) {
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_FCOUNT);
    if (ctx_mode(c, it) != MODE_FULL) return;
    if (dst_major_active(c, it, n, f.dst_major, f.dst_bottom_up != 0)) return;  // counted by dense_dst_kernel
    frontier_count_body((it & 1) ? f.fbits[1] : f.fbits[0], n, idx_off, outdeg, bcount, counter, ctx_out(c, it),
                        c.keep_lists, c.edges, c.wedge_limit);
}

__global__ void __launch_bounds__(CB_THREADS) loop_frontier_list_kernel(LoopCtx c, FrontierBufs f, uint64_t n,
                                                                        const uint64_t *idx_off,
                                                                        const uint32_t *outdeg,
                                                                        const uint64_t *bcount) {
    const uint64_t it = ctx_iter(c);
    WG_KTS(it, KTS_FLIST);
    if (ctx_mode(c, it) != MODE_FULL) return;
    const int k = (int)(it & 1);
    frontier_list_words(k ? f.fbits[1] : f.fbits[0], n, idx_off, outdeg, bcount, k ? f.fvert[1] : f.fvert[0],
                        k ? f.fpref[1] : f.fpref[0], k ? f.tstart[1] : f.tstart[0], ctx_out(c, it), blockIdx.x);
}

// ---------------- K3: Wedge transform --------------------------------------
// Load-balanced over index ENTRIES (not vertices), so hub sources with huge
// out-lists do not serialise a thread (the CPU transform lost up to 89% of its
// time to imbalance).  A block takes tiles of TR_TILE entries;
// the list items overlapping the tile are staged in shared memory; each thread
// then walks TR_EPT consecutive entries, OR-ing group bits pos >> shift and
// skipping repeats (a source's positions ascend, so equal groups are adjacent).



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
        // four members per thread and round trip: a tile of a low-degree frontier
        // covers up to TR_TILE members, and the member -> idx_off[v] chain of one
        // member per step (8 dependent steps per thread) was most of a small
        // transform's time
        for (uint64_t k0 = threadIdx.x; k0 < nitems; k0 += 4ull * blockDim.x) {
            uint32_t v[4], p[4];
            uint64_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t k = k0 + (uint64_t)j * blockDim.x;
                v[j] = k < nitems ? fvert[i0 + k] : 0u;
                p[j] = k < nitems ? fpref[i0 + k] : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = k0 + (uint64_t)j * blockDim.x < nitems ? idx_off[v[j]] : 0ull;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t k = k0 + (uint64_t)j * blockDim.x;
                if (k < nitems) {
                    sm.pref[k] = p[j];
                    sm.base[k] = o[j] - p[j];
                }
            }
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
    WG_KTS(it, KTS_TRANSFORM);
    if (ctx_mode(c, it) != MODE_WEDGE) return;
    __shared__ TransformSmem sm;
    transform_phase(c, it, fvert0, fvert1, fpref0, fpref1, tstart0, tstart1, idx_off, idx_pos, shift, gbits,
                    append, glist, ngroups, sm, blockIdx.x, gridDim.x);
}

}  // namespace wg
