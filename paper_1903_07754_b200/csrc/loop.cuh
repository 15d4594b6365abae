// loop.cuh — iteration context shared by every kernel of the device loop.
//
// The device-resident loop (engine.py:330-388 restated for the GPU) keeps one
// wg_iter_rec per iteration in a ring.  Iteration `it` (1-based) consumes the
// frontier produced by iteration it-1 (list parity (it-1)&1, record
// (it-1)%ring; iteration 0 is the initial frontier) and produces list it&1.
// Every kernel re-derives the gate from the previous record, so a batch of
// enqueued iterations needs no host round trip and iterations after
// convergence are no-ops.
#pragma once
#include "common.cuh"

namespace wg {

enum : int { MODE_NONE = 0, MODE_FULL = 1, MODE_WEDGE = 2 };

struct LoopCtx {
    wg_iter_rec *recs;
    uint32_t ring;
    int32_t forced_mode;    // != 0: per-call kernel (backend protocol), no gate
    const uint64_t *ctrl;   // device iteration base (graph replay) or null
    uint64_t it_arg;
    uint64_t wedge_limit;   // wedge iff edges > 0 and edge_sum < wedge_limit
    uint64_t edges;
    int32_t keep_lists;     // WG_RUN_KEEP_LISTS: build every frontier list (traces, exchange)
    int32_t gate_local;     // WG_RUN_LOCAL_GATE: gate on the shard's own index entries
};

__device__ __forceinline__ uint64_t ctx_iter(const LoopCtx &c) {
    return c.it_arg + (c.ctrl ? *(volatile const uint64_t *)c.ctrl : 0ull);
}

// Gate (frontier.py:163-171; engine.py:356-362): the first iteration always
// runs; afterwards iteration it runs iff the frontier produced by it-1 has
// out-edges, and uses the Wedge path iff its edge sum is below the limit.
__device__ __forceinline__ int ctx_mode(const LoopCtx &c, uint64_t it) {
    if (c.forced_mode) return c.forced_mode;
    // graph launches carry an iteration limit in ctrl[1]
    if (c.ctrl && it > *(volatile const uint64_t *)&c.ctrl[1]) return MODE_NONE;
    const wg_iter_rec &p = c.recs[(it - 1) % c.ring];
    const uint64_t sum = *(volatile const uint64_t *)&p.out_edge_sum;
    if (it > 1 && sum == 0) return MODE_NONE;  // convergence is global
    const uint64_t key = c.gate_local ? (*(volatile const uint64_t *)&p.nz_packed & 0xffffffffull) : sum;
    return (c.edges > 0 && key < c.wedge_limit) ? MODE_WEDGE : MODE_FULL;
}

// Debug timeline of the loop's kernels (wg_debug_kernel_timeline; null =
// off): per (iteration, kernel id) the earliest block start and the latest
// block end, %globaltimer ns, stamped by thread 0 of every block.
enum : int {
    KTS_DECIDE = 0, KTS_SPARSE_GATE, KTS_TRANSFORM, KTS_GROUP_COUNT, KTS_GROUP_LIST, KTS_PULL_WEDGE,
    KTS_PULL_SPARSE, KTS_DENSE_DST, KTS_DENSE_TMA, KTS_BOTTOM_UP, KTS_FLOOR, KTS_IDENT, KTS_FCOUNT, KTS_FLIST,
    KTS_FINALIZE, KTS_STEP, KTS_SEED, KTS_PERSIST, KTS_IDS
};
static __device__ uint64_t *g_kts = nullptr;
static __device__ uint64_t g_kts_cap = 0;

__device__ __forceinline__ uint64_t kts_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int ID>
struct KtsScope {
    uint64_t it;  // the only state kept live across the kernel
    __device__ __forceinline__ explicit KtsScope(uint64_t i) : it(i) {
        uint64_t *buf = g_kts;
        if (buf != nullptr && threadIdx.x == 0 && it < g_kts_cap)
            atomicMin((unsigned long long *)(buf + (it * KTS_IDS + ID) * 2), (unsigned long long)kts_now());
    }
    __device__ __forceinline__ ~KtsScope() {
        uint64_t *buf = g_kts;
        if (buf != nullptr && threadIdx.x == 0 && it < g_kts_cap)
            atomicMax((unsigned long long *)(buf + (it * KTS_IDS + ID) * 2 + 1), (unsigned long long)kts_now());
    }
};
#define WG_KTS(it, id) ::wg::KtsScope<id> _wg_kts_scope((it))

__device__ __forceinline__ wg_iter_rec *ctx_out(const LoopCtx &c, uint64_t it) {
    return &c.recs[it % c.ring];
}
__device__ __forceinline__ const wg_iter_rec *ctx_in(const LoopCtx &c, uint64_t it) {
    return &c.recs[(it - 1) % c.ring];
}

// Destination-major dense pulls (pull.cuh dense_dst_kernel): always for the
// floor (CC-like) kind; for the bottom-up (BFS) kind once the visited set
// (record reserved[4]: members of the initial and every produced frontier so
// far) holds at least V/1024 vertices -- a dense pull from a single root
// finds no hits and scans whole in-lists, which the vector-parallel TMA
// pipeline streams faster; from there on the per-destination early exit wins
// (BFS s26 iteration 2, 0.9% visited: 2.83 + 0.09 ms against 3.77 + 0.32 ms;
// V/16 before the lane redistribution of dense_dst_phase).
constexpr uint64_t DST_BU_VISITED_DIV = 1024;

__device__ __forceinline__ bool dst_major_active(const LoopCtx &c, uint64_t it, uint64_t n, uint32_t dst_major,
                                                 bool bottom_up) {
    if (!dst_major) return false;
    if (!bottom_up) return true;
    // frontier(it-1)'s size from its counts (set by the pull / compaction that
    // produced it, before its end-of-iteration record) plus every earlier
    // frontier's (the cumulative count end_of_iteration keeps in reserved[4])
    const wg_iter_rec *in = ctx_in(c, it);
    uint64_t seen = (*(volatile const uint64_t *)&in->nz_packed >> 32) + *(volatile const uint64_t *)&in->z_count;
    if (it >= 2) {
        const wg_iter_rec *pp = &c.recs[(it - 2) % c.ring];
        seen += it == 2 ? *(volatile const uint64_t *)&pp->frontier_out : *(volatile const uint64_t *)&pp->reserved[4];
    }
    return seen * DST_BU_VISITED_DIV >= n;
}

}  // namespace wg
