/*
 * wedge_b200.h — C ABI of the B200-native Wedge-Frontier pull engine.
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every pointer named
 * `d_*` or documented as "device" is a CUDA device pointer; `stream` is a
 * cudaStream_t passed as void*.  Every function returns WG_OK (0) or a
 * negative WG_E* code; the message of the last error on the calling thread is
 * available from wg_last_error().  Nothing is allocated behind the caller's
 * back: scratch space comes from caller-provided workspaces whose sizes are
 * queried first.
 *
 * Reference interface each entry point replaces (wedgegraph 0.1.0,
 * /root/reference/pkg/src/wedgegraph):
 *
 *   wg_build_layout      build_pull_topology  graph.py:220-263
 *                        build_edge_index     graph.py:283-301
 *                        compute_out_degrees  graph.py:277-280
 *   wg_transform         Backend.transform    kernels.py:116-125 -> _kernels.pyx:55-62
 *                        (transform_frontier  frontier.py:174-209)
 *   wg_pull_full         Backend.pull_full    kernels.py:81-95   -> _kernels.pyx:98-110
 *   wg_pull_wedge        Backend.pull_wedge   kernels.py:97-114  -> _kernels.pyx:176-189
 *   wg_covered_groups    covered_positions    _kernels_py.py:24-32 (wedge_covered_vectors,
 *                                                                  frontier.py:156-160)
 *   wg_run_*             run_until_convergence engine.py:330-388 (device-resident loop)
 *   wg_pagerank          (no reference symbol; BASELINE.json config 5)
 *   wg_rmat_edges        _generate_rmat       graph_io.py:188-202 (bit-identical PCG64 stream)
 *   wg_weights_hash      synthesize_weights   graph_io.py:205-221
 *   wg_canonical_edges   symmetrize(dedup)    graph_io.py:87-112 (+ directed dedup)
 */
#ifndef WEDGE_B200_H
#define WEDGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WG_ABI_VERSION 1

#define WG_OK 0
#define WG_EINVAL -1     /* bad argument (null pointer, size, unsupported width) */
#define WG_ECUDA -2      /* CUDA runtime error (launch, copy, device fault) */
#define WG_ENOSPACE -3   /* workspace too small / capacity exceeded */
#define WG_EOVERFLOW -4  /* a uint32 value would have exceeded 0xFFFFFFFE (run is invalid) */

/* Vertex value encodings. */
#define WG_VAL_U32 0 /* uint32 values, 0xFFFFFFFF = unreached (fast path) */
#define WG_VAL_I64 1 /* int64 values with the reference sentinel (engine.py:41-43) */

#define WG_NO_LANE 0xFFFFFFFFu /* padding lane in vsrc */
#define WG_TRANSFORM_TILE 2048u /* edge-index entries per transform tile */

/* Device-resident pull layout.  All pointers device.
 * vsrc / vdst / vw must stay readable for 16 vectors past nvec (the dense
 * pull streams them with TMA bulk copies rounded up to 16 bytes). */
typedef struct wg_graph {
    uint32_t n;          /* vertices */
    uint32_t width;      /* lanes per vector: 1, 2, 4, 8 (graph.py:215-217) */
    uint64_t nvec;       /* vectors */
    uint64_t edges;      /* |E| as stored (PullTopology.edge_count) */
    uint64_t entries;    /* edge-index entries (EdgeIndex.positions length) */
    const uint32_t *vsrc;    /* [nvec*width] lane sources, WG_NO_LANE padded */
    const uint32_t *vdst;    /* [nvec] destination of each vector */
    const uint32_t *vw;      /* [nvec*width] lane weights or NULL */
    const uint64_t *idx_off; /* [n+1] edge-index offsets */
    const uint32_t *idx_pos; /* [entries] ascending de-duplicated vector positions */
    const uint32_t *outdeg;  /* [n] out-degrees */
    uint32_t flags;          /* WG_GRAPH_* */
    const uint8_t *vw8;      /* optional [nvec*width] lane weights as bytes (every weight <= 255,
                                wg_narrow_weights); the dense pull then streams these instead of
                                vw (16 bytes of readable slack past the end) */
    const uint32_t *voff;    /* optional [n+1] first vector of each destination (the run-length form
                                of vdst, wg_vector_offsets_from_dst): enables the destination-major
                                dense pulls (a thread / warp per destination, no vdst stream) */
    const uint32_t *vfirst;  /* optional (with voff) [n] first lane of each destination's first vector =
                                its smallest source, WG_NO_LANE without in-edges: the destination-major
                                pulls' first probe as one coalesced load */
} wg_graph;

/* Every vertex's edge-index length equals its out-degree (no parallel edges;
 * set by the layout builders when verified): frontier compaction then reads
 * only the 4-byte degrees. */
#define WG_GRAPH_LENS_ARE_DEGREES 1

/* MinPlusKernel (engine.py:50-63). */
typedef struct wg_minplus {
    int32_t filter_unvisited;
    int32_t use_weight;
    int64_t apply_increment;
    int64_t sentinel; /* WG_VAL_I64 only: the reference's UNREACHED */
} wg_minplus;

const char *wg_last_error(void);
int wg_abi_version(void);
int wg_device_sm_count(int *out);

/* ---------------- layout construction (graph.py:220-301) ---------------- */
/* Upper bound on vectors for m edges over n vertices at `width`. */
uint64_t wg_vector_capacity(uint64_t m, uint32_t n, uint32_t width);
/* Scratch bytes for wg_build_layout. */
size_t wg_layout_scratch_bytes(uint64_t m, uint32_t n);
/* Edges (d_src, d_dst, optional d_w; device, length m) -> layout.  Outputs are
 * caller-allocated: d_vsrc/d_vw [cap*width], d_vdst [cap], d_idx_off [n+1],
 * d_idx_pos [m], d_outdeg [n].  h_counts (host) receives {nvec, entries}.
 * Synchronises `stream` to read the counts back. */
int wg_build_layout(uint32_t n, uint64_t m, const uint32_t *d_src, const uint32_t *d_dst,
                    const uint32_t *d_w, uint32_t width, uint64_t vec_capacity, uint32_t *d_vsrc,
                    uint32_t *d_vdst, uint32_t *d_vw, uint64_t *d_idx_off, uint32_t *d_idx_pos,
                    uint32_t *d_outdeg, void *d_scratch, size_t scratch_bytes,
                    uint64_t *h_counts, void *stream);

/* Rebuild the derived parts of a layout from its lanes (g->vsrc, n, width,
 * nvec, edges = valid lanes): the edge index d_idx_off [n+1] / d_idx_pos
 * [edges] (build_edge_index graph.py:283-301) and d_outdeg [n]
 * (compute_out_degrees graph.py:277-280); h_entries (host) receives the
 * index length.  Synchronises `stream`. */
size_t wg_index_scratch_bytes(uint64_t lanes, uint32_t n);
int wg_build_index(const wg_graph *g, uint64_t *d_idx_off, uint32_t *d_idx_pos, uint32_t *d_outdeg,
                   void *d_scratch, size_t scratch_bytes, uint64_t *h_entries, void *stream);
/* The same index built chunk by chunk as the lanes arrive (chunks in
 * ascending vector order, each of at most max_chunk_lanes lanes; chunk 0
 * first): wg_index_chunk sorts a chunk's (source, vector) pairs and ranks
 * them behind the earlier chunks' entries (asynchronous); wg_index_finish
 * scatters every entry to its place and writes d_idx_off / d_idx_pos /
 * d_outdeg (synchronises; falls back to wg_build_index -- then the scratch
 * must also hold wg_index_scratch_bytes -- when the graph has parallel
 * edges). */
size_t wg_index_chunked_scratch_bytes(uint64_t lanes, uint64_t max_chunk_lanes, uint32_t n);
int wg_index_chunk(const wg_graph *g, uint64_t v_begin, uint64_t v_end, uint32_t chunk,
                   uint64_t max_chunk_lanes, void *d_scratch, size_t scratch_bytes, void *stream);
int wg_index_finish(const wg_graph *g, uint64_t max_chunk_lanes, uint64_t *d_idx_off, uint32_t *d_idx_pos,
                    uint32_t *d_outdeg, void *d_scratch, size_t scratch_bytes, uint64_t *h_entries,
                    void *stream);
/* vec_dst from per-destination vector offsets d_voff [n+1] (the run-length
 * form of PullTopology.vec_dst, graph.py:240-243): run heads + max-scan, with
 * d_scratch of wg_expand_scratch_bytes(nvec) bytes.  Asynchronous. */
size_t wg_expand_scratch_bytes(uint64_t nvec);
/* Degrees in the compact upload form: d_deg[v] = d_deg8[v] (min(deg, 255)),
 * then d_big holds nbig (vertex, degree) pairs for the larger ones. */
int wg_widen_degrees(uint32_t n, const uint8_t *d_deg8, const uint32_t *d_big, uint64_t nbig, uint32_t *d_deg,
                     void *stream);
/* d_voff [n+1] = exclusive scan of ceil(indeg / width): the per-destination
 * vector offsets from the in-degrees. */
size_t wg_vector_offsets_scratch_bytes(uint32_t n);
int wg_vector_offsets(uint32_t n, const uint32_t *d_indeg, uint32_t width, uint32_t *d_voff, void *d_scratch,
                      size_t scratch_bytes, void *stream);
int wg_expand_destinations(uint32_t n, const uint32_t *d_voff, uint64_t nvec, uint32_t *d_vdst, void *d_scratch,
                           size_t scratch_bytes, void *stream);

/* Lane weights as bytes: writes d_vw8 [nvec*width] and sets *h_fits (host) to
 * 1 iff every weight is <= 255 (else d_vw8 must not be used).  Synchronises. */
int wg_narrow_weights(const wg_graph *g, uint8_t *d_vw8, int *h_fits, void *stream);
/* The inverse: vw [lanes] = vw8 (e2e uploads of byte weights). Asynchronous. */
int wg_widen_weights(uint64_t lanes, const uint8_t *d_vw8, uint32_t *d_vw, void *stream);

/* Lane sources as fixed-width bit fields (the compact e2e upload format):
 * bits = wg_lane_bits(n) = bit length of n, so every id < n and the empty
 * lane (all ones) fit; lane l occupies bits [l*bits, (l+1)*bits) of the
 * little-endian uint32 word stream of wg_packed_lane_words(lanes, bits)
 * words.  Lane ranges whose begin is a multiple of 32 start on a word, so
 * chunks of the stream can be copied and unpacked independently. */
uint32_t wg_lane_bits(uint32_t n);
uint64_t wg_packed_lane_words(uint64_t lanes, uint32_t bits);
int wg_pack_lanes(uint64_t lanes, const uint32_t *d_lanes, uint32_t bits, uint32_t *d_packed,
                  void *stream);
/* d_lanes[l] for l in [lane_begin, lane_end) from the packed stream. */
int wg_unpack_lanes(const uint32_t *d_packed, uint32_t bits, uint64_t lane_begin, uint64_t lane_end,
                    uint32_t *d_lanes, void *stream);

/* Delta-coded lane sources (the compact e2e upload format, codec.cu): lane
 * codes 0 = empty, src+1 at the first lane of a destination or of a block,
 * else src - previous src + 1; each vector's W codes take width[v] (its
 * largest code's bit length) bits, the vectors of a block of
 * WG_CODED_BLOCK_VECTORS back to back, every block starting on a uint32 word
 * at bit block_base[b] (block_base has wg_coded_blocks(nvec) + 1 entries, the
 * last = total bits).  Lanes must ascend within each destination (the pull
 * layout, graph.py:220-263). */
#define WG_CODED_BLOCK_VECTORS 1024
uint64_t wg_coded_blocks(uint64_t nvec);
uint64_t wg_coded_max_words(uint64_t nvec, uint32_t width);
/* uint32 words of the width array: width - 1 of each vector in 5 bits, 160
 * words per block. */
uint64_t wg_coded_width_words(uint64_t nvec);
size_t wg_coded_scratch_bytes(uint64_t nvec);
/* Encode g's lanes: d_stream [wg_coded_max_words], d_widths [wg_coded_width_words],
 * d_block_base [blocks + 1]; *h_words = stream words used.  Synchronises;
 * WG_EINVAL when a destination's lanes are not ascending. */
int wg_encode_lanes(const wg_graph *g, uint32_t *d_stream, uint32_t *d_widths, uint64_t *d_block_base,
                    void *d_scratch, size_t scratch_bytes, uint64_t *h_words, void *stream);
/* Decode blocks [block_begin, block_end) into d_vsrc (needs d_vdst of every
 * vector of those blocks and the one before). */
int wg_decode_lanes(uint64_t nvec, uint32_t width, const uint32_t *d_vdst, const uint32_t *d_stream,
                    const uint32_t *d_widths, const uint64_t *d_block_base, uint64_t block_begin,
                    uint64_t block_end, uint32_t *d_vsrc, void *stream);

/* Placed index: the edge index of wg_build_index up to the order inside each
 * source's position list (the engine does not depend on it), built without a
 * sort from the out-degrees g->outdeg (the `degrees` input of
 * run_until_convergence, engine.py:330) under the claim that every index
 * length equals the degree (no parallel edges).  begin: d_idx_off = scan of
 * the degrees; chunk / coded: each lane of the vectors (blocks) takes the
 * next slot of its source (coded also decodes the blocks into g->vsrc);
 * end: synchronises, *h_ok = 1 iff the claim held and the index is complete
 * (else rebuild it with wg_build_index; placement never writes past
 * g->entries slots).  Scratch of
 * wg_index_placed_scratch_bytes(n) bytes, shared by the calls. */
size_t wg_index_placed_scratch_bytes(uint32_t n);
int wg_index_place_begin(const wg_graph *g, uint64_t *d_idx_off, void *d_scratch, size_t scratch_bytes,
                         void *stream);
int wg_index_place_chunk(const wg_graph *g, uint64_t v_begin, uint64_t v_end, uint64_t *d_idx_off,
                         uint32_t *d_idx_pos, void *d_scratch, size_t scratch_bytes, void *stream);
int wg_index_place_coded(const wg_graph *g, const uint32_t *d_stream, const uint32_t *d_widths,
                         const uint64_t *d_block_base, uint64_t block_begin, uint64_t block_end,
                         uint64_t *d_idx_off, uint32_t *d_idx_pos, void *d_scratch, size_t scratch_bytes,
                         void *stream);
int wg_index_place_end(const wg_graph *g, void *d_scratch, size_t scratch_bytes, int *h_ok, void *stream);

/* wg_index_chunk over delta-coded blocks [block_begin, block_end): decodes
 * them into g->vsrc (needs g->vdst) and adds their index entries. */
int wg_index_chunk_coded(const wg_graph *g, const uint32_t *d_stream, const uint32_t *d_widths,
                         const uint64_t *d_block_base, uint64_t block_begin, uint64_t block_end, uint32_t chunk,
                         uint64_t max_chunk_lanes, void *d_scratch, size_t scratch_bytes, void *stream);

/* ---------------- per-call kernels (backend protocol, kernels.py:55-125) --- */
/* Workspace for wg_transform / wg_pull_wedge / wg_covered_groups. */
size_t wg_kernel_workspace_bytes(const wg_graph *g, int shift);
/* Transform: frontier bitmap (uint32 LE words over n) -> wedge group bitmap
 * (OR-ed into d_wedge_words, words over ceil(nvec>>shift)).  h_visited
 * (host) receives the index entries visited.  Synchronises. */
int wg_transform(const wg_graph *g, const uint32_t *d_frontier_words, int shift,
                 uint32_t *d_wedge_words, void *d_ws, size_t ws_bytes, uint64_t *h_visited,
                 void *stream);
/* Dense pull over all vectors.  d_prev/d_nxt hold values of `val_type`;
 * d_nxt must equal d_prev on entry (engine.py:264).  Bits of updated
 * destinations are OR-ed into d_out_words.  h_touched (host) receives
 * vectors touched.  Synchronises. */
int wg_pull_full(const wg_graph *g, int val_type, const void *d_prev, void *d_nxt,
                 uint32_t *d_out_words, const wg_minplus *k, void *d_ws, size_t ws_bytes,
                 uint64_t *h_touched, void *stream);
/* Pull restricted to vectors covered by set bits of d_wedge_words at `shift`. */
int wg_pull_wedge(const wg_graph *g, const uint32_t *d_wedge_words, int shift, int val_type,
                  const void *d_prev, void *d_nxt, uint32_t *d_out_words, const wg_minplus *k,
                  void *d_ws, size_t ws_bytes, uint64_t *h_touched, void *stream);
/* Ascending list of set group ids of d_wedge_words (group_count bits) into
 * d_groups; h_count (host) receives their number. */
int wg_covered_groups(const uint32_t *d_wedge_words, uint64_t group_count, uint32_t *d_groups,
                      void *d_ws, size_t ws_bytes, uint64_t *h_count, void *stream);

/* ---------------- device-resident convergence loop (engine.py:330-388) ---- */
/* Per-iteration record written by the device (16 x uint64). */
typedef struct wg_iter_rec {
    uint64_t mode;             /* 0 not run, 1 FullScan, 2 Wedge */
    uint64_t active_edges;     /* sum outdeg of the consumed frontier (engine.py:361) */
    uint64_t vectors_touched;
    uint64_t frontier_out;     /* produced frontier size */
    uint64_t out_edge_sum;     /* sum outdeg of the produced frontier */
    uint64_t nz_packed;        /* (members with out-edges << 32) | their index entries */
    uint64_t z_count;          /* produced members without out-edges */
    uint64_t covered_vectors;  /* WedgeFrontier.covered_vector_count (frontier.py:143-150) */
    uint64_t transform_entries;/* WedgeFrontier.entries_visited */
    uint64_t groups;           /* selected wedge groups */
    uint64_t overflow;         /* WG_VAL_U32 overflow flag */
    uint64_t reserved[5];
    uint64_t lanes_read;       /* destination-major dense pulls: edge lanes read (vectors x W, or
                                  single first-lane probes) ... */
    uint64_t gathers;          /* ... and value gathers / frontier-bit tests made */
    uint64_t spare[14];        /* (records are 32 words) */
} wg_iter_rec;

/* Device buffers of a run; all caller-allocated (sizes from
 * wg_run_buffer_sizes).  vals[2] hold `val_type` values. */
typedef struct wg_run_bufs {
    void *vals[2];          /* [n] each */
    uint32_t *fbits[2];     /* [ceil(n/32)] each, zero on init */
    uint32_t *fvert[2];     /* [n] frontier lists */
    uint32_t *fpref[2];     /* [n] entry prefixes of the lists */
    uint32_t *tstart[2];    /* [entries/WG_TRANSFORM_TILE + 2] list position of the member
                               covering each transform tile's first entry */
    uint32_t *gbits;        /* [ceil(groups/32)] zero on init */
    uint32_t *glist;        /* [groups] */
    uint64_t *bcount;       /* [blocks] compaction scratch */
    wg_iter_rec *recs;      /* [ring] */
    uint64_t *ctrl;         /* [4]: base iteration, ... */
    uint32_t ring;          /* record ring length */
    uint32_t *gbits_alt;    /* optional second group bitmap [ceil(groups/32)], zero on init, and */
    uint32_t *glist_alt;    /* group list [groups]: with both, the persistent sparse loop fuses the
                               transform of iteration k+1 into the pull of k (one barrier per
                               iteration); without, it runs transform and pull as two phases */
    uint32_t *work;         /* optional [n] scratch of the destination-major dense pulls (their list of
                               destinations with long in-lists, handled a warp each); required when
                               the graph carries voff */
} wg_run_bufs;

typedef struct wg_run_params {
    int32_t val_type;
    int32_t shift;          /* log2(vectors per group) */
    wg_minplus kern;
    uint64_t wedge_limit;   /* wedge iff E>0 and edge_sum < wedge_limit (= ceil(num*E/den)) */
    void *timer;            /* optional wg_timer*: CUDA events around each launch group */
    int32_t flags;          /* WG_RUN_* */
    int64_t level_base;     /* WG_RUN_FIRST_HIT: the common value of the initial frontier (the
                               members of frontier k then all hold level_base + k*increment) */
} wg_run_params;

/* The caller asserts level-synchronous values (a filtered, unweighted kernel
 * whose initially finite values are all equal and all in the initial
 * frontier, e.g. bfs_program): then every finite in-neighbour of an
 * unvisited destination carries the same level, so the first one found is
 * the minimum and the filtered pulls skip the rest of that destination's
 * vectors (bottom-up early exit).  Results and counters
 * are unchanged. */
#define WG_RUN_FIRST_HIT 1
/* (With WG_RUN_FIRST_HIT, dense pulls after the first iteration are
 * bottom-up: an unvisited destination tests its sources against the
 * previous frontier's bitmap instead of gathering their values.) */
/* Build every produced frontier's member list (traces, exchange).  Without
 * it a dense pull whose frontier gates the next iteration to FullScan skips
 * the list (nothing consumes it; its record has reserved[2] = 1). */
#define WG_RUN_KEEP_LISTS 2
/* The caller asserts that the initial values are the vertex ids (value[v] ==
 * v, e.g. cc_program): the first iteration's unweighted, unfiltered dense
 * pull then needs no gathers -- a destination's smallest message is its
 * smallest source, lane 0 of its first vector (the layout's lanes ascend
 * within a destination, graph.py:235), one load per destination.  Results
 * and counters unchanged. */
#define WG_RUN_IDENTITY_INIT 8
/* uint32 values, unfiltered program: a dense pull reads prev[d] ahead and a
 * destination already at 0 -- below which no candidate can go -- gathers
 * nothing (it is still counted as touched); unweighted, from the third
 * iteration on, the dense pull is an init pass plus an atomic-min pull over
 * the vectors of destinations not at 0 (env WG_FLOOR_KERNELS=0 keeps the
 * pipeline).  Results and counters unchanged. */
#define WG_RUN_FLOOR_SKIP 16
/* Per-shard independent gate (destination-sharded runs; SURVEY 8(f) row 3,
 * PAPER.md:251 future work): the Wedge / FullScan decision of an iteration
 * uses this shard's share of the frontier's out-edges -- the index entries
 * of its members in the shard's LOCAL edge index -- against the shard's own
 * entry count (wedge_limit then = ceil(num * local entries / den)), instead
 * of the global edge sum.  Values and frontiers are unchanged (any covering
 * of the active edges gives the same pull, Appendix A.7); modes and work
 * counters become per shard.  Convergence stays global. */
#define WG_RUN_LOCAL_GATE 32

/* Element counts: [0] fbits words, [1] groups, [2] gbits words, [3] bcount
 * entries, [4] tstart entries (the caller multiplies by element sizes). */
int wg_run_buffer_sizes(const wg_graph *g, int shift, uint64_t *h_sizes5);
/* Seed iteration 0 from the initial-frontier bitmap d_init_words (uint32
 * words over n): builds list 0 and record 0, zeroes record 1.  The caller has
 * already written vals[0] == vals[1] == initial values. */
int wg_run_init(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                const uint32_t *d_init_words, void *stream);
/* wg_run_init plus both value buffers written from d_init_values ([n] values
 * of p->val_type) -- one launch for the whole initialisation
 * (ValueBuffers.initialize, engine.py:100; VertexFrontier.from_vertices,
 * frontier.py:79).  h_all_counts4 (optional, host): frontier 0 is EVERY vertex
 * (engine apps: CC) and these are its counts -- members with index entries,
 * their entries, members without, out-degree sum -- so no compaction pass
 * runs; only valid when iteration 1 is dense and no member lists are kept
 * (WG_EINVAL otherwise); d_init_words may then be null. */
int wg_run_seed(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, const void *d_init_values,
                const uint32_t *d_init_words, const uint64_t *h_all_counts4, void *stream);
/* Enqueue iterations [it_begin, it_begin + count) (1-based).  Each kernel
 * re-derives the gate and the converged flag on device from the previous
 * record, so iterations after convergence are no-ops.  Asynchronous. */
int wg_run_enqueue(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                   uint64_t it_begin, uint32_t count, void *stream);
/* Enqueue only the launches of one iteration (for CUDA-graph capture); the
 * iteration number comes from the device counter b->ctrl[0] which the last
 * launch advances. */
int wg_run_enqueue_counter(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                           uint32_t count, void *stream);

/* CUDA graph of `count` iterations driven by the device iteration counter
 * (b->ctrl[0]); each launch advances the counter by `count`.  The graph is
 * captured on `stream` once and replayed with wg_run_graph_launch; the host
 * reads the records after each replay.  Returns an opaque handle or NULL. */
void *wg_run_graph_create(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                          uint32_t count, void *stream);
int wg_run_graph_launch(void *graph, void *stream);
void wg_run_graph_destroy(void *graph);
/* Device-resident loop as ONE CUDA graph: a conditional WHILE node whose body
 * is one iteration followed by a single-thread kernel that advances the
 * device iteration counter and clears the loop condition when the produced
 * frontier has no out-edges (engine.py:386) or the iteration limit is hit.
 * wg_run_loop_launch runs iterations ctrl[0]+1 .. at most max_iteration with
 * no host round trip; the host then reads ctrl[0] and the records. */
void *wg_run_loop_graph_create(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                               void *stream);
int wg_run_loop_launch(void *graph, const wg_run_bufs *b, uint64_t max_iteration, void *stream);
/* The same loop graph with the run's seed (wg_run_seed) captured in front of
 * it, reading the initial values / frontier words from d_seed_values /
 * d_seed_words (the graph's own buffers): a whole run is ONE launch.
 * launch_seeded first copies the caller's initial state into those buffers
 * (skipped when the pointers are the same). */
void *wg_run_loop_graph_create_seeded(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                                      const void *d_seed_values, const uint32_t *d_seed_words,
                                      const uint64_t *h_all_counts4, void *stream);
int wg_run_loop_launch_seeded(void *graph, const wg_run_bufs *b, uint64_t max_iteration, const void *d_init_values,
                              void *d_seed_values, size_t value_bytes, const uint32_t *d_init_words,
                              uint32_t *d_seed_words, size_t word_bytes, void *stream);
/* The persistent cooperative Wedge loop on its own (outside any graph): runs
 * consecutive Wedge iterations ctrl[0]+1 .. up to max_iteration and stops at
 * the first non-Wedge iteration; used by drivers and profilers. */
int wg_run_persistent(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p,
                      uint64_t max_iteration, void *stream);
/* Profiling aid: record 4 %globaltimer stamps per persistent-loop iteration
 * (start, after transform, after pull, after end-of-iteration) into d_buf
 * (4*iterations uint64); pass NULL to disable. */
/* Debug: kernel timeline of the device loop.  d_buf: [iterations][wg_debug_kernel_ids()][2]
 * uint64 (start = earliest block start, initialise to ~0; end = latest block end, initialise
 * to 0; %globaltimer ns); null switches it off. */
int wg_debug_kernel_timeline(uint64_t *d_buf, uint64_t iterations);
uint32_t wg_debug_kernel_ids(void);
int wg_debug_phase_buffer(uint64_t *d_buf, uint64_t iterations);

/* ---------------- multi-GPU exchange ----------------------- */
/* Destination-range sharding: each rank's layout holds the vectors of its
 * destination range (global ids) and a local edge index; values and the
 * frontier are replicated.  After wg_run_enqueue(it, 1):
 *   wg_exchange_pack   copies the members produced by iteration `it` on this
 *                      rank and their new values into d_verts / d_vals
 *                      (capacity entries); h_count receives the count;
 *   wg_exchange_apply  writes every rank's (vertex, value) pairs into both
 *                      value buffers, marks them in the frontier bitmap and
 *                      rebuilds the frontier list and record of `it` for the
 *                      GLOBAL frontier (so every rank's next gate agrees). */
int wg_exchange_pack(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                     uint32_t *d_verts, void *d_vals, uint64_t capacity, uint64_t *h_count,
                     void *stream);
int wg_exchange_apply(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                      const uint32_t *d_verts, const void *d_vals, uint64_t count, void *stream);
/* Host-sync-free form for fixed-size collectives.  A message is a 16-byte
 * header (u64 entry count, u64 overflow flag of the sender's record) + (vertex, value)
 * entries of 8 bytes (WG_VAL_U32)
 * or 16 bytes (WG_VAL_I64); wg_exchange_bytes(k, val_type) is the size of a
 * message truncated to k entries.  pack_all writes this rank's members of
 * iteration `it` (up to `capacity`); after an all-gather of equal prefixes
 * of cap entries, apply_all applies every rank's first min(count, cap)
 * entries, rebuilds the global frontier and writes the largest count into
 * d_status[0] (> cap: gather a longer prefix and apply again -- idempotent)
 * and 1 into d_status[1] when any rank's iteration overflowed uint32
 * (d_status: 2 words). */
/* Dense iterations (most vertices may change): instead of (vertex, value)
 * pairs, every rank contributes its owned value slice [lo, hi) of iteration
 * `it` (slice_pack copies it into d_slice); after an all-gather of S-value
 * slices (S >= every rank's range), apply_slices writes all n values into
 * both buffers, keeps this rank's (`self`) own frontier bits and derives the
 * other ranks' from the values (new < previous: values never increase), and
 * rebuilds the list and record of `it`.  d_bounds: device uint32 [world+1]. */
int wg_exchange_slice_pack(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                           uint32_t lo, uint32_t hi, void *d_slice, void *stream);
int wg_exchange_apply_slices(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                             const void *d_slices, const uint32_t *d_bounds, uint32_t world, uint32_t self,
                             uint64_t S, void *stream);
uint64_t wg_exchange_bytes(uint64_t entries, int val_type);
int wg_exchange_pack_all(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                         void *d_buf, uint64_t capacity, void *stream);
int wg_exchange_apply_all(const wg_graph *g, const wg_run_bufs *b, const wg_run_params *p, uint64_t it,
                          const void *d_parts, uint32_t world, uint64_t cap, uint64_t *d_status,
                          void *stream);

/* ---------------- measurement --------------------------------------------- */
/* Event timer: when attached to wg_run_params.timer, wg_run_enqueue records a
 * CUDA event pair (on the launch stream) around the Wedge preparation
 * (transform + group compaction, kind 1), the pull (kind 2) and the
 * end-of-iteration kernel (kind 3) of every enqueued iteration. */
void *wg_timer_create(int capacity);
void wg_timer_destroy(void *timer);
int wg_timer_reset(void *timer);
/* Elapsed ms of each recorded pair (stream must be complete); h_kind and
 * h_iter receive the launch group and the iteration.  *h_count = pairs. */
int wg_timer_read(void *timer, float *h_ms, int32_t *h_kind, int64_t *h_iter, int capacity,
                  int *h_count);
/* Kernels launched by this library since load (all entry points). */
uint64_t wg_launch_count(void);

/* ---------------- PageRank (BASELINE config 5) ---------------------------- */
/* float32 ranks, damping, fixed iterations, dangling mass spread uniformly.
 * d_rank [n] out; d_acc [n], d_contrib [n] scratch; d_scal [4] doubles scratch. */
/* Deterministic (no float atomics: bit-identical runs on the same GPU and
 * build).  d_ws: wg_pagerank_ws_bytes(g) bytes of device scratch. */
size_t wg_pagerank_ws_bytes(const wg_graph *g);
int wg_pagerank(const wg_graph *g, int iterations, double damping, float *d_rank, float *d_acc,
                float *d_contrib, double *d_scal, void *d_ws, size_t ws_bytes, void *stream);
/* Hot-source layout for PageRank (no reference symbol; BASELINE.json config
 * 5).  The pull gathers contrib[src] once per edge; RMAT's heavy sources are
 * scattered over the id space.  wg_pagerank_hot_layout numbers the vertices
 * that have out-edges by descending out-degree (stable): d_order [n] = slot ->
 * vertex (slots >= *h_nsrc are the vertices without out-edges, ascending),
 * d_od_hot [n] = out-degree per slot, d_vsrc_hot [nvec*width, same slack as
 * vsrc] = g's lanes with each source replaced by its slot.  Lane order is kept,
 * so every sum is taken in the order wg_pagerank takes it.  Synchronises.
 * d_ws: wg_pagerank_hot_ws_bytes(g).  wg_pagerank_hot = wg_pagerank through
 * that layout (d_contrib needs *h_nsrc floats; d_ws: wg_pagerank_ws_bytes). */
size_t wg_pagerank_hot_ws_bytes(const wg_graph *g);
int wg_pagerank_hot_layout(const wg_graph *g, uint32_t *d_vsrc_hot, uint32_t *d_order, uint32_t *d_od_hot,
                           uint64_t *h_nsrc, void *d_ws, size_t ws_bytes, void *stream);
int wg_pagerank_hot(const wg_graph *g, const uint32_t *d_vsrc_hot, const uint32_t *d_order,
                    const uint32_t *d_od_hot, uint64_t nsrc, int iterations, double damping, float *d_rank,
                    float *d_acc, float *d_contrib, double *d_scal, void *d_ws, size_t ws_bytes, void *stream);
/* The two halves of one iteration, for destination-sharded runs (SURVEY
 * §8(e)): prep(it) applies the accumulated sums of iteration it-1 to all n
 * ranks (it = 0: 1/n), writes d_rank when non-null, zeroes d_acc, builds the
 * contributions r/outdeg and the dangling mass of iteration it (d_scal[4],
 * zeroed at it = 0).  prep(iterations) with d_rank yields the result.
 * d_ws: wg_pagerank_prep_ws_bytes(n) bytes (shared by prep and pull). */
size_t wg_pagerank_prep_ws_bytes(uint32_t n);
int wg_pagerank_prep(uint32_t n, int it, double damping, const uint32_t *d_outdeg, float *d_acc,
                     float *d_contrib, float *d_rank, double *d_scal, void *d_ws, size_t ws_bytes,
                     void *stream);
/* Sum the contributions of g's vectors into d_acc[dst - dst_base] (the
 * caller zeroes the destinations g holds first).  d_ws as for prep. */
int wg_pagerank_pull(const wg_graph *g, const float *d_contrib, float *d_acc, uint32_t dst_base,
                     void *d_ws, size_t ws_bytes, void *stream);

/* ---------------- input generation (graph_io.py:87-221) ------------------- */
/* RMAT edges m = edge_factor << scale from PCG64(state, inc) exactly like
 * numpy's default_rng(PCG64(seed)).random((m, scale)) (graph_io.py:188-202).
 * state/inc are 128-bit values split into hi/lo words.  thresholds = {a, a+b,
 * a+b+c} as computed in float64. */
int wg_rmat_edges(uint32_t scale, uint64_t m, uint64_t state_hi, uint64_t state_lo,
                  uint64_t inc_hi, uint64_t inc_lo, const double *h_thresholds3, uint32_t *d_src,
                  uint32_t *d_dst, void *stream);
/* Canonical edge list: optional self-loop removal, optional symmetrize, sort
 * by (src, dst) and de-duplicate.  In-place on d_src/d_dst (capacity
 * 2*m when symmetrizing); d_scratch from wg_canonical_scratch_bytes.
 * h_m_out (host) receives the resulting edge count.  Synchronises. */
size_t wg_canonical_scratch_bytes(uint64_t m);
int wg_canonical_edges(uint64_t m, uint32_t *d_src, uint32_t *d_dst, int drop_loops,
                       int symmetrize, void *d_scratch, size_t scratch_bytes, uint64_t *h_m_out,
                       void *stream);
/* weight = 1 + ((((s*K) ^ d) * K) >> 48) % max_weight  (graph_io.py:215-220). */
int wg_weights_hash(uint64_t m, const uint32_t *d_src, const uint32_t *d_dst, uint32_t max_weight,
                    uint32_t *d_w, void *stream);
/* 4-neighbour rows x cols grid, each undirected edge kept with probability
 * keep_per_million/1e6 and weight uniform in [1, max_weight], both directions
 * with the same weight; counter-based hash stream keyed by seed.  Outputs up
 * to 4*rows*cols directed edges; h_m_out receives the count.  Synchronises. */
int wg_grid_edges(uint32_t rows, uint32_t cols, uint64_t seed, uint32_t keep_per_million,
                  uint32_t max_weight, uint32_t *d_src, uint32_t *d_dst, uint32_t *d_w,
                  uint64_t *d_counter, uint64_t *h_m_out, void *stream);

/* voff[d] = first vector of destination d (lower bound of d in the sorted
 * vdst), voff[n] = nvec: the per-destination form of PullTopology.vec_dst
 * (graph.py:240-243).  d_voff: [n+1]. */
int wg_vector_offsets_from_dst(const wg_graph *g, uint32_t *d_voff, void *stream);
/* vfirst[d] = vsrc[voff[d] * width] (WG_NO_LANE when d has no vectors); needs d_voff. */
int wg_first_lanes(const wg_graph *g, const uint32_t *d_voff, uint32_t *d_vfirst, void *stream);

/* ---------------------------------------------------------------------- */
/* Ingest of the plugin call's reference-layout host arrays (ingest.cu).   */
/* The backend copies the caller's int64 arrays to the device raw, chunk by */
/* chunk, and narrows/validates each chunk here (B200Backend, backend.py):  */
/*   PullTopology vec_dst / lane_count / lane_src / lane_weight  graph.py:109-164 */
/*   EdgeIndex offsets / positions                            graph.py:190-212 */
/*   out-degrees (compute_out_degrees)                        graph.py:277-280 */
/*   initial values (ValueBuffers.initialize)                 engine.py:90-116 */
/* Violations OR bits into *d_err (read once by the caller).                */
/* ---------------------------------------------------------------------- */
#define WG_INGEST_BAD_DST 1u      /* vec_dst outside [0, n) */
#define WG_INGEST_BAD_SRC 2u      /* a valid lane's source outside [0, n) */
#define WG_INGEST_BAD_COUNT 4u    /* lane_count outside [0, width] */
#define WG_INGEST_BAD_WEIGHT 8u   /* a valid lane's weight outside [0, 2^32) */
#define WG_INGEST_BAD_POS 16u     /* an index position outside [0, nvec) */
#define WG_INGEST_BAD_DEGREE 32u  /* an out-degree outside [0, 2^32) */
#define WG_INGEST_BAD_OFFSETS 64u /* offsets not monotone / not [0 .. entries] */
#define WG_INGEST_LENS_DIFFER 128u /* some index length differs from the out-degree (informational) */

/* count vectors: vdst[p] = vec_dst[p], vsrc[p*W+k] = lane_src[p*W+k] for k <
 * lane_count[p] else WG_NO_LANE, vw likewise (0 in padding); pointers are the
 * chunk's (already offset) device arrays. */
int wg_ingest_vectors(uint64_t count, uint32_t width, uint32_t n, const int64_t *d_vec_dst,
                      const int64_t *d_lane_count, const int64_t *d_lane_src, const int64_t *d_lane_w,
                      uint32_t *d_vdst, uint32_t *d_vsrc, uint32_t *d_vw, uint32_t *d_err, void *stream);
/* out[i] = in[i] as uint32; `flag` set in *d_err when in[i] is outside [0, limit). */
int wg_ingest_u32(uint64_t count, const int64_t *d_in, int64_t limit, uint32_t *d_out, uint32_t flag,
                  uint32_t *d_err, void *stream);
/* validate the CSR offsets (0 .. entries, monotone); WG_INGEST_LENS_DIFFER
 * when d_outdeg is given and some offsets[v+1]-offsets[v] != outdeg[v]. */
int wg_ingest_offsets(uint32_t n, const uint64_t *d_idx_off, uint64_t entries, const uint32_t *d_outdeg,
                      uint32_t *d_err, void *stream);

#define WG_VALUES_NOT_U32 1u      /* some finite value outside [0, 0xFFFFFFFF) */
#define WG_VALUES_NOT_IDENTITY 2u /* init[v] != v for some v */
/* d_enc[v] = uint32 encoding (sentinel -> 0xFFFFFFFF); d_stats4 = {flags,
 * finite count, min finite, max finite (int64 bits)}. */
int wg_values_scan(uint32_t n, const int64_t *d_init, int64_t sentinel, uint32_t *d_enc, uint64_t *d_stats4,
                   void *stream);

#ifdef __cplusplus
}
#endif
#endif /* WEDGE_B200_H */
