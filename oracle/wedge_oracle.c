/*
 * wedge_oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot path (wedgegraph 0.1.0,
 * /root/reference/pkg/src/wedgegraph), used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg as the checker and the CPU timing arm.  Nothing in the product package
 * (paper_1903_07754_b200/) links or calls this file.
 *
 * Semantics follow the reference exactly: int64 vertex values with a
 * caller-supplied sentinel (engine.py:41-43), strict min-plus update
 * `cand = agg + inc; update iff cand < prev[d]` (_kernels.pyx:91-94),
 * uint64 little-endian bitmaps (bitmask.py:15-32), destination-grouped
 * W-lane vectors ordered by (dst, src) (graph.py:220-263) and a per-source
 * CSR of ascending, de-duplicated vector positions (graph.py:283-301).
 *
 * Parity of this restatement is pinned by tests/test_oracle.py against the
 * golden vectors in tests/golden/ (generated from the reference itself by
 * tests/golden/make_golden.py) and, when /root/reference is present,
 * against the reference's compiled kernels built into oracle/_ref/.
 *
 * Threading: the pulls split vectors into destination-aligned ranges like
 * kernels.py:39-52 (so value writes are disjoint) and the transform splits
 * the frontier into fixed vertex slices like kernels.py:116-125; shared
 * bitmap words are set with an atomic OR, so results do not depend on the
 * thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline void or_bit(uint64_t *words, int64_t i) {
    __atomic_fetch_or(&words[i >> 6], (uint64_t)1 << (i & 63), __ATOMIC_RELAXED);
}

static inline int test_bit(const uint64_t *words, int64_t i) {
    return (int)((words[i >> 6] >> (i & 63)) & 1u);
}

/* ------------------------------------------------------------------------ */
/* Frontier transform (frontier.py:174-209; _kernels.pyx:35-52;             */
/* _kernels_py.py:96-114): for every frontier member v and every index      */
/* entry j of v, set wedge bit positions[j] >> shift.  Returns the number   */
/* of index entries visited (sum of the members' list lengths).             */
/* ------------------------------------------------------------------------ */
int64_t orc_transform(const uint64_t *fwords, int64_t vertex_count,
                      const int64_t *offsets, const int64_t *positions,
                      int shift, uint64_t *wwords, int64_t slice, int threads)
{
    if (slice < 1) slice = 4096;
    int64_t nslices = (vertex_count + slice - 1) / slice;
    int64_t total = 0;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
    #pragma omp parallel for schedule(dynamic, 1) reduction(+:total) num_threads(threads)
#endif
    for (int64_t s = 0; s < nslices; ++s) {
        int64_t lo = s * slice;
        int64_t hi = lo + slice < vertex_count ? lo + slice : vertex_count;
        for (int64_t v = lo; v < hi; ++v) {
            if (!test_bit(fwords, v)) continue;
            int64_t a = offsets[v], b = offsets[v + 1];
            for (int64_t j = a; j < b; ++j) or_bit(wwords, positions[j] >> shift);
            total += b - a;
        }
    }
    return total;
}

/* ------------------------------------------------------------------------ */
/* Min-plus pulls (engine.py:251-327; _kernels.pyx:65-95, 113-173).         */
/* lane_src / lane_wgt are row-major [nvec, W] int64; lane_wgt may be NULL  */
/* when use_weight is 0.                                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
    const int64_t *vec_dst, *lane_src, *lane_wgt, *lane_count;
    int64_t width;
    const int64_t *prev;
    int64_t *nxt;
    uint64_t *out_words;
    int filter_unvisited, use_weight;
    int64_t inc, sentinel;
} pull_args;

/* Fold vector p's valid lanes into agg. */
static inline int64_t fold_vector(const pull_args *a, int64_t p, int64_t agg) {
    const int64_t *src = a->lane_src + p * a->width;
    const int64_t *wgt = a->use_weight ? a->lane_wgt + p * a->width : NULL;
    int64_t cnt = a->lane_count[p];
    for (int64_t k = 0; k < cnt; ++k) {
        int64_t msg = a->prev[src[k]] + (wgt ? wgt[k] : 0);
        if (msg < agg) agg = msg;
    }
    return agg;
}

static inline void apply_dst(const pull_args *a, int64_t d, int64_t agg) {
    int64_t cand = agg + a->inc;
    if (cand < a->prev[d]) {
        a->nxt[d] = cand;
        or_bit(a->out_words, d);
    }
}

static int64_t pull_full_span(const pull_args *a, int64_t lo, int64_t hi) {
    int64_t touched = 0, p = lo;
    while (p < hi) {
        int64_t d = a->vec_dst[p];
        int64_t end = p;
        while (end < hi && a->vec_dst[end] == d) ++end;
        if (!(a->filter_unvisited && a->prev[d] != a->sentinel)) {
            int64_t agg = a->sentinel;
            for (int64_t q = p; q < end; ++q) agg = fold_vector(a, q, agg);
            touched += end - p;
            apply_dst(a, d, agg);
        }
        p = end;
    }
    return touched;
}

/* Covered positions are walked ascending; one aggregate per destination run
 * of the covered subsequence, even across uncovered gaps. */
static int64_t pull_wedge_span(const pull_args *a, const uint64_t *wwords, int shift,
                               int64_t lo, int64_t hi) {
    int64_t touched = 0;
    int64_t cur = -1, agg = 0;
    int skip = 0;
    int64_t g0 = lo >> shift, g1 = (hi - 1) >> shift;
    for (int64_t g = g0; g <= g1; ++g) {
        if (!test_bit(wwords, g)) continue;
        int64_t s = g << shift, e = (g + 1) << shift;
        if (s < lo) s = lo;
        if (e > hi) e = hi;
        for (int64_t p = s; p < e; ++p) {
            int64_t d = a->vec_dst[p];
            if (d != cur) {
                if (cur >= 0 && !skip) apply_dst(a, cur, agg);
                cur = d;
                agg = a->sentinel;
                skip = a->filter_unvisited && a->prev[d] != a->sentinel;
            }
            if (skip) continue;
            agg = fold_vector(a, p, agg);
            ++touched;
        }
    }
    if (cur >= 0 && !skip) apply_dst(a, cur, agg);
    return touched;
}

/* Destination-aligned split of [0, nvec) into up to `parts` ranges
 * (kernels.py:39-52).  bounds must hold parts+1 entries; returns #ranges. */
static int64_t dst_ranges(const int64_t *vec_dst, int64_t nvec, int64_t parts, int64_t *bounds) {
    if (nvec == 0) return 0;
    int64_t nb = 0;
    bounds[nb++] = 0;
    for (int64_t k = 1; k < parts; ++k) {
        int64_t b = (k * nvec) / parts;
        while (b > 0 && b < nvec && vec_dst[b] == vec_dst[b - 1]) ++b;
        if (b > bounds[nb - 1] && b < nvec) bounds[nb++] = b;
    }
    bounds[nb++] = nvec;
    return nb - 1;
}

static int64_t run_pull(const pull_args *a, int64_t nvec, const uint64_t *wwords, int shift,
                        int threads) {
    if (nvec == 0) return 0;
    if (threads < 1) threads = 1;
    int64_t parts = threads > 1 ? (int64_t)threads * 4 : 1;
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(parts + 1));
    int64_t nr = dst_ranges(a->vec_dst, nvec, parts, bounds);
    int64_t touched = 0;
#ifdef _OPENMP
    #pragma omp parallel for schedule(dynamic, 1) reduction(+:touched) num_threads(threads)
#endif
    for (int64_t r = 0; r < nr; ++r) {
        touched += wwords ? pull_wedge_span(a, wwords, shift, bounds[r], bounds[r + 1])
                          : pull_full_span(a, bounds[r], bounds[r + 1]);
    }
    free(bounds);
    return touched;
}

int64_t orc_pull_full(int64_t nvec, int64_t width, const int64_t *vec_dst, const int64_t *lane_src,
                      const int64_t *lane_wgt, const int64_t *lane_count,
                      const int64_t *prev, int64_t *nxt, uint64_t *out_words,
                      int filter_unvisited, int use_weight, int64_t inc, int64_t sentinel,
                      int threads)
{
    pull_args a = {vec_dst, lane_src, lane_wgt, lane_count, width, prev, nxt, out_words,
                   filter_unvisited, use_weight, inc, sentinel};
    return run_pull(&a, nvec, NULL, 0, threads);
}

int64_t orc_pull_wedge(int64_t nvec, int64_t width, const int64_t *vec_dst, const int64_t *lane_src,
                       const int64_t *lane_wgt, const int64_t *lane_count,
                       const uint64_t *wedge_words, int shift,
                       const int64_t *prev, int64_t *nxt, uint64_t *out_words,
                       int filter_unvisited, int use_weight, int64_t inc, int64_t sentinel,
                       int threads)
{
    pull_args a = {vec_dst, lane_src, lane_wgt, lane_count, width, prev, nxt, out_words,
                   filter_unvisited, use_weight, inc, sentinel};
    return run_pull(&a, nvec, wedge_words, shift, threads);
}

/* ------------------------------------------------------------------------ */
/* Layout construction (graph.py:220-263, 277-301) by two stable counting   */
/* sorts: by src, then by dst, giving (dst, src) order with duplicates in   */
/* input order, as np.lexsort((src, dst)) does.                             */
/* ------------------------------------------------------------------------ */
static void counting_order(int64_t n, int64_t m, const int64_t *key, const int64_t *in_order,
                           int64_t *out_order) {
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t e = 0; e < m; ++e) cnt[key[e] + 1]++;
    for (int64_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
    for (int64_t i = 0; i < m; ++i) {
        int64_t e = in_order ? in_order[i] : i;
        out_order[cnt[key[e]]++] = e;
    }
    free(cnt);
}

/* Number of vectors: sum over destinations of ceil(indeg / W). */
int64_t orc_vector_count(int64_t n, int64_t m, const int64_t *dst, int64_t width) {
    int64_t *indeg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t e = 0; e < m; ++e) indeg[dst[e]]++;
    int64_t nvec = 0;
    for (int64_t v = 0; v < n; ++v) nvec += (indeg[v] + width - 1) / width;
    free(indeg);
    return nvec;
}

/* Fill vec_dst[nvec], lane_src/lane_wgt[nvec*W] (zero padded like the
 * reference), lane_count[nvec]. */
void orc_build_pull(int64_t n, int64_t m, const int64_t *src, const int64_t *dst, const int64_t *wgt,
                    int64_t width, int64_t *vec_dst, int64_t *lane_src, int64_t *lane_wgt,
                    int64_t *lane_count)
{
    int64_t *by_src = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    counting_order(n, m, src, NULL, by_src);
    counting_order(n, m, dst, by_src, order);
    free(by_src);
    int64_t p = -1, prev_d = -1, rank = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t e = order[i];
        int64_t d = dst[e];
        if (d != prev_d) { rank = 0; prev_d = d; }
        int64_t lane = rank % width;
        if (lane == 0) {
            ++p;
            vec_dst[p] = d;
            lane_count[p] = 0;
            for (int64_t k = 0; k < width; ++k) {
                lane_src[p * width + k] = 0;
                if (lane_wgt) lane_wgt[p * width + k] = 0;
            }
        }
        lane_src[p * width + lane] = src[e];
        if (lane_wgt) lane_wgt[p * width + lane] = wgt[e];
        lane_count[p]++;
        ++rank;
    }
    free(order);
}

void orc_out_degrees(int64_t n, int64_t m, const int64_t *src, int64_t *deg) {
    memset(deg, 0, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < m; ++e) deg[src[e]]++;
}

/* Edge index: offsets[n+1] and positions[] (capacity = number of valid
 * lanes); returns the number of entries written. */
int64_t orc_build_index(int64_t n, int64_t nvec, int64_t width, const int64_t *lane_src,
                        const int64_t *lane_count, int64_t *offsets, int64_t *positions)
{
    int64_t lanes = 0;
    for (int64_t p = 0; p < nvec; ++p) lanes += lane_count[p];
    int64_t *cursor = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *last = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t v = 0; v < n; ++v) last[v] = -1;
    /* pass 1: distinct (src, pos) pairs per source; positions arrive
     * ascending so a duplicate is always the previous entry. */
    for (int64_t p = 0; p < nvec; ++p)
        for (int64_t k = 0; k < lane_count[p]; ++k) {
            int64_t s = lane_src[p * width + k];
            if (last[s] != p) { last[s] = p; cursor[s + 1]++; }
        }
    for (int64_t v = 0; v < n; ++v) cursor[v + 1] += cursor[v];
    memcpy(offsets, cursor, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t v = 0; v < n; ++v) last[v] = -1;
    for (int64_t p = 0; p < nvec; ++p)
        for (int64_t k = 0; k < lane_count[p]; ++k) {
            int64_t s = lane_src[p * width + k];
            if (last[s] != p) { last[s] = p; positions[cursor[s]++] = p; }
        }
    free(cursor);
    free(last);
    (void)lanes;
    return offsets[n];
}

/* ------------------------------------------------------------------------ */
/* PageRank (no reference implementation exists: SPEC.md:403).  BASELINE   */
/* config 5 semantics, float64: r0 = 1/N;                                   */
/* r'(v) = (1-d)/N + d * (sum_{u->v} r(u)/outdeg(u) + D/N),                 */
/* D = sum of r(u) over outdeg(u) == 0.                                     */
/* ------------------------------------------------------------------------ */
void orc_pagerank(int64_t n, int64_t nvec, int64_t width, const int64_t *vec_dst,
                  const int64_t *lane_src, const int64_t *lane_count, const int64_t *outdeg,
                  int iterations, double damping, double *rank, int threads)
{
    double *contrib = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double *acc = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t v = 0; v < n; ++v) rank[v] = 1.0 / (double)n;
    if (threads < 1) threads = 1;
    for (int it = 0; it < iterations; ++it) {
        double dangling = 0.0;
        for (int64_t v = 0; v < n; ++v) {
            if (outdeg[v] > 0) contrib[v] = rank[v] / (double)outdeg[v];
            else { contrib[v] = 0.0; dangling += rank[v]; }
            acc[v] = 0.0;
        }
#ifdef _OPENMP
        #pragma omp parallel for schedule(static) num_threads(threads)
#endif
        for (int64_t p = 0; p < nvec; ++p) {
            double s = 0.0;
            for (int64_t k = 0; k < lane_count[p]; ++k) s += contrib[lane_src[p * width + k]];
#ifdef _OPENMP
            #pragma omp atomic
#endif
            acc[vec_dst[p]] += s;
        }
        double base = (1.0 - damping) / (double)n + damping * dangling / (double)n;
        for (int64_t v = 0; v < n; ++v) rank[v] = base + damping * acc[v];
    }
    free(contrib);
    free(acc);
}

/* ------------------------------------------------------------------------ */
/* Input preparation for the CPU arms (graph_io.py:87-112, 188-202),        */
/* multi-threaded so the --impl reference leg prepares a 128M-edge input in */
/* seconds instead of the reference generators' minutes.  Same outputs as  */
/* the numpy restatements in oracle/__init__.py (tests/test_oracle.py).     */
/* ------------------------------------------------------------------------ */
typedef unsigned __int128 u128_t;

/* numpy PCG64: 128-bit LCG, XSL-RR output taken after the step; random()
 * = (next >> 11) * 2^-53 */
static inline uint64_t pcg_xslrr(u128_t st) {
    uint64_t x = (uint64_t)(st >> 64) ^ (uint64_t)st;
    unsigned rot = (unsigned)(st >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static u128_t pcg_jump(u128_t state, u128_t inc, u128_t mult, uint64_t delta) {
    u128_t am = 1, ap = 0, cm = mult, cp = inc;
    while (delta) {
        if (delta & 1u) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    return am * state + ap;
}

/* R-MAT rows [0, m): row r uses draws r*scale .. r*scale+scale-1 of the
 * stream; quadrant q = [u>=t0]+[u>=t1]+[u>=t2], src bit q>>1, dst bit q&1,
 * most significant level first (graph_io.py:195-201). */
void orc_rmat(int scale, int64_t m, uint64_t shi, uint64_t slo, uint64_t ihi, uint64_t ilo,
              const double *th, int64_t *src, int64_t *dst) {
    const u128_t mult = ((u128_t)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    const u128_t st0 = ((u128_t)shi << 64) | slo, inc = ((u128_t)ihi << 64) | ilo;
    const int64_t chunk = 1 << 16;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t lo = 0; lo < m; lo += chunk) {
        int64_t hi = lo + chunk < m ? lo + chunk : m;
        u128_t st = pcg_jump(st0, inc, mult, (uint64_t)lo * (uint64_t)scale);
        for (int64_t r = lo; r < hi; ++r) {
            int64_t s = 0, d = 0;
            for (int l = 0; l < scale; ++l) {
                st = st * mult + inc;
                double u = (double)(pcg_xslrr(st) >> 11) * (1.0 / 9007199254740992.0);
                int q = (u >= th[0]) + (u >= th[1]) + (u >= th[2]);
                int sh = scale - 1 - l;
                s |= (int64_t)(q >> 1) << sh;
                d |= (int64_t)(q & 1) << sh;
            }
            src[r] = s;
            dst[r] = d;
        }
    }
}

/* Sort 64-bit keys ascending (LSD radix, 8-bit digits, threaded) and drop
 * duplicates; `bits` = significant key bits.  Returns the unique count. */
int64_t orc_sort_unique_u64(uint64_t *keys, int64_t m, int bits) {
    if (m <= 0) return 0;
    uint64_t *tmp = (uint64_t *)malloc((size_t)m * sizeof(uint64_t));
    uint64_t *a = keys, *b = tmp;
    int T = 1;
#ifdef _OPENMP
    T = omp_get_max_threads();
#endif
    int64_t *hist = (int64_t *)calloc((size_t)T * 256, sizeof(int64_t));
    for (int shift = 0; shift < bits; shift += 8) {
        memset(hist, 0, (size_t)T * 256 * sizeof(int64_t));
        #pragma omp parallel num_threads(T)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            int64_t lo = m * t / T, hi = m * (t + 1) / T;
            int64_t *h = hist + (size_t)t * 256;
            for (int64_t i = lo; i < hi; ++i) h[(a[i] >> shift) & 255]++;
            #pragma omp barrier
            #pragma omp single
            {
                int64_t run = 0;
                for (int dgt = 0; dgt < 256; ++dgt)
                    for (int u = 0; u < T; ++u) {
                        int64_t c = hist[(size_t)u * 256 + dgt];
                        hist[(size_t)u * 256 + dgt] = run;
                        run += c;
                    }
            }
            for (int64_t i = lo; i < hi; ++i) b[h[(a[i] >> shift) & 255]++] = a[i];
        }
        uint64_t *x = a; a = b; b = x;
    }
    int64_t k = 0;
    for (int64_t i = 0; i < m; ++i)
        if (i == 0 || a[i] != a[i - 1]) keys[k++] = a[i];
    free(hist);
    free(tmp);
    return k;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
