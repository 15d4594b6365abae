"""CPU oracle for the Wedge-Frontier pull path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the CPU timing arm.  The product package ``paper_1903_07754_b200`` never
imports it (tests/test_boundary.py asserts that).

Contents
--------
* ``liboracle.so`` (``wedge_oracle.c``): a plain-C restatement of the
  reference's native kernels and layout builders, int64 values with the
  reference's sentinel semantics.
* ``_ref/_kernels*.so``: the reference's OWN Cython kernels
  (pkg/src/wedgegraph/_kernels.pyx), compiled by ``oracle/Makefile`` from the
  sources under /root/reference when present (build output only, git-ignored,
  travels to the GPU box with the snapshot).
* A numpy restatement of the reference driver ``run_until_convergence``
  (engine.py:330-388) that can run on either kernel set.
* The reference generators restated (graph_io.py:87-221) to produce seeded
  CPU-side inputs.
* A float64 PageRank oracle (no reference implementation exists).

Parity pin: tests/test_oracle.py checks every function here against the
golden vectors under tests/golden/, which tests/golden/make_golden.py produced
by importing the reference package itself.
"""

from __future__ import annotations

import ctypes
import importlib.util
import os
import subprocess
from dataclasses import dataclass, field
from fractions import Fraction
from pathlib import Path
from time import perf_counter
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
UNREACHED = 1 << 62  # engine.py:43
MODE_FULL, MODE_WEDGE = "FullScan", "Wedge"  # engine.py:45-46

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f64p = ctypes.POINTER(ctypes.c_double)
_LIB = None
_REF = None


def build() -> None:
    """Run oracle/Makefile (liboracle.so, and oracle/_ref when the reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = HERE / "liboracle.so"
        if not path.exists():
            build()
        L = ctypes.CDLL(str(path))
        L.orc_transform.restype = ctypes.c_int64
        L.orc_transform.argtypes = [_u64p, ctypes.c_int64, _i64p, _i64p, ctypes.c_int, _u64p,
                                    ctypes.c_int64, ctypes.c_int]
        pull = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, _i64p, _i64p]
        tail = [_i64p, _i64p, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                ctypes.c_int]
        L.orc_pull_full.restype = ctypes.c_int64
        L.orc_pull_full.argtypes = pull + tail
        L.orc_pull_wedge.restype = ctypes.c_int64
        L.orc_pull_wedge.argtypes = pull + [_u64p, ctypes.c_int] + tail
        L.orc_vector_count.restype = ctypes.c_int64
        L.orc_vector_count.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int64]
        L.orc_build_pull.restype = None
        L.orc_build_pull.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, _i64p,
                                     ctypes.c_int64, _i64p, _i64p, _i64p, _i64p]
        L.orc_out_degrees.restype = None
        L.orc_out_degrees.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p]
        L.orc_build_index.restype = ctypes.c_int64
        L.orc_build_index.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, _i64p,
                                      _i64p, _i64p]
        L.orc_pagerank.restype = None
        L.orc_pagerank.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, _i64p,
                                   _i64p, _i64p, ctypes.c_int, ctypes.c_double, _f64p, ctypes.c_int]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_rmat.restype = None
        L.orc_rmat.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_uint64, ctypes.c_uint64, _f64p, _i64p, _i64p]
        L.orc_sort_unique_u64.restype = ctypes.c_int64
        L.orc_sort_unique_u64.argtypes = [_u64p, ctypes.c_int64, ctypes.c_int]
        _LIB = L
    return _LIB


def ref_kernels():
    """The reference's compiled kernels from oracle/_ref, or None if not built."""
    global _REF
    if _REF is None:
        cands = sorted((HERE / "_ref").glob("_kernels*.so"))
        if not cands:
            return None
        spec = importlib.util.spec_from_file_location("_kernels", cands[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _p(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------------
# Reference-layout structures (graph.py:109-212), int64 like the reference.
# --------------------------------------------------------------------------
@dataclass
class RefTopology:
    """Duck-type of the reference ``PullTopology`` (graph.py:109-164)."""

    vertex_count: int
    vector_width: int
    edge_count: int
    vec_dst: np.ndarray
    lane_src: np.ndarray
    lane_weight: Optional[np.ndarray]
    lane_count: np.ndarray

    @property
    def vector_count(self) -> int:
        return int(self.vec_dst.shape[0])

    def is_weighted(self) -> bool:
        return self.lane_weight is not None

    def lane_valid(self) -> np.ndarray:
        return self.lane_count[:, None] > np.arange(self.vector_width)[None, :]


@dataclass
class RefIndex:
    """Duck-type of the reference ``EdgeIndex`` (graph.py:190-212)."""

    vertex_count: int
    vector_count: int
    offsets: np.ndarray
    positions: np.ndarray


def build_pull_topology(n: int, src, dst, weight=None, width: int = 4) -> RefTopology:
    """Restates build_pull_topology (graph.py:220-263)."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    wgt = None if weight is None else np.ascontiguousarray(weight, dtype=np.int64)
    m = int(src.shape[0])
    L = lib()
    nvec = int(L.orc_vector_count(n, m, _p(dst, _i64p), width))
    vec_dst = np.empty(nvec, np.int64)
    lane_src = np.empty((nvec, width), np.int64)
    lane_w = np.empty((nvec, width), np.int64) if wgt is not None else None
    lane_count = np.empty(nvec, np.int64)
    L.orc_build_pull(n, m, _p(src, _i64p), _p(dst, _i64p), _p(wgt, _i64p), width,
                     _p(vec_dst, _i64p), _p(lane_src, _i64p), _p(lane_w, _i64p), _p(lane_count, _i64p))
    return RefTopology(n, width, m, vec_dst, lane_src, lane_w, lane_count)


def build_edge_index(topo: RefTopology) -> RefIndex:
    """Restates build_edge_index (graph.py:283-301)."""
    n, nvec = topo.vertex_count, topo.vector_count
    offsets = np.empty(n + 1, np.int64)
    positions = np.empty(int(topo.lane_count.sum()), np.int64)
    ls = np.ascontiguousarray(topo.lane_src)
    k = lib().orc_build_index(n, nvec, topo.vector_width, _p(ls, _i64p), _p(topo.lane_count, _i64p),
                              _p(offsets, _i64p), _p(positions, _i64p))
    return RefIndex(n, nvec, offsets, positions[:k].copy())


def compute_out_degrees(n: int, src) -> np.ndarray:
    """Restates compute_out_degrees (graph.py:277-280)."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    deg = np.empty(n, np.int64)
    lib().orc_out_degrees(n, int(src.shape[0]), _p(src, _i64p), _p(deg, _i64p))
    return deg


# --------------------------------------------------------------------------
# Kernel protocol (kernels.py:55-125): identical signatures to the
# reference backends, so the oracle can stand in for them in tests.
# --------------------------------------------------------------------------
class PortBackend:
    """The C restatement behind the reference backend protocol."""

    name = "oracle-port"

    def __init__(self, threads: int = 1):
        self.threads = threads

    def _lanes(self, topo):
        ls = np.ascontiguousarray(topo.lane_src, dtype=np.int64)
        lw = topo.lane_weight
        lw = np.ascontiguousarray(lw, dtype=np.int64) if lw is not None else None
        return ls, lw

    def pull_full(self, topology, prev, nxt, out_words, kern, sentinel, workers=1):
        ls, lw = self._lanes(topology)
        if kern.use_weight and lw is None:
            raise ValueError("weights required")
        return int(lib().orc_pull_full(
            topology.vector_count, topology.vector_width, _p(topology.vec_dst, _i64p), _p(ls, _i64p),
            _p(lw, _i64p), _p(topology.lane_count, _i64p), _p(prev, _i64p), _p(nxt, _i64p),
            _p(out_words, _u64p), int(kern.filter_unvisited), int(kern.use_weight),
            int(kern.apply_increment), int(sentinel), max(self.threads, 1)))

    def pull_wedge(self, topology, wedge_words, shift, group_count, prev, nxt, out_words, kern,
                   sentinel, workers=1):
        ls, lw = self._lanes(topology)
        if kern.use_weight and lw is None:
            raise ValueError("weights required")
        ww = np.ascontiguousarray(wedge_words, dtype=np.uint64)
        return int(lib().orc_pull_wedge(
            topology.vector_count, topology.vector_width, _p(topology.vec_dst, _i64p), _p(ls, _i64p),
            _p(lw, _i64p), _p(topology.lane_count, _i64p), _p(ww, _u64p), int(shift),
            _p(prev, _i64p), _p(nxt, _i64p), _p(out_words, _u64p), int(kern.filter_unvisited),
            int(kern.use_weight), int(kern.apply_increment), int(sentinel), max(self.threads, 1)))

    def transform(self, frontier_words, vertex_count, offsets, positions, shift, wedge_words,
                  slice_size=4096, workers=1):
        fw = np.ascontiguousarray(frontier_words, dtype=np.uint64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        pos = np.ascontiguousarray(positions, dtype=np.int64)
        return int(lib().orc_transform(_p(fw, _u64p), int(vertex_count), _p(off, _i64p),
                                       _p(pos, _i64p), int(shift), _p(wedge_words, _u64p),
                                       int(slice_size), max(self.threads, 1)))


class RefBackend:
    """The reference's own compiled kernels (oracle/_ref) driven exactly as
    NativeBackend drives them (kernels.py:72-125), including its
    destination-aligned ranges and a thread pool per call."""

    name = "reference-native"

    def __init__(self, threads: int = 1):
        mod = ref_kernels()
        if mod is None:
            raise RuntimeError("oracle/_ref not built (reference sources absent)")
        self.mod = mod
        self.threads = threads

    @staticmethod
    def _ranges(vec_dst, parts):
        nvec = len(vec_dst)
        if nvec == 0:
            return []
        bounds = [0]
        for k in range(1, parts):
            b = (k * nvec) // parts
            while 0 < b < nvec and vec_dst[b] == vec_dst[b - 1]:
                b += 1
            if b > bounds[-1] and b < nvec:
                bounds.append(b)
        bounds.append(nvec)
        return list(zip(bounds[:-1], bounds[1:]))

    def _run(self, tasks):
        if self.threads <= 1 or len(tasks) <= 1:
            return sum(t() for t in tasks)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=self.threads) as pool:
            return sum(pool.map(lambda t: t(), tasks))

    def pull_full(self, topology, prev, nxt, out_words, kern, sentinel, workers=1):
        ls = topology.lane_src
        lw = topology.lane_weight if topology.lane_weight is not None else ls
        parts = self.threads * 4 if self.threads > 1 else 1
        m = self.mod
        tasks = [(lambda lo=lo, hi=hi: m.pull_full_range(
            topology.vec_dst, ls, lw, topology.lane_count, prev, nxt, out_words,
            kern.filter_unvisited, kern.use_weight, kern.apply_increment, sentinel, lo, hi))
            for lo, hi in self._ranges(topology.vec_dst, parts)]
        return self._run(tasks)

    def pull_wedge(self, topology, wedge_words, shift, group_count, prev, nxt, out_words, kern,
                   sentinel, workers=1):
        if topology.vector_count == 0:
            return 0
        ls = topology.lane_src
        lw = topology.lane_weight if topology.lane_weight is not None else ls
        parts = self.threads * 4 if self.threads > 1 else 1
        m = self.mod
        tasks = [(lambda lo=lo, hi=hi: m.pull_wedge_range(
            topology.vec_dst, ls, lw, topology.lane_count, wedge_words, shift, prev, nxt, out_words,
            kern.filter_unvisited, kern.use_weight, kern.apply_increment, sentinel, lo, hi))
            for lo, hi in self._ranges(topology.vec_dst, parts) if hi > lo]
        return self._run(tasks)

    def transform(self, frontier_words, vertex_count, offsets, positions, shift, wedge_words,
                  slice_size=4096, workers=1):
        m = self.mod
        tasks = [(lambda lo=lo: m.transform_range(frontier_words, lo, min(lo + slice_size, vertex_count),
                                                  offsets, positions, shift, wedge_words))
                 for lo in range(0, vertex_count, slice_size)]
        return self._run(tasks)


# --------------------------------------------------------------------------
# Bitmask helpers (bitmask.py:15-32)
# --------------------------------------------------------------------------
def word_count(size: int) -> int:
    return (size + 63) >> 6


def bit_indices(words: np.ndarray, size: int) -> np.ndarray:
    if size == 0:
        return np.empty(0, np.int64)
    flat = np.unpackbits(words.view(np.uint8), bitorder="little")[:size]
    return np.nonzero(flat)[0].astype(np.int64)


def set_bits(words: np.ndarray, ids) -> None:
    ids = np.asarray(ids, dtype=np.uint64)
    if ids.size:
        np.bitwise_or.at(words, (ids >> np.uint64(6)).astype(np.int64), np.uint64(1) << (ids & np.uint64(63)))


# --------------------------------------------------------------------------
# Driver restatement (engine.py:245-388)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Kern:
    """MinPlusKernel triple (engine.py:50-63)."""

    filter_unvisited: bool
    use_weight: bool
    apply_increment: int


BFS = Kern(True, False, 1)    # apps.py:28-53
CC = Kern(False, False, 0)    # apps.py:56-73
SSSP = Kern(False, True, 0)   # apps.py:76-100


@dataclass
class Stat:
    iteration: int
    mode: str
    active_edges: int
    vectors_touched: int
    frontier_out_size: int
    covered_vectors: int = 0
    transform_entries: int = 0
    transform_time: float = 0.0
    pull_time: float = 0.0


@dataclass
class RunOut:
    values: np.ndarray
    stats: list = field(default_factory=list)
    converged: bool = False


def initial_state(app: str, n: int, root: int = 0):
    """Initial values and frontier per application (apps.py:28-100)."""
    if app == "cc":
        return np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64)
    vals = np.full(n, UNREACHED, np.int64)
    vals[root] = 0
    return vals, np.array([root], np.int64)


def kern_of(app: str) -> Kern:
    return {"bfs": BFS, "cc": CC, "sssp": SSSP}[app]


def run_until_convergence(topo, index, degrees, kern: Kern, init_values, init_frontier,
                          threshold: Fraction, vpg: int, max_iterations: int = 1_000_000,
                          backend=None, slice_size: int = 4096, frontier_log=None,
                          value_log=None) -> RunOut:
    """Restates run_until_convergence (engine.py:330-388) with int64 values."""
    backend = backend or PortBackend()
    n = topo.vertex_count
    total_edges = topo.edge_count
    shift = vpg.bit_length() - 1
    nvec = topo.vector_count
    groups = (nvec + vpg - 1) // vpg
    prev = np.ascontiguousarray(init_values, dtype=np.int64).copy()
    nxt = prev.copy()
    members = np.unique(np.asarray(init_frontier, dtype=np.int64))
    fwords = np.zeros(word_count(n), np.uint64)
    set_bits(fwords, members)
    edge_sum = int(degrees[members].sum()) if members.size else 0
    stats: list[Stat] = []
    converged = False
    num, den = threshold.numerator, threshold.denominator
    while not converged and len(stats) < max_iterations:
        in_edges = edge_sum
        np.copyto(nxt, prev)
        out = np.zeros(word_count(n), np.uint64)
        if total_edges > 0 and edge_sum * den < num * total_edges:
            t0 = perf_counter()
            wwords = np.zeros(word_count(groups), np.uint64)
            entries = backend.transform(fwords, n, index.offsets, index.positions, shift, wwords,
                                        slice_size, 1)
            t1 = perf_counter()
            touched = backend.pull_wedge(topo, wwords, shift, groups, prev, nxt, out, kern,
                                         UNREACHED, 1)
            t2 = perf_counter()
            setc = int(np.bitwise_count(wwords).sum())
            covered = setc * vpg
            over = groups * vpg - nvec
            if over and groups and (wwords[(groups - 1) >> 6] >> np.uint64((groups - 1) & 63)) & np.uint64(1):
                covered -= over
            st = Stat(0, MODE_WEDGE, 0, int(touched), 0, covered, int(entries), t1 - t0, t2 - t1)
        else:
            t1 = perf_counter()
            touched = backend.pull_full(topo, prev, nxt, out, kern, UNREACHED, 1)
            st = Stat(0, MODE_FULL, 0, int(touched), 0, pull_time=perf_counter() - t1)
        members = bit_indices(out, n)
        edge_sum = int(degrees[members].sum()) if members.size else 0
        st.iteration = len(stats) + 1
        st.active_edges = in_edges
        st.frontier_out_size = int(members.size)
        prev, nxt = nxt, prev
        fwords = out
        stats.append(st)
        if frontier_log is not None:
            frontier_log.append(members)
        if value_log is not None:
            value_log.append(prev.copy())
        converged = edge_sum == 0
    return RunOut(prev, stats, converged)


def result_digest(values) -> str:
    """blake2b-64 over int64 LE values (engine.py:173-176)."""
    import hashlib
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.int64), dtype="<i8")
    return hashlib.blake2b(arr.tobytes(), digest_size=8).hexdigest()


def signature(stats) -> tuple:
    """(iteration, mode, active_edges, work, frontier_out) rows (engine.py:179-185)."""
    return tuple((s.iteration, s.mode, s.active_edges, s.vectors_touched, s.frontier_out_size)
                 for s in stats)


def trace(stats) -> tuple:
    """Layout-independent per-iteration trace."""
    return tuple((s.iteration, s.mode, s.active_edges, s.frontier_out_size) for s in stats)


# --------------------------------------------------------------------------
# PageRank float64 oracle (BASELINE config 5; no reference implementation)
# --------------------------------------------------------------------------
def pagerank(topo, degrees, iterations: int = 20, damping: float = 0.85, threads: int = 1):
    n = topo.vertex_count
    rank = np.empty(n, np.float64)
    ls = np.ascontiguousarray(topo.lane_src, dtype=np.int64)
    deg = np.ascontiguousarray(degrees, dtype=np.int64)
    lib().orc_pagerank(n, topo.vector_count, topo.vector_width, _p(topo.vec_dst, _i64p),
                       _p(ls, _i64p), _p(topo.lane_count, _i64p), _p(deg, _i64p), int(iterations),
                       float(damping), _p(rank, _f64p), max(threads, 1))
    return rank


def pagerank_numpy(n, src, dst, iterations=20, damping=0.85):
    """Independent edge-list form of the same PR semantics (cross-check)."""
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    deg = np.bincount(src, minlength=n).astype(np.float64)
    r = np.full(n, 1.0 / n)
    for _ in range(iterations):
        contrib = np.where(deg > 0, r / np.maximum(deg, 1), 0.0)
        dangling = r[deg == 0].sum()
        acc = np.bincount(dst, weights=contrib[src], minlength=n)
        r = (1 - damping) / n + damping * (acc + dangling / n)
    return r


# --------------------------------------------------------------------------
# Generators restated (graph_io.py:87-221) for seeded CPU-side inputs.
# --------------------------------------------------------------------------
RMAT_PROBS = (0.57, 0.19, 0.19, 0.05)
HASH_K = 0x9E3779B97F4A7C15


def rmat_edges(scale: int, edge_factor: int, seed: int = 1, probs=RMAT_PROBS, chunk: int = 1 << 20):
    """RMAT sampler of graph_io.py:188-202, generated in row chunks (same stream)."""
    n = 1 << scale
    m = edge_factor * n
    a, b, c, _ = probs
    rng = np.random.default_rng(np.random.PCG64(seed))
    src = np.zeros(m, np.int64)
    dst = np.zeros(m, np.int64)
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        draws = rng.random((hi - lo, scale))
        q = (draws >= a).astype(np.int64) + (draws >= a + b) + (draws >= a + b + c)
        s = np.zeros(hi - lo, np.int64)
        d = np.zeros(hi - lo, np.int64)
        for level in range(scale):
            sh = scale - 1 - level
            s |= (q[:, level] >> 1) << sh
            d |= (q[:, level] & 1) << sh
        src[lo:hi], dst[lo:hi] = s, d
    return n, src, dst


def rmat_edges_fast(scale: int, edge_factor: int, seed: int = 1, probs=RMAT_PROBS):
    """rmat_edges in threaded C (orc_rmat): the same PCG64 stream jumped ahead
    per row chunk; identical output (tests/test_oracle.py)."""
    n = 1 << scale
    m = edge_factor * n
    st = np.random.PCG64(seed).state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    a, b, c, _ = probs
    th = np.array([a, a + b, a + b + c], np.float64)
    src = np.empty(m, np.int64)
    dst = np.empty(m, np.int64)
    M = (1 << 64) - 1
    lib().orc_rmat(scale, m, state >> 64, state & M, inc >> 64, inc & M, _p(th, _f64p),
                   _p(src, _i64p), _p(dst, _i64p))
    return n, src, dst


def _sorted_unique_pairs(src, dst, n):
    bits = max(1, int(n - 1).bit_length()) if n > 1 else 1
    key = (np.asarray(src, np.int64).astype(np.uint64) << np.uint64(bits)) | np.asarray(dst, np.int64).astype(np.uint64)
    k = int(lib().orc_sort_unique_u64(_p(key, _u64p), key.size, 2 * bits))
    key = key[:k]
    return (key >> np.uint64(bits)).astype(np.int64), (key & np.uint64((1 << bits) - 1)).astype(np.int64)


def prepare_unweighted(n, src, dst, symmetric: bool):
    """Drop self-loops, then symmetrize(dedup=True) (graph_io.py:87-112) or
    de-duplicate directed edges; (src, dst)-sorted like oracle.symmetrize /
    dedup_directed, computed with the threaded radix sort."""
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    keep = src != dst
    s, d = src[keep], dst[keep]
    if symmetric:
        s, d = np.concatenate([s, d]), np.concatenate([d, s])
    return _sorted_unique_pairs(s, d, n)


def symmetrize(src, dst, weight=None, dedup=False):
    """graph_io.py:87-112: add reverses (self-loops once); optional dedup (min weight)."""
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    loops = src == dst
    s = np.concatenate([src, dst[~loops]])
    d = np.concatenate([dst, src[~loops]])
    w = None if weight is None else np.concatenate([weight, np.asarray(weight)[~loops]])
    if not dedup:
        return s, d, w
    order = np.lexsort((d, s)) if w is None else np.lexsort((w, d, s))
    s, d = s[order], d[order]
    w = None if w is None else w[order]
    keep = np.ones(len(s), bool)
    keep[1:] = (s[1:] != s[:-1]) | (d[1:] != d[:-1])
    return s[keep], d[keep], (None if w is None else w[keep])


def dedup_directed(src, dst):
    """Canonical (src, dst)-sorted unique edge list."""
    key = np.asarray(src, np.int64) * (1 << 32) + np.asarray(dst, np.int64)
    key = np.unique(key)
    return key >> 32, key & 0xFFFFFFFF


def synthesize_weights(src, dst, max_weight: int):
    """graph_io.py:205-221 multiplicative hash weights in [1, max_weight]."""
    k = np.uint64(HASH_K)
    s = np.asarray(src).astype(np.uint64)
    d = np.asarray(dst).astype(np.uint64)
    with np.errstate(over="ignore"):
        h = ((s * k) ^ d) * k
    return 1 + ((h >> np.uint64(48)) % np.uint64(max_weight)).astype(np.int64)


def _mix64(seed: int, u: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of seed ^ (u * golden), as wg_grid_edges uses."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) ^ (u * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def grid_edges(rows: int, cols: int, seed: int, keep: float = 0.9, max_weight: int = 1000):
    """Restatement of the device grid generator (BASELINE config 3; the
    reference has none): undirected edge u (row-major horizontals, then
    verticals) is kept iff mix64(seed, u) % 1e6 < keep*1e6, weight
    1 + (h >> 32) % max_weight, stored in both directions."""
    H = rows * (cols - 1)
    V = (rows - 1) * cols
    u = np.arange(H + V, dtype=np.uint64)
    a = np.empty(H + V, np.int64)
    b = np.empty(H + V, np.int64)
    if H:
        uh = u[:H].astype(np.int64)
        a[:H] = (uh // (cols - 1)) * cols + uh % (cols - 1)
        b[:H] = a[:H] + 1
    if V:
        a[H:] = u[H:].astype(np.int64) - H
        b[H:] = a[H:] + cols
    h = _mix64(seed, u)
    kept = (h % np.uint64(1_000_000)) < np.uint64(int(round(keep * 1_000_000)))
    w = (1 + (h >> np.uint64(32)) % np.uint64(max_weight)).astype(np.int64)
    a, b, w = a[kept], b[kept], w[kept]
    return rows * cols, np.concatenate([a, b]), np.concatenate([b, a]), np.concatenate([w, w])
