"""Pull-only engine API (reference engine.py:1-388) on the B200 backend.

``run_until_convergence`` delegates the whole loop to the backend when the
backend offers ``run_until_convergence`` (the B200 backend does): the gate,
the Wedge transform, the wedge / dense pulls, the O(|F|) double-buffer sync
and the convergence test all run on the device, and the host reads one
16-word record per iteration after each batch.  For a
backend that only implements the per-call protocol, the same loop is driven
from the host (``_host_loop``), call for call like engine.py:330-388.

Only ``MinPlusKernel`` programs run on the device (the three applications
are all of that family, apps.py:28-100); a program without a kernel
descriptor raises ``NotImplementedError`` instead of silently running a CPU
path.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass
from fractions import Fraction
from time import perf_counter
from typing import Any, Callable, Optional, Sequence

import numpy as np

from .frontier import (DEFAULT_SLICE_SIZE, Bitmask, FrontierPrecision, FullnessThreshold,
                       VertexFrontier, WedgeFrontier, should_transform, transform_frontier)

UNREACHED = 1 << 62  # engine.py:43: sentinel + weight + 1 never overflows int64
MODE_FULL = "FullScan"
MODE_WEDGE = "Wedge"


@dataclass(frozen=True)
class MinPlusKernel:
    """engine.py:50-63: messages prev[src] (+ weight), combined by min;
    update to min + apply_increment iff strictly smaller."""

    filter_unvisited: bool
    use_weight: bool
    apply_increment: int


@dataclass(frozen=True)
class ApplicationProgram:
    """engine.py:66-87 (callables kept for API parity; the device runs ``kernel``)."""

    name: str
    initial_value: Callable[[int], Any]
    initial_frontier: Callable[[int], Sequence[int]]
    gather: Callable[[Any, Any], Any]
    combine: Callable[[Any, Any], Any]
    apply: Callable[[Any, Any], tuple]
    should_process: Callable[[Any], bool] = lambda value: True
    needs_weights: bool = False
    kernel: Optional[MinPlusKernel] = None
    initial_values: Optional[Callable[[int], np.ndarray]] = None


class ValueBuffers:
    """engine.py:90-116: strict double buffer (read previous, write next)."""

    __slots__ = ("previous", "next")

    def __init__(self, previous, next):
        self.previous = previous
        self.next = next

    @classmethod
    def initialize(cls, program: ApplicationProgram, vertex_count: int) -> "ValueBuffers":
        prev = _initial_values(program, vertex_count)
        return cls(prev, prev.copy())

    def swap(self) -> None:
        self.previous, self.next = self.next, self.previous

    def __len__(self) -> int:
        return len(self.previous)


@dataclass
class IterationStats:
    mode: str
    pull_time: float
    vectors_touched: int
    frontier_out_size: int
    iteration: int = 0
    transform_time: float = 0.0
    active_edges: int = 0
    active_edge_fraction: Optional[Fraction] = None
    covered_vectors: int = 0
    transform_entries: int = 0


@dataclass(frozen=True)
class EngineConfig:
    threshold: FullnessThreshold = FullnessThreshold(Fraction(1, 5))
    precision: FrontierPrecision = FrontierPrecision(4)
    workers: int = 1
    slice_size: int = DEFAULT_SLICE_SIZE
    max_iterations: int = 1_000_000

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.slice_size < 1:
            raise ValueError("slice_size must be >= 1")


@dataclass
class RunResult:
    values: Any
    stats: list
    converged: bool
    device_ms: float = 0.0

    @property
    def iterations(self) -> int:
        return len(self.stats)


def result_digest(values) -> str:
    """engine.py:173-176: blake2b-64 of int64 little-endian values."""
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.int64), dtype="<i8")
    return hashlib.blake2b(arr.tobytes(), digest_size=8).hexdigest()


def stats_signature(stats: Sequence) -> tuple:
    """engine.py:179-185: stats without timings."""
    return tuple((s.iteration, s.mode, s.active_edges,
                  getattr(s, "vectors_touched", getattr(s, "edges_touched", 0)), s.frontier_out_size)
                 for s in stats)


def _initial_values(program: ApplicationProgram, n: int) -> np.ndarray:
    if getattr(program, "initial_values", None) is not None:
        return np.ascontiguousarray(program.initial_values(n), dtype=np.int64)
    return np.fromiter((program.initial_value(v) for v in range(n)), dtype=np.int64, count=n)


def _require_kernel(program: ApplicationProgram) -> MinPlusKernel:
    if program.kernel is None:
        raise NotImplementedError(
            f"program {program.name!r} has no MinPlusKernel descriptor; the B200 engine runs "
            "min-plus programs (BFS / CC / SSSP) only")
    return program.kernel


def _check_buffers(buffers: ValueBuffers, n: int) -> None:
    if len(buffers.previous) != n or len(buffers.next) != n:
        raise ValueError(f"value buffers must have length {n}")


def _check_weights(topology, program: ApplicationProgram) -> None:
    if program.needs_weights and not topology.is_weighted():
        raise ValueError(f"program {program.name!r} requires edge weights")


def _finish(out: Bitmask, degrees) -> tuple:
    members = out.indices()
    s = int(np.asarray(degrees)[members].sum()) if members.size else 0
    return VertexFrontier(out, s), int(members.size)


def run_iteration_full(topology, buffers: ValueBuffers, program: ApplicationProgram, degrees,
                       workers: int = 1, backend=None):
    """engine.py:251-279: one pull over every vector."""
    from .backend import get_backend
    n = topology.vertex_count
    _check_buffers(buffers, n)
    _check_weights(topology, program)
    kern = _require_kernel(program)
    prev, nxt = buffers.previous, buffers.next
    np.copyto(nxt, prev)
    out = Bitmask(n)
    t0 = perf_counter()
    touched = get_backend(backend).pull_full(topology, prev, nxt, out.words, kern, UNREACHED, workers)
    dt = perf_counter() - t0
    frontier, size = _finish(out, degrees)
    return frontier, IterationStats(MODE_FULL, dt, int(touched), size)


def run_iteration_wedge(topology, wedge: WedgeFrontier, buffers: ValueBuffers,
                        program: ApplicationProgram, degrees, workers: int = 1, backend=None):
    """engine.py:282-327: one pull restricted to the covered vectors."""
    from .backend import get_backend
    n = topology.vertex_count
    _check_buffers(buffers, n)
    _check_weights(topology, program)
    if wedge.vector_count != topology.vector_count:
        raise ValueError(f"wedge frontier built for {wedge.vector_count} vectors, topology has "
                         f"{topology.vector_count}")
    kern = _require_kernel(program)
    prev, nxt = buffers.previous, buffers.next
    np.copyto(nxt, prev)
    out = Bitmask(n)
    t0 = perf_counter()
    touched = get_backend(backend).pull_wedge(topology, wedge.bits.words, wedge.precision.shift,
                                              wedge.group_count, prev, nxt, out.words, kern,
                                              UNREACHED, workers)
    dt = perf_counter() - t0
    frontier, size = _finish(out, degrees)
    st = IterationStats(MODE_WEDGE, dt, int(touched), size)
    st.covered_vectors = wedge.covered_vector_count()
    st.transform_entries = wedge.entries_visited
    return frontier, st


def run_until_convergence(topology, index, program: ApplicationProgram, degrees,
                          config: EngineConfig, backend=None, frontier_log: list | None = None,
                          value_log: list | None = None) -> RunResult:
    """engine.py:330-388."""
    from .backend import get_backend
    n = topology.vertex_count
    if index.vertex_count != n or index.vector_count != topology.vector_count:
        raise ValueError("edge index does not match topology")
    _check_weights(topology, program)
    be = get_backend(backend)
    if hasattr(be, "run_until_convergence"):
        return be.run_until_convergence(topology, index, program, degrees, config,
                                        frontier_log=frontier_log, value_log=value_log)
    return _host_loop(topology, index, program, degrees, config, be, frontier_log, value_log)


def _host_loop(topology, index, program, degrees, config, be, frontier_log, value_log) -> RunResult:
    """The reference loop driven from the host over a per-call backend."""
    n = topology.vertex_count
    buffers = ValueBuffers.initialize(program, n)
    frontier = VertexFrontier.from_vertices(program.initial_frontier(n), degrees, n)
    total = topology.edge_count
    stats: list = []
    converged = False
    while not converged and len(stats) < config.max_iterations:
        in_edges = frontier.member_edge_sum
        if total > 0 and should_transform(frontier, total, config.threshold):
            t0 = perf_counter()
            wedge = transform_frontier(frontier, index, config.precision, config.slice_size,
                                       config.workers, be)
            tt = perf_counter() - t0
            frontier, st = run_iteration_wedge(topology, wedge, buffers, program, degrees,
                                               config.workers, be)
            st.transform_time = tt
        else:
            frontier, st = run_iteration_full(topology, buffers, program, degrees, config.workers, be)
        st.iteration = len(stats) + 1
        st.active_edges = in_edges
        st.active_edge_fraction = Fraction(in_edges, total) if total else Fraction(0)
        buffers.swap()
        stats.append(st)
        if frontier_log is not None:
            frontier_log.append(frontier.members())
        if value_log is not None:
            value_log.append(buffers.previous.copy())
        converged = frontier.member_edge_sum == 0
    return RunResult(values=buffers.previous, stats=stats, converged=converged)


# ---------------------------------------------------------------------------
# Device-resident loop (called through B200Backend.run_until_convergence)
# ---------------------------------------------------------------------------
def _initial_members(program: ApplicationProgram, n: int):
    ids = program.initial_frontier(n)
    if isinstance(ids, range) and ids == range(n):
        return None  # every vertex (CC, apps.py:56-73)
    arr = ids if isinstance(ids, np.ndarray) else np.fromiter(ids, dtype=np.int64)
    return np.unique(np.asarray(arr, dtype=np.int64))


def device_run(be, topology, index, program: ApplicationProgram, degrees, config: EngineConfig,
               frontier_log=None, value_log=None) -> RunResult:
    from . import device as dv
    from ._lib import OverflowError32, WG_VAL_I64, WG_VAL_U32
    import torch

    kern = _require_kernel(program)
    n = topology.vertex_count
    init = _initial_values(program, n)
    members = _initial_members(program, n)
    total = int(topology.edge_count)

    if total == 0 or n == 0:
        # no edges: one FullScan that touches nothing (engine.py:356-388)
        mem = np.arange(n, dtype=np.int64) if members is None else members
        if mem.size and (mem.min() < 0 or mem.max() >= n):
            raise IndexError("bit position out of range")
        st = IterationStats(MODE_FULL, 0.0, 0, 0, iteration=1,
                            active_edges=int(np.asarray(degrees)[mem].sum()) if mem.size else 0,
                            active_edge_fraction=Fraction(0))
        if frontier_log is not None:
            frontier_log.append(np.empty(0, np.int64))
        if value_log is not None:
            value_log.append(init.copy())
        return RunResult(values=init, stats=[st], converged=True)

    g = be.device_graph(topology, index, degrees)
    g = _with_degrees(be, g, degrees)
    iv = dv.prepare_initial_values(init, kern, members)
    val_type = WG_VAL_U32 if iv.fits_u32 else WG_VAL_I64
    words = dv.all_words(n) if members is None else dv.initial_words(n, members)
    while True:
        loop = _loop_for(be, g, config.precision.shift, val_type)
        trace = None
        if frontier_log is not None or value_log is not None:
            def trace(lp, it):
                if frontier_log is not None:
                    frontier_log.append(lp.frontier_members(it))
                if value_log is not None:
                    value_log.append(dv.values_to_int64(lp.values_after(it), val_type))
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        p = loop.seed(iv.seed(val_type), words, kern, config.threshold.fraction, first_hit=iv.first_hit,
                      level_base=iv.level_base, identity_init=iv.identity, defer=True)
        timer = None
        if getattr(be, "per_iteration_timing", False):
            # CUDA events around each launch group (one iteration per launch)
            from ._lib import EventTimer
            timer = EventTimer(8 * min(config.max_iterations, 4096) + 64)
            p.timer = timer.handle
        try:
            recs, converged, last = loop.drive(p, config.max_iterations, trace)
        except OverflowError32:
            if val_type == WG_VAL_I64:
                raise
            val_type = WG_VAL_I64  # exact int64 path (never overflows, engine.py:41-43)
            if frontier_log is not None:
                frontier_log.clear()
            if value_log is not None:
                value_log.clear()
            continue
        stop.record()
        stop.synchronize()
        break
    ms = start.elapsed_time(stop)
    values = dv.values_to_int64(loop.values_after(last), val_type)
    per = (ms / 1000.0) / max(len(recs), 1)
    split = {}
    if timer is not None:
        for kind, it, t in timer.read():
            d = split.setdefault(it, [0.0, 0.0])
            d[0 if kind == 1 else 1] += t / 1000.0  # kind 1: transform; 2-4: pull + end of iteration
    stats = []
    for r in recs:
        tt, pt = split.get(r.iteration, (0.0, per))
        st = IterationStats(r.mode, pt, r.vectors_touched, r.frontier_out_size, iteration=r.iteration,
                            transform_time=tt if r.mode == MODE_WEDGE else 0.0,
                            active_edges=r.active_edges,
                            active_edge_fraction=Fraction(r.active_edges, total),
                            covered_vectors=r.covered_vectors, transform_entries=r.transform_entries)
        stats.append(st)
    return RunResult(values=values, stats=stats, converged=converged, device_ms=ms)


def _with_degrees(be, g, degrees):
    """Use the caller's out-degree table for the gate (engine.py:361) when it
    differs from the layout's own (uploaded once per degrees object)."""
    if degrees is None:
        return g
    if getattr(g, "_degrees_src", None) is degrees:
        return g  # the graph was uploaded with exactly these degrees
    deg = np.asarray(degrees)
    own = getattr(g, "_outdeg_host", None)
    if own is None:
        own = g.outdeg_np()
        g._outdeg_host = own
    if deg.shape == own.shape and np.array_equal(deg, own):
        return g
    from . import device as dv

    def make():
        h = dv.DeviceGraph(g.n, g.width, g.edges, g.nvec, g.entries, g.vsrc, g.vdst, g.vw, g.idx_off,
                           g.idx_pos, dv.to_dev_u32(deg if deg.size else np.zeros(1, np.int64)))
        h._outdeg_host = deg.astype(np.int64)
        return h
    return be._cache.get([g, degrees], make)


def _loop_for(be, g, shift: int, val_type: int):
    from .device import DeviceLoop
    cache = be.__dict__.setdefault("_loops", {})
    key = (id(g), shift, val_type)
    hit = cache.get(key)
    if hit is not None and hit.g is g:
        return hit
    if len(cache) > 4:
        cache.clear()
    loop = DeviceLoop(g, shift, val_type)
    cache[key] = loop
    return loop
