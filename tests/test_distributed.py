"""Multi-rank destination sharding on CPU: world_size 2 over gloo.

The product's sharded driver (paper_1903_07754_b200.distributed.run_sharded,
its partitioning and its all-gather exchange) runs unchanged; each rank's
local compute is a CPU stand-in built from the oracle (test infrastructure)
over that rank's destination shard.  The union must reproduce the
single-process reference run: identical values and per-iteration traces
(mode, active edges, produced frontier size)."""

from __future__ import annotations

import os
import socket
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1903_07754_b200.distributed import ShardRecord, destination_bounds, run_sharded


class OracleShard:
    """CPU stand-in for DeviceShard: the shard's vectors and local index in
    the reference layout, driven through the same step / apply protocol."""

    device = "cpu"

    def __init__(self, n, src, dst, w, width, bounds, rank, app, root, threshold, vpg):
        lo, hi = bounds[rank], bounds[rank + 1]
        m = (dst >= lo) & (dst < hi)
        self.topo = oracle.build_pull_topology(n, src[m], dst[m], None if w is None else w[m], width)
        self.idx = oracle.build_edge_index(self.topo)
        self.deg = oracle.compute_out_degrees(n, src)  # global out-degrees
        self.E = len(src)
        self.n, self.app, self.root, self.thr, self.vpg = n, app, root, threshold, vpg
        self.kern = oracle.kern_of(app)

    def seed(self):
        vals, front = oracle.initial_state(self.app, self.n, self.root)
        self.prev, self.nxt = vals.copy(), vals.copy()
        self.fwords = np.zeros(oracle.word_count(self.n), np.uint64)
        oracle.set_bits(self.fwords, front)
        self.edge_sum = int(self.deg[np.unique(front)].sum())

    def step(self, it):
        be = oracle.PortBackend(1)
        np.copyto(self.nxt, self.prev)
        out = np.zeros(oracle.word_count(self.n), np.uint64)
        self.active = self.edge_sum
        num, den = self.thr.numerator, self.thr.denominator
        shift = self.vpg.bit_length() - 1
        if self.E > 0 and self.edge_sum * den < num * self.E:
            groups = (self.topo.vector_count + self.vpg - 1) // self.vpg
            ww = np.zeros(oracle.word_count(groups), np.uint64)
            be.transform(self.fwords, self.n, self.idx.offsets, self.idx.positions, shift, ww)
            self.touched = be.pull_wedge(self.topo, ww, shift, groups, self.prev, self.nxt, out, self.kern,
                                         oracle.UNREACHED)
            self.mode = "Wedge"
        else:
            self.touched = be.pull_full(self.topo, self.prev, self.nxt, out, self.kern, oracle.UNREACHED)
            self.mode = "FullScan"
        ch = oracle.bit_indices(out, self.n)
        return torch.from_numpy(ch.astype(np.int64)), torch.from_numpy(self.nxt[ch].copy())

    def apply(self, it, verts, vals):
        v = verts.numpy()
        self.nxt[v] = vals.numpy()
        self.prev, self.nxt = self.nxt, self.prev
        self.fwords = np.zeros(oracle.word_count(self.n), np.uint64)
        oracle.set_bits(self.fwords, v)
        self.edge_sum = int(self.deg[v].sum()) if v.size else 0
        return ShardRecord(it, self.mode, self.active, self.touched, int(v.size), self.edge_sum)

    def values_int64(self):
        return self.prev


class PackedOracleShard(OracleShard):
    """The fixed-size exchange protocol of DeviceShard (step packs; exchange
    all-gathers messages truncated to `cap` entries and reports the largest
    count) in numpy, so run_sharded's capacity / redo logic runs on gloo."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        b = a[5]  # the bounds argument
        self.capacity = max(b[r + 1] - b[r] for r in range(len(b) - 1))
        self.exchanged_caps = []

    def step(self, it):
        v, x = OracleShard.step(self, it)
        self.msg = np.zeros(1 + 2 * self.capacity, np.int64)
        self.msg[0] = v.numel()
        self.msg[1: 1 + v.numel()] = v.numpy()
        self.msg[1 + self.capacity: 1 + self.capacity + v.numel()] = x.numpy()

    def exchange(self, it, cap, group=None):
        world = dist.get_world_size(group)
        mine = torch.from_numpy(np.concatenate([self.msg[:1 + cap],
                                                self.msg[1 + self.capacity: 1 + self.capacity + cap]]))
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        vs, xs, maxc = [], [], 0
        for p in parts:
            c = int(p[0])
            maxc = max(maxc, c)
            m = min(c, cap)
            vs.append(p[1:1 + m])
            xs.append(p[1 + cap: 1 + cap + m])
        self.exchanged_caps.append(cap)
        return OracleShard.apply(self, it, torch.cat(vs), torch.cat(xs)), maxc


class SliceOracleShard(PackedOracleShard):
    """Adds DeviceShard's dense-iteration form: every rank all-gathers its
    owned value slice (padded to S) and derives the frontier from the value
    decrease, instead of exchanging (vertex, value) pairs."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.bounds = list(a[5])
        self.rank = a[6]
        self.S = self.capacity
        self.slice_iters = []

    def initial_edge_sum(self):
        vals, front = oracle.initial_state(self.app, self.n, self.root)
        return int(self.deg[np.unique(front)].sum())

    def gate_dense(self, edge_sum):
        num, den = self.thr.numerator, self.thr.denominator
        return not (self.E > 0 and edge_sum * den < num * self.E)

    def exchange_slices(self, it, group=None):
        world = dist.get_world_size(group)
        lo, hi = self.bounds[self.rank], self.bounds[self.rank + 1]
        mine = torch.zeros(self.S, dtype=torch.int64)
        mine[: hi - lo] = torch.from_numpy(self.nxt[lo:hi].copy())
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        new = np.concatenate([parts[r][: self.bounds[r + 1] - self.bounds[r]].numpy() for r in range(world)])
        changed = np.flatnonzero(new < self.prev)
        self.slice_iters.append(it)
        return OracleShard.apply(self, it, torch.from_numpy(changed), torch.from_numpy(new[changed]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q, packed=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, src, dst, w, app, thr, vpg = case
        bounds = destination_bounds(np.bincount(dst, minlength=n), 4, world)
        if packed == "slices":
            import paper_1903_07754_b200.distributed as D
            D.PACKED_MIN_CAP = 4
            shard = SliceOracleShard(n, src, dst, w, 4, bounds, rank, app, 0, thr, vpg)
        elif packed:
            import paper_1903_07754_b200.distributed as D
            D.PACKED_MIN_CAP = 4  # small messages, so truncated gathers and full-size redos both run
            shard = PackedOracleShard(n, src, dst, w, 4, bounds, rank, app, 0, thr, vpg)
        else:
            shard = OracleShard(n, src, dst, w, 4, bounds, rank, app, 0, thr, vpg)
        vals, recs, conv = run_sharded(shard, 10_000)
        if packed == "slices" and rank == 0:
            assert shard.slice_iters and shard.exchanged_caps  # both exchange forms ran
        elif packed and rank == 0:
            assert any(c < shard.capacity for c in shard.exchanged_caps)  # truncated gathers happened
        if rank == 0:
            q.put((vals, [(r.iteration, r.mode, r.active_edges, r.frontier_out_size) for r in recs], conv,
                   bounds))
    finally:
        dist.destroy_process_group()


def _single(case):
    n, src, dst, w, app, thr, vpg = case
    topo = oracle.build_pull_topology(n, src, dst, w, 4)
    idx = oracle.build_edge_index(topo)
    deg = oracle.compute_out_degrees(n, src)
    vals, front = oracle.initial_state(app, n, 0)
    out = oracle.run_until_convergence(topo, idx, deg, oracle.kern_of(app), vals, front, thr, vpg)
    return out.values, list(oracle.trace(out.stats)), out.converged


def _case(app, scale=10):
    n, s, d = oracle.rmat_edges(scale, 8, 5)
    keep = s != d
    s, d, _ = oracle.symmetrize(s[keep], d[keep], None, dedup=True)
    w = oracle.synthesize_weights(s, d, 255) if app == "sssp" else None
    thr = {"bfs": Fraction(1, 100), "cc": Fraction(1, 5), "sssp": Fraction(1, 5)}[app]
    vpg = 8 if app == "bfs" else 4
    return n, s, d, w, app, thr, vpg


@pytest.mark.parametrize("app,packed", [("bfs", False), ("cc", False), ("sssp", False), ("cc", True),
                                        ("sssp", True), ("cc", "slices"), ("bfs", "slices"),
                                        ("sssp", "slices")])
def test_two_rank_sharded_run_matches_single(app, packed):
    case = _case(app)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q, packed)) for r in range(2)]
    for p in procs:
        p.start()
    vals, trace, conv, bounds = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_vals, want_trace, want_conv = _single(case)
    assert 0 < bounds[1] < case[0]
    assert np.array_equal(vals, want_vals)
    assert [tuple(t) for t in trace] == [tuple(t) for t in want_trace]
    assert conv == want_conv


def test_destination_bounds_balance_and_alignment():
    rng = np.random.default_rng(0)
    deg = (rng.pareto(0.7, 5000) * 4).astype(np.int64)
    for world in (1, 2, 4, 8):
        b = destination_bounds(deg, 4, world)
        assert b[0] == 0 and b[-1] == len(deg) and all(x <= y for x, y in zip(b, b[1:]))
        vec = (deg + 3) // 4
        parts = [vec[b[i]:b[i + 1]].sum() for i in range(world)]
        assert sum(parts) == vec.sum()
        assert max(parts) - min(parts) <= 2 * vec.max() + 1


class OraclePageRankShard:
    """CPU stand-in for DevicePageRankShard (float64, edge-list form of the
    oracle's PageRank semantics) behind the same prep / pull / unpack protocol."""

    device = "cpu"

    def __init__(self, n, src, dst, bounds, rank, damping=0.85):
        lo, hi = bounds[rank], bounds[rank + 1]
        m = (dst >= lo) & (dst < hi)
        self.src, self.dst = src[m].astype(np.int64), dst[m].astype(np.int64)
        self.deg = np.bincount(src, minlength=n).astype(np.float64)
        self.n, self.lo, self.hi, self.bounds, self.d = n, lo, hi, bounds, damping
        world = len(bounds) - 1
        self.S = max(max(bounds[r + 1] - bounds[r] for r in range(world)), 1)
        self.acc = np.zeros(n)
        self.r = None
        self.gathered = torch.zeros(world * self.S, dtype=torch.float64)

    def prep(self, it):
        self.r = np.full(self.n, 1.0 / self.n) if it == 0 else \
            (1 - self.d) / self.n + self.d * (self.acc + self.dangling / self.n)
        self.contrib = np.where(self.deg > 0, self.r / np.maximum(self.deg, 1), 0.0)
        self.dangling = self.r[self.deg == 0].sum()

    def pull(self):
        part = np.zeros(self.S)
        part[: self.hi - self.lo] = np.bincount(self.dst - self.lo, weights=self.contrib[self.src],
                                                minlength=self.hi - self.lo)[: self.hi - self.lo]
        return torch.from_numpy(part)

    def unpack(self):
        g = self.gathered.numpy()
        for r in range(len(self.bounds) - 1):
            lo, hi = self.bounds[r], self.bounds[r + 1]
            self.acc[lo:hi] = g[r * self.S: r * self.S + hi - lo]

    def finish(self, iterations):
        self.prep(iterations)
        return self.r


def _pr_worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1903_07754_b200.distributed import run_pagerank_sharded
        n, src, dst = case
        bounds = destination_bounds(np.bincount(dst, minlength=n), 4, world)
        r = run_pagerank_sharded(OraclePageRankShard(n, src, dst, bounds, rank), 20)
        q.put((rank, r, bounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pagerank_matches_single(world):
    n, s, d = oracle.rmat_edges(10, 8, 7)
    keep = s != d
    s, d = s[keep], d[keep]  # directed, with dangling vertices
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pr_worker, args=(r, world, port, (n, s, d), q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.pagerank_numpy(n, s, d, 20)
    assert (np.bincount(s, minlength=n) == 0).any()
    for rank, r, bounds in got:
        assert len(set(bounds)) == world + 1
        assert np.max(np.abs(r - want)) <= 1e-12, rank


def _partition_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1903_07754_b200.distributed import partition_edges
        n, s, d = oracle.rmat_edges(10, 8, 3)
        # every rank contributes a different part of the edge list
        m = len(s)
        lo, hi = rank * m // world, (rank + 1) * m // world
        bounds = destination_bounds(np.bincount(d, minlength=n), 4, world)
        ls, ld, lw = partition_edges(torch.from_numpy(s[lo:hi]), torch.from_numpy(d[lo:hi]),
                                     torch.from_numpy(s[lo:hi] * 7 + 1), bounds)
        q.put((rank, ls.numpy(), ld.numpy(), lw.numpy(), bounds))
    finally:
        dist.destroy_process_group()


def test_partition_edges_routes_every_edge_to_its_owner():
    """partition_edges (the sharded ingest's all-to-all): every edge arrives
    exactly once, at the rank owning its destination, with its attributes."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partition_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, s, d = oracle.rmat_edges(10, 8, 3)
    all_s, all_d = [], []
    for rank, ls, ld, lw, bounds in got:
        assert np.all((ld >= bounds[rank]) & (ld < bounds[rank + 1]))
        assert np.array_equal(lw, ls * 7 + 1)
        all_s.append(ls)
        all_d.append(ld)
    key = lambda a, b: np.sort(a.astype(np.int64) * (1 << 32) + b)
    assert np.array_equal(key(np.concatenate(all_s), np.concatenate(all_d)), key(s, d))
