"""Destination-range sharding across GPUs (the paper's
multi-socket design, which the reference does not implement).

Rank r owns a contiguous destination range chosen on destination boundaries
so that every rank holds about the same number of vectors (balanced by edges,
not vertices: RMAT puts the hubs at low ids and ~half the vertices have no
in-edges).  Each rank keeps its own vectors, a local edge index over ALL
sources (positions local to its slice), the global out-degrees, and full
replicas of the values and of the frontier.  Per iteration:

  1. every rank runs the gate on the same global frontier edge sum, so the
     mode (Wedge / FullScan) is a global decision;
  2. local Wedge transform + local pull (wg_run_enqueue, one iteration);
  3. exchange: each rank packs the destinations it updated and their new
     values (wg_exchange_pack) and all ranks all-gather them (NCCL over
     NVLink on GPUs; the same code runs on gloo in the CPU tests); counts
     first, then a padded all-gather (NCCL has no all-gatherv);
  4. wg_exchange_apply writes the union into both value buffers and rebuilds
     the global frontier list / edge sum for the next gate.

The driver (``run_sharded``) is written against a small shard interface so
that the exchange protocol is tested on CPU with world_size 2 (gloo) while
the device shard (``DeviceShard``) runs the sm_100a kernels.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np


# ---------------------------------------------------------------------------
# Partitioning
# ---------------------------------------------------------------------------
def destination_bounds(indeg, width: int, world: int) -> list[int]:
    """Split [0, n) into `world` destination ranges holding ~equal numbers of
    W-lane vectors (vectors of d = ceil(indeg(d)/W), graph.py:240-243).
    Ranges never split a destination (the kernels.py:39-52 invariant)."""
    deg = np.asarray(indeg, dtype=np.int64)
    n = int(deg.shape[0])
    vec = (deg + width - 1) // width
    cum = np.cumsum(vec)
    total = int(cum[-1]) if n else 0
    bounds = [0]
    for k in range(1, world):
        target = (k * total) // world
        d = int(np.searchsorted(cum, target, side="left")) + 1 if total else 0
        d = min(max(d, bounds[-1]), n)
        bounds.append(d)
    bounds.append(n)
    return bounds


# ---------------------------------------------------------------------------
# Partitioned ingest: no rank ever holds the whole edge list
# ---------------------------------------------------------------------------
def partition_edges(src, dst, weight, bounds, group=None):
    """Send every edge to the rank owning its destination (one all-to-all
    per array, counts first); returns this rank's (src, dst, weight) -- the
    edges of its destination range.  torch tensors (any device the process
    group serves); works on nccl and gloo."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = src.device
    cut = torch.tensor(bounds[1:-1], dtype=torch.int64, device=dev)
    d64 = dst.to(torch.int64) & 0xFFFFFFFF if dst.dtype == torch.int32 else dst.to(torch.int64)
    owner = torch.bucketize(d64, cut, right=True)
    order = torch.argsort(owner, stable=True)
    send_counts = torch.bincount(owner, minlength=world).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    sc, rc = send_counts.cpu().tolist(), recv_counts.cpu().tolist()

    def move(t):
        if t is None:
            return None
        out = torch.empty(sum(rc), dtype=t.dtype, device=dev)
        dist.all_to_all_single(out, t[order].contiguous(), output_split_sizes=rc, input_split_sizes=sc,
                               group=group)
        return out
    return move(src), move(dst), move(weight)


def rmat_partitioned(scale: int, edge_factor: int, seed: int, symmetric: bool, width: int = 4, group=None):
    """BASELINE's RMAT inputs built by destination shards:
    rank r generates rows [r*m/G, (r+1)*m/G) of the reference's PCG64 stream
    (graph_io.py:188-202; the generator jumps ahead, PCG64.advance), drops
    self-loops, adds the reverse edges when symmetric, and ships every edge
    to its destination's owner; each rank then de-duplicates its own edges
    (duplicates share a destination).  Returns (n, E, bounds, src, dst,
    global out-degrees) with the bounds balanced on the in-degrees."""
    import torch
    import torch.distributed as dist
    from . import device as dv
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = 1 << scale
    m = edge_factor * n
    lo, hi = rank * m // world, (rank + 1) * m // world
    s, d = dv.rmat_edges_rows(scale, lo, hi, seed)
    s64, d64 = s.to(torch.int64) & 0xFFFFFFFF, d.to(torch.int64) & 0xFFFFFFFF
    keep = s64 != d64
    s, d = s[keep], d[keep]
    if symmetric:
        s, d = torch.cat([s, d]), torch.cat([d, s])
    # destination bounds from the global (pre-dedup) in-degree histogram
    hist = torch.bincount(d.to(torch.int64) & 0xFFFFFFFF, minlength=n)
    dist.all_reduce(hist, group=group)
    bounds = destination_bounds(hist.cpu().numpy(), width, world)
    s, d, _ = partition_edges(s, d, None, bounds, group)
    s, d = dv.canonical_edges(s, d, drop_loops=False, symmetrize=False)  # local dedup
    outdeg = torch.bincount(s.to(torch.int64) & 0xFFFFFFFF, minlength=n)
    dist.all_reduce(outdeg, group=group)
    E = torch.tensor([s.numel()], dtype=torch.int64, device=s.device)
    dist.all_reduce(E, group=group)
    return n, int(E.item()), bounds, s, d, outdeg.to(torch.int32)


# ---------------------------------------------------------------------------
# Exchange
# ---------------------------------------------------------------------------
def all_gather_var(t, group=None):
    """All-gather tensors of different lengths: counts first, then a padded
    all-gather of equal-size buffers (works on nccl and gloo)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    cnt = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    maxc = max(counts)
    if maxc == 0:
        return t[:0]
    buf = torch.zeros(maxc, dtype=t.dtype, device=t.device)
    buf[: t.numel()].copy_(t)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def all_gather_pairs(verts, vals, group=None):
    """All-gather (vertex, value) update lists of different lengths with one
    count exchange and one padded all-gather: each rank sends its vertices
    and values as the int32 words of a single buffer."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    k = int(verts.numel())
    a = verts.element_size() // 4  # int32 words per vertex id
    b = vals.element_size() // 4   # int32 words per value
    cnt = torch.tensor([k], dtype=torch.int64, device=verts.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = torch.cat(counts).cpu().tolist()
    maxc = max(counts)
    if maxc == 0:
        return verts[:0], vals[:0]
    buf = torch.zeros(maxc * (a + b), dtype=torch.int32, device=verts.device)
    buf[: k * a].copy_(verts.contiguous().view(torch.int32))
    buf[maxc * a: maxc * a + k * b].copy_(vals.contiguous().view(torch.int32))
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    av = torch.cat([p[: c * a] for p, c in zip(parts, counts)]).view(verts.dtype)
    ax = torch.cat([p[maxc * a: maxc * a + c * b] for p, c in zip(parts, counts)]).view(vals.dtype)
    return av, ax


PACKED_MIN_CAP = 4096  # smallest message capacity (entries) of the packed exchange


@dataclass
class ShardRecord:
    iteration: int
    mode: str
    active_edges: int
    vectors_touched: int
    frontier_out_size: int
    out_edge_sum: int
    covered_vectors: int = 0
    transform_entries: int = 0


def run_sharded(shard, max_iterations: int, group=None, values: bool = True):
    """The reference loop (engine.py:330-388) over destination shards:
    local step, exchange of updated values, global frontier for the gate.
    values=False skips the host copy of the final values (timed runs; read
    them afterwards with shard.values_int64())."""
    import torch
    import torch.distributed as dist
    if dist.get_world_size(group) == 1 and hasattr(shard, "run_alone"):
        # one rank: every exchange would be the identity -- the whole loop
        # runs as the single-GPU loop graph, no per-iteration host round trip
        return shard.run_alone(max_iterations, values)
    shard.seed()
    recs: list[ShardRecord] = []
    converged = False
    it = 0
    packed = hasattr(shard, "exchange")
    slices = hasattr(shard, "exchange_slices")
    cap = getattr(shard, "capacity", 0)
    prev_sum = shard.initial_edge_sum() if slices else None
    while it < max_iterations:
        it += 1
        if slices and shard.gate_dense(prev_sum):
            # dense iteration (the global gate, evaluated alike on every rank):
            # every rank's owned value slice (4 or 8 B per owned vertex) rather
            # than (vertex, value) pairs for most of its vertices
            shard.step(it)
            rec = shard.exchange_slices(it, group)
        elif packed:
            # one fixed-size all-gather of truncated messages per iteration;
            # the largest count (global, so every rank decides alike) sizes
            # the next one and triggers a full-size redo when exceeded
            shard.step(it)
            rec, maxc = shard.exchange(it, cap, group)
            if maxc > cap:
                rec, maxc = shard.exchange(it, shard.capacity, group)
            cap = min(shard.capacity, max(PACKED_MIN_CAP, 2 * maxc))
        else:
            verts, vals = shard.step(it)
            all_v, all_x = all_gather_pairs(verts, vals, group)
            rec = shard.apply(it, all_v, all_x)
        recs.append(rec)
        prev_sum = rec.out_edge_sum
        if rec.out_edge_sum == 0:
            converged = True
            break
    # work counters are per shard: sum them across ranks (traces are global already)
    if recs:
        dev = shard.device if hasattr(shard, "device") else "cpu"
        w = torch.tensor([[r.vectors_touched, r.covered_vectors, r.transform_entries] for r in recs],
                         dtype=torch.int64, device=dev)
        dist.all_reduce(w, group=group)
        for r, row in zip(recs, w.cpu().tolist()):
            r.vectors_touched, r.covered_vectors, r.transform_entries = row
    return (shard.values_int64() if values else None), recs, converged


# ---------------------------------------------------------------------------
# Device shard
# ---------------------------------------------------------------------------
class DeviceShard:
    """One rank's destination shard on its GPU (uses the device loop for the
    local iteration and the C-ABI exchange kernels)."""

    device = "cuda"

    def __init__(self, n: int, src, dst, weight, width: int, bounds: list[int], rank: int, kern,
                 init_values: np.ndarray, init_members: Optional[np.ndarray], threshold: Fraction,
                 shift: int, val_type: int, local: Optional[tuple] = None, gate: str = "global"):
        """src/dst/weight: the whole edge list (masked to this rank's range
        here), or -- with local=(E, global out-degrees) -- only this rank's
        edges already (partition_edges / rmat_partitioned).  gate: "global"
        (the reference's decision, identical on every rank: reference-parity
        modes and counters) or "local" (WG_RUN_LOCAL_GATE: each shard picks
        Wedge / FullScan from its own share of the frontier's edges; same
        values and frontiers)."""
        if gate not in ("global", "local"):
            raise ValueError("gate must be 'global' or 'local'")
        self.gate = gate
        import torch
        from . import _lib
        from . import device as dv
        self.dv, self._lib = dv, _lib
        lo, hi = bounds[rank], bounds[rank + 1]
        s = dv.to_dev_u32(src)
        d = dv.to_dev_u32(dst)
        w = dv.to_dev_u32(weight) if weight is not None else None
        if local is None:
            d64 = d.to(torch.int64) & 0xFFFFFFFF
            mask = (d64 >= lo) & (d64 < hi)
            E = int(s.numel())
            gdeg = torch.bincount(s.to(torch.int64) & 0xFFFFFFFF, minlength=n).to(torch.int32)
            s, d, w = s[mask], d[mask], (w[mask] if w is not None else None)
        else:
            E, gdeg = int(local[0]), dv.to_dev_u32(local[1])
        g = dv.DeviceGraph.build(n, s, d, w, width)
        # global out-degrees and |E| drive the (global) gate
        # (a shard's index lengths are its LOCAL out-edge counts: they equal the
        # global out-degrees only when the shard holds every destination)
        whole = lo == 0 and hi == n and g.edges == E
        self.g = dv.DeviceGraph(n, width, E, g.nvec, g.entries, g.vsrc, g.vdst, g.vw, g.idx_off,
                                g.idx_pos, gdeg, lens_are_degrees=whole and g.lens_are_degrees, vw8=g.vw8)
        self.lo, self.hi, self.n, self.rank = lo, hi, n, rank
        self.kern, self.threshold, self.shift, self.val_type = kern, threshold, shift, val_type
        self.loop = dv.DeviceLoop(self.g, shift, val_type)
        self.init = dv.encode_values(init_values, val_type)
        self.words = dv.all_words(n) if init_members is None else dv.initial_words(n, init_members)
        # the run flags the single-GPU engine derives from the initial state
        # (results and counters unchanged; the lockstep GPU test checks them)
        iv = np.asarray(init_values, dtype=np.int64)
        self.first_hit = dv.first_hit_ok(kern, iv, init_members)
        self.level_base = dv.first_hit_level(iv) if self.first_hit else 0
        self.identity = dv.identity_values(iv)
        cap = max(hi - lo, 1)
        self.out_v = torch.empty(cap, dtype=torch.int32, device="cuda")
        self.out_x = torch.empty(cap, dtype=torch.int32 if val_type == _lib.WG_VAL_U32 else torch.int64,
                                 device="cuda")
        # packed exchange buffers: capacity = the largest shard's destination
        # count (a rank updates only its own destinations)
        world = len(bounds) - 1
        self.capacity = max(bounds[r + 1] - bounds[r] for r in range(world)) if world else 1
        L = _lib.load()
        nb = int(L.wg_exchange_bytes(self.capacity, val_type))
        self.send = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        self.recv = torch.empty(world * nb, dtype=torch.uint8, device="cuda")
        self.status = torch.zeros(2, dtype=torch.int64, device="cuda")
        self.host_status = torch.zeros(2, dtype=torch.int64).pin_memory()
        # dense-iteration exchange: owned value slices, padded to S
        self.world, self.bounds = world, list(bounds)
        self.S = self.capacity
        vt = torch.int32 if val_type == _lib.WG_VAL_U32 else torch.int64
        self.slice_send = torch.empty(self.S, dtype=vt, device="cuda")
        self.slice_recv = torch.empty(world * self.S, dtype=vt, device="cuda")
        self.d_bounds = torch.tensor(np.asarray(bounds, dtype=np.uint32).view(np.int32), device="cuda")
        self.ovf = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.E = E
        self.init_members = init_members
        self.p = None

    def seed(self):
        self._last = None
        # wg_exchange_pack reads the member lists of every iteration
        flags = self._lib.WG_RUN_KEEP_LISTS | (self._lib.WG_RUN_LOCAL_GATE if self.gate == "local" else 0)
        self.p = self.loop.seed(self.init, self.words, self.kern, self.threshold, first_hit=self.first_hit,
                                level_base=self.level_base, identity_init=self.identity, extra_flags=flags)
        self.global_limit = self.dv.wedge_limit(self.threshold, self.E) if self.E > 0 else 0

    def initial_edge_sum(self) -> int:
        """Out-degree sum of the initial frontier (the first gate's input; cached)."""
        if getattr(self, "_init_sum", None) is None:
            import torch
            deg = self.g.outdeg[: self.n].to(torch.int64) & 0xFFFFFFFF
            if self.init_members is not None:
                m = torch.from_numpy(np.unique(np.asarray(self.init_members, dtype=np.int64))).to(deg.device)
                deg = deg[m]
            self._init_sum = int(deg.sum().item())
        return self._init_sum

    def gate_dense(self, edge_sum: int) -> bool:
        """The global gate (frontier.py:163-171) for the next iteration: it
        picks the exchange form (alike on every rank whatever the local modes)."""
        return not (self.E > 0 and edge_sum < self.global_limit)

    def exchange_slices(self, it: int, group=None):
        """Dense iterations: all-gather every rank's owned value slice, apply
        them (values + frontier bits from the value decrease) and rebuild the
        global frontier; an overflow on any rank raises on every rank."""
        import torch
        import torch.distributed as dist
        L = self._lib.load()
        lo, hi = self.lo, self.hi
        self._lib.check(L.wg_exchange_slice_pack(ctypes.byref(self.g.struct()), ctypes.byref(self.loop.bufs),
                                                 ctypes.byref(self.p), it, lo, hi, self.slice_send.data_ptr(),
                                                 self._lib.stream_ptr()))
        dist.all_gather_into_tensor(self.slice_recv, self.slice_send, group=group)
        return self.apply_slices(it, self.slice_recv, group)

    def apply_slices(self, it: int, recv, group=None, overflow_any=None):
        """Apply gathered slices (world x S values)."""
        import torch.distributed as dist
        L = self._lib.load()
        # the local overflow flag of `it`, made global (one tiny all-reduce)
        self.ovf.copy_(self.loop.recs.view(-1, self._lib.REC_U64)[it % self.loop.ring, 10:11])
        if overflow_any is None:
            dist.all_reduce(self.ovf, op=dist.ReduceOp.MAX, group=group)
        else:
            self.ovf.fill_(int(overflow_any))
        self._lib.check(L.wg_exchange_apply_slices(ctypes.byref(self.g.struct()), ctypes.byref(self.loop.bufs),
                                                   ctypes.byref(self.p), it, recv.data_ptr(),
                                                   self.d_bounds.data_ptr(), self.world, self.rank, self.S,
                                                   self._lib.stream_ptr()))
        rec, ovf = self._record(it, raise_overflow=False)
        if ovf or int(self.ovf.item()):
            raise self._lib.OverflowError32(self._lib.WG_EOVERFLOW, "uint32 overflow in sharded loop (some rank)")
        return rec

    def run_alone(self, max_iterations: int, values: bool = True):
        """World size 1: the device loop to convergence (DeviceLoop.drive)."""
        self.p = self.loop.seed(self.init, self.words, self.kern, self.threshold, first_hit=self.first_hit,
                                level_base=self.level_base, identity_init=self.identity,
                                extra_flags=self._lib.WG_RUN_LOCAL_GATE if self.gate == "local" else 0,
                                defer=True)  # the seed runs as the loop graph's prologue: one launch per run
        recs, conv, last = self.loop.drive(self.p, max_iterations)
        self._last = last
        # a produced frontier's out-edge sum is the next iteration's active edges
        nxt = [r.active_edges for r in recs[1:]] + [0]
        out = [ShardRecord(r.iteration, r.mode, r.active_edges, r.vectors_touched, r.frontier_out_size,
                           e, r.covered_vectors, r.transform_entries) for r, e in zip(recs, nxt)]
        vals = self.dv.values_to_int64(self.loop.values_after(last), self.val_type) if values else None
        return vals, out, conv

    def step(self, it: int):
        """Local iteration + pack of its members (no host synchronisation)."""
        L = self._lib.load()
        if os.environ.get("WG_SHARD_GRAPH", "1") != "0":
            self.loop.launch(self.p, it)  # the loop graph, stopped after iteration `it`
        else:
            self.loop.enqueue(self.p, it, 1)
        self._lib.check(L.wg_exchange_pack_all(ctypes.byref(self.g.struct()), ctypes.byref(self.loop.bufs),
                                               ctypes.byref(self.p), it, self.send.data_ptr(), self.capacity,
                                               self._lib.stream_ptr()))

    def exchange(self, it: int, cap: int, group=None):
        """All-gather every rank's message truncated to `cap` entries, apply
        them and rebuild the global frontier; returns (record, largest count)."""
        import torch.distributed as dist
        nb = self.message_bytes(cap)
        world = dist.get_world_size(group)
        recv = self.recv[: world * nb]
        dist.all_gather_into_tensor(recv, self.send[:nb], group=group)
        return self.apply_packed(it, recv, world, cap)

    def message_bytes(self, cap: int) -> int:
        return int(self._lib.load().wg_exchange_bytes(cap, self.val_type))

    def apply_packed(self, it: int, recv, world: int, cap: int):
        """Apply gathered messages (world parts of message_bytes(cap) bytes)."""
        L = self._lib.load()
        self._lib.check(L.wg_exchange_apply_all(ctypes.byref(self.g.struct()), ctypes.byref(self.loop.bufs),
                                                ctypes.byref(self.p), it, recv.data_ptr(), world, cap,
                                                self.status.data_ptr(), self._lib.stream_ptr()))
        self.host_status.copy_(self.status, non_blocking=True)
        rec, _ = self._record(it, raise_overflow=False)  # synchronises
        if int(self.host_status[1]):  # every rank's message carries its overflow flag
            raise self._lib.OverflowError32(self._lib.WG_EOVERFLOW, "uint32 overflow in sharded loop (some rank)")
        return rec, int(self.host_status[0])

    def step_pairs(self, it: int):
        """Variable-size form (wg_exchange_pack): the local iteration and its
        (vertex, value) pairs, for callers that exchange them themselves."""
        L = self._lib.load()
        self.loop.enqueue(self.p, it, 1)
        cnt = ctypes.c_uint64(0)
        self._lib.check(L.wg_exchange_pack(ctypes.byref(self.g.struct()), ctypes.byref(self.loop.bufs),
                                           ctypes.byref(self.p), it, self.out_v.data_ptr(),
                                           self.out_x.data_ptr(), self.out_v.numel(), ctypes.byref(cnt),
                                           self._lib.stream_ptr()))
        k = int(cnt.value)
        return self.out_v[:k], self.out_x[:k]

    def apply(self, it: int, verts, vals) -> ShardRecord:
        L = self._lib.load()
        self._lib.check(L.wg_exchange_apply(ctypes.byref(self.g.struct()), ctypes.byref(self.loop.bufs),
                                            ctypes.byref(self.p), it, verts.data_ptr() if verts.numel() else None,
                                            vals.data_ptr() if vals.numel() else None, int(verts.numel()),
                                            self._lib.stream_ptr()))
        return self._record(it)

    def _record(self, it: int, raise_overflow: bool = True):
        r = self.loop._read(it, 1)[0]
        ovf = bool(int(r[10]))
        if ovf and raise_overflow:
            raise self._lib.OverflowError32(self._lib.WG_EOVERFLOW, "uint32 overflow in sharded loop")
        mode = {1: "FullScan", 2: "Wedge"}.get(int(r[0]), "None")
        rec = ShardRecord(it, mode, int(r[1]), int(r[2]), int(r[3]), int(r[4]),
                          int(r[7]) if mode == "Wedge" else 0, int(r[8]) if mode == "Wedge" else 0)
        return rec if raise_overflow else (rec, ovf)

    def values_int64(self) -> np.ndarray:
        # after wg_exchange_apply both value buffers hold the global state
        if getattr(self, "_last", None) is not None:  # run_alone: the last iteration's buffer
            return self.dv.values_to_int64(self.loop.values_after(self._last), self.val_type)
        return self.dv.values_to_int64(self.loop.vals[0], self.val_type)


def run_sharded_device(n: int, src, dst, weight, width: int, program, config, group=None):
    """Device entry point: run a MinPlusKernel program over destination
    shards (one rank per GPU, torch.distributed initialised by the caller)."""
    import torch
    import torch.distributed as dist
    from . import _lib
    from .engine import _initial_members, _initial_values
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    d = torch.as_tensor(np.asarray(dst) if not isinstance(dst, torch.Tensor) else dst)
    indeg = torch.bincount(d.to(torch.int64).cuda() & 0xFFFFFFFF, minlength=n).cpu().numpy()
    bounds = destination_bounds(indeg, width, world)
    init = _initial_values(program, n)
    members = _initial_members(program, n)
    from . import device as dv
    val_type = _lib.WG_VAL_U32 if dv.fits_u32(init, program.kernel, None) else _lib.WG_VAL_I64
    while True:
        shard = DeviceShard(n, src, dst, weight, width, bounds, rank, program.kernel, init, members,
                            config.threshold.fraction, config.precision.shift, val_type)
        try:
            return run_sharded(shard, config.max_iterations, group)
        except _lib.OverflowError32:
            # every rank saw the flag in the same exchange: all restart exactly in int64
            if val_type == _lib.WG_VAL_I64:
                raise
            val_type = _lib.WG_VAL_I64


# ---------------------------------------------------------------------------
# PageRank over destination shards ("PR: allgather of rank (or
# contrib) slices")
# ---------------------------------------------------------------------------
def run_pagerank_sharded(shard, iterations: int, group=None):
    """Per iteration: every rank applies the previous sums to the full rank
    vector and builds the contributions (replicated, V-sized), pulls its own
    destinations, and one all-gather of the padded per-rank sum slices
    rebuilds the full sum vector on every rank.  The dangling mass needs no
    collective: each rank derives it from the replicated ranks."""
    import torch.distributed as dist
    if dist.get_world_size(group) == 1 and hasattr(shard, "run_alone"):
        return shard.run_alone(iterations)  # one rank: the single-GPU PageRank (hot-source layout)
    for it in range(iterations):
        shard.prep(it)
        part = shard.pull()
        dist.all_gather_into_tensor(shard.gathered, part, group=group)
        shard.unpack()
    return shard.finish(iterations)


class DevicePageRankShard:
    """One rank's PageRank shard: its destinations' vectors, the global
    out-degrees, replicated float32 sums/contributions, and the padded slice
    buffers of the all-gather (slot r*S holds rank r's destinations)."""

    device = "cuda"

    def __init__(self, n: int, src, dst, width: int, bounds: list[int], rank: int, damping: float = 0.85):
        import torch
        from . import device as dv
        from . import _lib
        self._lib = _lib
        lo, hi = bounds[rank], bounds[rank + 1]
        s = dv.to_dev_u32(src)
        d = dv.to_dev_u32(dst)
        d64 = d.to(torch.int64) & 0xFFFFFFFF
        mask = (d64 >= lo) & (d64 < hi)
        self.outdeg = torch.bincount(s.to(torch.int64) & 0xFFFFFFFF, minlength=n).to(torch.int32)
        self.g = dv.DeviceGraph.build(n, s[mask], d[mask], None, width)
        self.n, self.lo, self.hi, self.rank, self.bounds = n, lo, hi, rank, list(bounds)
        self.damping = float(damping)
        world = len(bounds) - 1
        self.S = max(max(bounds[r + 1] - bounds[r] for r in range(world)), 1)
        f32 = dict(dtype=torch.float32, device="cuda")
        self.acc = torch.zeros(n, **f32)
        self.contrib = torch.empty(n, **f32)
        self.rank_out = torch.empty(n, **f32)
        self.scal = torch.zeros(4, dtype=torch.float64, device="cuda")
        self.part = torch.zeros(self.S, **f32)
        self.gathered = torch.empty(world * self.S, **f32)
        L = _lib.load()
        self.ws = torch.empty(max(int(L.wg_pagerank_prep_ws_bytes(n)),
                                  int(L.wg_pagerank_ws_bytes(ctypes.byref(self.g.struct())))),
                              dtype=torch.uint8, device="cuda")

    def prep(self, it: int, rank_out=None):
        L = self._lib.load()
        self._lib.check(L.wg_pagerank_prep(self.n, it, self.damping, self.outdeg.data_ptr(), self.acc.data_ptr(),
                                           self.contrib.data_ptr(),
                                           rank_out.data_ptr() if rank_out is not None else None,
                                           self.scal.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                           self._lib.stream_ptr()))

    def pull(self):
        L = self._lib.load()
        self.part.zero_()
        self._lib.check(L.wg_pagerank_pull(ctypes.byref(self.g.struct()), self.contrib.data_ptr(),
                                           self.part.data_ptr(), self.lo, self.ws.data_ptr(), self.ws.numel(),
                                           self._lib.stream_ptr()))
        return self.part

    def unpack(self):
        for r in range(len(self.bounds) - 1):
            lo, hi = self.bounds[r], self.bounds[r + 1]
            if hi > lo:
                self.acc[lo:hi].copy_(self.gathered[r * self.S: r * self.S + hi - lo])

    def finish(self, iterations: int):
        self.prep(iterations, self.rank_out)
        return self.rank_out

    def run_alone(self, iterations: int):
        """World size 1: this shard holds every destination, so the whole run
        is device.pagerank on its graph (with the global out-degrees)."""
        from . import device as dv
        g = getattr(self, "_whole", None)
        if g is None:
            l = self.g
            g = self._whole = dv.DeviceGraph(self.n, l.width, l.edges, l.nvec, l.entries, l.vsrc, l.vdst, l.vw,
                                             l.idx_off, l.idx_pos, self.outdeg, lens_are_degrees=l.lens_are_degrees)
        bufs = (self.rank_out, self.acc, self.contrib, self.scal)
        return dv.pagerank(g, iterations, self.damping, bufs=bufs)


def run_pagerank_sharded_device(n: int, src, dst, width: int = 4, iterations: int = 20, damping: float = 0.85,
                                group=None):
    """Device entry point (one rank per GPU, torch.distributed initialised by
    the caller): float32 ranks of all n vertices on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    from . import device as dv
    d = dv.to_dev_u32(dst)
    indeg = torch.bincount(d.to(torch.int64) & 0xFFFFFFFF, minlength=n).cpu().numpy()
    bounds = destination_bounds(indeg, width, world)
    shard = DevicePageRankShard(n, src, dst, width, bounds, rank, damping)
    return run_pagerank_sharded(shard, iterations, group)
