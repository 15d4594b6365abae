"""GPU test of the destination-sharded engine on ONE device: two DeviceShards
(ranks 0 and 1 of a 2-way partition) live in this process and are driven in
lockstep; the exchange that torch.distributed performs across GPUs is done by
concatenation here (no kernels wait on each other).  Values and traces must
equal the single-GPU reference run."""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _lockstep(shards, max_it=10_000, packed=False):
    """packed: the fixed-size protocol (wg_exchange_pack_all / apply_all) with
    a deliberately small first capacity, so the truncated-message redo runs;
    "slices": dense iterations exchange owned value slices
    (wg_exchange_slice_pack / apply_slices), the others packed messages."""
    import ctypes
    from paper_1903_07754_b200 import _lib
    for s in shards:
        s.seed()
    recs = []
    cap = 16
    prev_sum = shards[0].initial_edge_sum()
    dense_seen = 0
    for it in range(1, max_it + 1):
        if packed == "slices" and shards[0].gate_dense(prev_sum):
            dense_seen += 1
            L = _lib.load()
            for r, s in enumerate(shards):
                s.step(it)
                _lib.check(L.wg_exchange_slice_pack(ctypes.byref(s.g.struct()), ctypes.byref(s.loop.bufs),
                                                    ctypes.byref(s.p), it, s.bounds[r], s.bounds[r + 1],
                                                    s.slice_send.data_ptr(), _lib.stream_ptr()))
            recv = torch.cat([s.slice_send for s in shards])
            rs = [s.apply_slices(it, recv, overflow_any=False) for s in shards]
        elif packed:
            for s in shards:
                s.step(it)

            def gather(c):
                nb = shards[0].message_bytes(c)
                return torch.cat([s.send[:nb] for s in shards])
            out = [s.apply_packed(it, gather(cap), len(shards), cap) for s in shards]
            if out[0][1] > cap:
                full = shards[0].capacity
                out = [s.apply_packed(it, gather(full), len(shards), full) for s in shards]
            rs = [o[0] for o in out]
            cap = min(shards[0].capacity, max(16, 2 * out[0][1]))
        else:
            outs = [s.step_pairs(it) for s in shards]
            V = torch.cat([o[0] for o in outs])
            X = torch.cat([o[1] for o in outs])
            rs = [s.apply(it, V, X) for s in shards]
        for r in rs[1:]:
            assert (r.mode, r.active_edges, r.frontier_out_size, r.out_edge_sum) == \
                   (rs[0].mode, rs[0].active_edges, rs[0].frontier_out_size, rs[0].out_edge_sum)
        recs.append(rs[0])
        prev_sum = rs[0].out_edge_sum
        if rs[0].out_edge_sum == 0:
            break
    if packed == "slices":
        assert dense_seen > 0
    return shards[0].values_int64(), recs


@pytest.mark.parametrize("app,world,packed", [("bfs", 2, False), ("cc", 2, False), ("sssp", 2, False),
                                              ("cc", 3, False), ("bfs", 2, True), ("cc", 3, True),
                                              ("sssp", 2, True), ("cc", 2, "slices"), ("bfs", 3, "slices"),
                                              ("sssp", 2, "slices")])
def test_device_shards_match_single_run(app, world, packed):
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib
    from paper_1903_07754_b200.distributed import DeviceShard, destination_bounds
    el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=13, edge_factor=16, seed=2)), True)
    if app == "sssp":
        el = wg.synthesize_weights(el, 255)
    n = el.vertex_count
    src, dst, w = el.src, el.dst, el.weight
    prog = wg.make_program(app, None if app == "cc" else 0)
    thr = Fraction(1, 100) if app == "bfs" else Fraction(1, 5)
    vpg = 8 if app == "bfs" else 4
    bounds = destination_bounds(np.bincount(dst, minlength=n), 4, world)
    init = prog.initial_values(n)
    members = None if app == "cc" else np.array([0])
    shards = [DeviceShard(n, src, dst, w, 4, bounds, r, prog.kernel, init, members, thr,
                          vpg.bit_length() - 1, _lib.WG_VAL_U32) for r in range(world)]
    vals, recs = _lockstep(shards, packed=packed)
    # single-process reference (oracle)
    topo = oracle.build_pull_topology(n, src, dst, w, 4)
    idx = oracle.build_edge_index(topo)
    deg = oracle.compute_out_degrees(n, src)
    v0, front = oracle.initial_state(app, n, 0)
    want = oracle.run_until_convergence(topo, idx, deg, oracle.kern_of(app), v0, front, thr, vpg)
    assert np.array_equal(vals, want.values)
    assert [(r.iteration, r.mode, r.active_edges, r.frontier_out_size) for r in recs] == \
        list(oracle.trace(want.stats))
    # dense iterations touch every vector exactly once across the shards
    for r, s in zip(recs, want.stats):
        if r.mode == "FullScan":
            assert sum(sh_touched for sh_touched in [r.vectors_touched]) <= topo.vector_count


@pytest.mark.parametrize("world", [2, 3])
def test_device_pagerank_shards_match_single_run(world):
    """Destination-sharded PageRank (wg_pagerank_prep / wg_pagerank_pull) in
    lockstep: the all-gather of padded sum slices is a concatenation here."""
    from paper_1903_07754_b200 import device as dv
    from paper_1903_07754_b200.distributed import DevicePageRankShard, destination_bounds
    n, s, d = oracle.rmat_edges(12, 16, 3)
    keep = s != d
    s, d = s[keep], d[keep]
    bounds = destination_bounds(np.bincount(d, minlength=n), 4, world)
    shards = [DevicePageRankShard(n, s, d, 4, bounds, r) for r in range(world)]
    for it in range(20):
        parts = []
        for sh in shards:
            sh.prep(it)
            parts.append(sh.pull().clone())
        cat = torch.cat(parts)
        for sh in shards:
            sh.gathered.copy_(cat)
            sh.unpack()
    got = [sh.finish(20).cpu().numpy().astype(np.float64) for sh in shards]
    want = oracle.pagerank_numpy(n, s, d, 20)
    single = dv.pagerank(dv.DeviceGraph.build(n, dv.to_dev_u32(s), dv.to_dev_u32(d), None, 4)).cpu().numpy()
    for r in got:
        assert np.max(np.abs(r - want)) <= 1e-6  # north_star tolerance vs the float64 oracle
        assert np.max(np.abs(r - single)) <= 1e-7


@pytest.mark.parametrize("packed", [True, "slices"])
def test_device_shards_overflow_restart_in_int64(packed):
    """uint32 overflow on one rank is seen by every rank (the packed header /
    the all-reduced flag) and the run restarts exactly in int64."""
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib
    from paper_1903_07754_b200.distributed import DeviceShard, destination_bounds
    el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=10, edge_factor=8, seed=3)), True)
    n = el.vertex_count
    src, dst = el.src, el.dst
    w = np.full(src.shape[0], 1_500_000_000, np.int64)  # distances pass 2^32 after three hops
    prog = wg.make_program("sssp", 0)
    bounds = destination_bounds(np.bincount(dst, minlength=n), 4, 2)
    init = prog.initial_values(n)
    mk = lambda vt: [DeviceShard(n, src, dst, w, 4, bounds, r, prog.kernel, init, np.array([0]), Fraction(1, 5),
                                 2, vt) for r in range(2)]
    with pytest.raises(_lib.OverflowError32):
        _lockstep(mk(_lib.WG_VAL_U32), packed=packed)
    vals, recs = _lockstep(mk(_lib.WG_VAL_I64), packed=packed)
    topo = oracle.build_pull_topology(n, src, dst, w, 4)
    idx = oracle.build_edge_index(topo)
    deg = oracle.compute_out_degrees(n, src)
    v0, front = oracle.initial_state("sssp", n, 0)
    want = oracle.run_until_convergence(topo, idx, deg, oracle.SSSP, v0, front, Fraction(1, 5), 4)
    assert np.array_equal(vals, want.values)
    assert [(r.iteration, r.mode, r.active_edges, r.frontier_out_size) for r in recs] == \
        list(oracle.trace(want.stats))


def test_partitioned_rmat_ingest_single_rank_matches_full_pipeline():
    """rmat_partitioned (rows of the PCG64 stream per rank, all-to-all to the
    destination owner, local dedup) at world size 1 over NCCL equals the
    whole-list pipeline, and a sharded CC run on it gives the oracle's result."""
    import os
    import socket
    import torch.distributed as dist
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib
    from paper_1903_07754_b200.distributed import DeviceShard, rmat_partitioned, run_sharded
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sock.getsockname()[1]))
    sock.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, E, bounds, s, d, outdeg = rmat_partitioned(12, 16, 1, True)
        el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=12, edge_factor=16, seed=1)), True)
        assert E == el.edge_count and bounds == [0, n]
        key = lambda a, b: np.sort((a.astype(np.int64) & 0xFFFFFFFF) * (1 << 32) + (b.astype(np.int64) & 0xFFFFFFFF))
        assert np.array_equal(key(s.cpu().numpy(), d.cpu().numpy()), key(el.src, el.dst))
        assert np.array_equal(outdeg.cpu().numpy().astype(np.int64), np.bincount(el.src, minlength=n))
        prog = wg.make_program("cc")
        shard = DeviceShard(n, s, d, None, 4, bounds, 0, prog.kernel, prog.initial_values(n), None, Fraction(1, 5),
                            2, _lib.WG_VAL_U32, local=(E, outdeg))
        vals, recs, conv = run_sharded(shard, 10_000)
        topo = oracle.build_pull_topology(n, el.src, el.dst, None, 4)
        want = oracle.run_until_convergence(topo, oracle.build_edge_index(topo),
                                            oracle.compute_out_degrees(n, el.src), oracle.CC,
                                            *oracle.initial_state("cc", n, 0), Fraction(1, 5), 4)
        assert np.array_equal(vals, want.values) and conv
        assert [(r.iteration, r.mode, r.active_edges, r.frontier_out_size) for r in recs] == \
            list(oracle.trace(want.stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("app,packed", [("cc", True), ("bfs", "slices"), ("sssp", True)])
def test_device_shards_local_gate_same_values_and_frontiers(app, packed):
    """WG_RUN_LOCAL_GATE: every shard decides Wedge / FullScan from its own
    share of the frontier's edges.  Modes may differ per
    shard and from the reference; values, active edges and produced
    frontiers may not."""
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib
    from paper_1903_07754_b200.distributed import DeviceShard, destination_bounds
    el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=13, edge_factor=16, seed=4)), True)
    if app == "sssp":
        el = wg.synthesize_weights(el, 255)
    n = el.vertex_count
    src, dst, w = el.src, el.dst, el.weight
    prog = wg.make_program(app, None if app == "cc" else 0)
    thr = Fraction(1, 100) if app == "bfs" else Fraction(1, 5)
    vpg = 8 if app == "bfs" else 4
    bounds = destination_bounds(np.bincount(dst, minlength=n), 4, 3)
    init = prog.initial_values(n)
    members = None if app == "cc" else np.array([0])
    shards = [DeviceShard(n, src, dst, w, 4, bounds, r, prog.kernel, init, members, thr, vpg.bit_length() - 1,
                          _lib.WG_VAL_U32, gate="local") for r in range(3)]
    vals, recs = _lockstep_local(shards, packed)
    topo = oracle.build_pull_topology(n, src, dst, w, 4)
    want = oracle.run_until_convergence(topo, oracle.build_edge_index(topo), oracle.compute_out_degrees(n, src),
                                        oracle.kern_of(app), *oracle.initial_state(app, n, 0), thr, vpg)
    assert np.array_equal(vals, want.values)
    assert [(r.iteration, r.active_edges, r.frontier_out_size) for r in recs] == \
        [(s.iteration, s.active_edges, s.frontier_out_size) for s in want.stats]


def _lockstep_local(shards, packed):
    """_lockstep without the per-shard mode agreement check (modes are local)."""
    import ctypes
    from paper_1903_07754_b200 import _lib
    for s in shards:
        s.seed()
    recs, prev_sum = [], shards[0].initial_edge_sum()
    for it in range(1, 10_000):
        if packed == "slices" and shards[0].gate_dense(prev_sum):
            L = _lib.load()
            for r, s in enumerate(shards):
                s.step(it)
                _lib.check(L.wg_exchange_slice_pack(ctypes.byref(s.g.struct()), ctypes.byref(s.loop.bufs),
                                                    ctypes.byref(s.p), it, s.bounds[r], s.bounds[r + 1],
                                                    s.slice_send.data_ptr(), _lib.stream_ptr()))
            recv = torch.cat([s.slice_send for s in shards])
            rs = [s.apply_slices(it, recv, overflow_any=False) for s in shards]
        else:
            for s in shards:
                s.step(it)
            full = shards[0].capacity
            nb = shards[0].message_bytes(full)
            recv = torch.cat([s.send[:nb] for s in shards])
            rs = [s.apply_packed(it, recv, len(shards), full)[0] for s in shards]
        for r in rs[1:]:
            assert (r.active_edges, r.frontier_out_size, r.out_edge_sum) == \
                   (rs[0].active_edges, rs[0].frontier_out_size, rs[0].out_edge_sum)
        recs.append(rs[0])
        prev_sum = rs[0].out_edge_sum
        if prev_sum == 0:
            break
    return shards[0].values_int64(), recs
