"""GPU parity: the sm_100a kernels behind the C ABI against the reference's
own outputs (golden fixtures) and the CPU oracle.  Bit-exact for every
integer result.  Marked gpu."""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import GT_EDGES, GT_VERTICES

pytestmark = pytest.mark.gpu

UNREACHED = oracle.UNREACHED


@pytest.fixture(scope="module")
def wg():
    import paper_1903_07754_b200 as wg
    return wg


def _graph(wg, n, src, dst, w, width):
    return wg.build_pull_topology(wg.EdgeList(n, src, dst, w), width)


# --------------------------------------------------------------- layout ---
def test_device_layout_matches_reference(wg, golden):
    z = golden.npz("layout")
    for c in golden.meta("layout"):
        nm = c["name"]
        w = z[f"{nm}/w"] if c["weighted"] else None
        topo = _graph(wg, c["n"], z[f"{nm}/src"], z[f"{nm}/dst"], w, c["width"])
        assert np.array_equal(topo.vec_dst, z[f"{nm}/vec_dst"]), nm
        assert np.array_equal(topo.lane_src, z[f"{nm}/lane_src"]), nm
        assert np.array_equal(topo.lane_count, z[f"{nm}/lane_count"]), nm
        if c["weighted"]:
            assert np.array_equal(topo.lane_weight, z[f"{nm}/lane_weight"]), nm
        idx = wg.build_edge_index(topo)
        assert np.array_equal(idx.offsets, z[f"{nm}/offsets"]), nm
        assert np.array_equal(idx.positions, z[f"{nm}/positions"]), nm
        assert np.array_equal(topo.device.outdeg_np(), z[f"{nm}/degrees"]), nm


def test_device_layout_edge_cases(wg):
    # empty graph, isolated vertices, all edges into one hub (multi-warp run)
    t = _graph(wg, 3, [], [], None, 4)
    assert t.vector_count == 0 and wg.build_edge_index(t).offsets.tolist() == [0, 0, 0, 0]
    hub = 5000
    src = np.arange(1, hub + 1)
    dst = np.zeros(hub, np.int64)
    t = _graph(wg, hub + 1, src, dst, None, 4)
    ref = oracle.build_pull_topology(hub + 1, src, dst, None, 4)
    assert np.array_equal(t.vec_dst, ref.vec_dst) and np.array_equal(t.lane_src, ref.lane_src)
    # duplicates and self-loops are processed like any edge (graph.py:36-41)
    src = [0, 0, 1, 1, 2, 2, 2]
    dst = [1, 1, 1, 2, 2, 0, 0]
    t = _graph(wg, 3, src, dst, [5, 3, 1, 1, 1, 2, 7], 2)
    ref = oracle.build_pull_topology(3, src, dst, [5, 3, 1, 1, 1, 2, 7], 2)
    assert np.array_equal(t.lane_weight, ref.lane_weight) and np.array_equal(t.lane_src, ref.lane_src)
    ri = oracle.build_edge_index(ref)
    assert np.array_equal(wg.build_edge_index(t).positions, ri.positions)


def _pack_np(lanes, bits):
    """The packed-lane format restated (wedge_b200.h wg_pack_lanes): lane l in
    bits [l*bits, (l+1)*bits) of a little-endian bit stream, empty = all ones."""
    mask = (1 << bits) - 1
    v = lanes.astype(np.uint64) & mask
    stream = np.zeros(len(lanes) * bits, dtype=np.uint8)
    for b in range(bits):
        stream[b::bits] = (v >> np.uint64(b)) & np.uint64(1)
    pad = (-len(stream)) % 32
    stream = np.concatenate([stream, np.zeros(pad, np.uint8)])
    return np.packbits(stream.reshape(-1, 32)[:, ::-1], axis=1).view(">u4").ravel().astype(np.uint32)


def _sorted_lists(off, pos):
    out = pos.copy()
    for a, b in zip(off[:-1], off[1:]):
        out[a:b].sort()
    return out


def _decode_np(h, vdst, W, BV=1024):
    """The delta-coded lane format restated (wedge_b200.h wg_encode_lanes),
    decoded sequentially on the host."""
    words = h["lane_stream"].numpy().view(np.uint32)
    wbits = np.unpackbits(h["lane_widths"].numpy().view(np.uint8), bitorder="little")
    nvec = len(vdst)
    widths = np.array([1 + int(np.dot(wbits[(v // BV) * 5120 + (v % BV) * 5:][:5].astype(np.int64),
                                      1 << np.arange(5))) for v in range(nvec)])
    base = h["lane_blocks"].numpy()
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")
    out = np.empty(len(widths) * W, np.uint32)
    pos = 0
    prev = 0
    for v in range(len(widths)):
        if v % BV == 0:
            pos = int(base[v // BV])
        head = v % BV == 0 or vdst[v] != vdst[v - 1]
        w = int(widths[v])
        for j in range(W):
            c = int(np.dot(bits[pos: pos + w].astype(np.int64), 1 << np.arange(w, dtype=np.int64)))
            pos += w
            if c == 0:
                out[v * W + j] = 0xFFFFFFFF
                continue
            prev = c - 1 if (head and j == 0) else prev + c - 1
            out[v * W + j] = prev
    return out


def test_layout_rebuilt_from_lanes(wg, golden):
    """wg_expand_destinations + wg_build_index (the e2e upload form: lanes and
    per-destination vector offsets only) reproduce vec_dst, the edge index
    and the out-degrees of the full builder, duplicates included."""
    import torch
    from paper_1903_07754_b200 import device as dv
    z = golden.npz("layout")
    cases = [(c["n"], z[f"{c['name']}/src"], z[f"{c['name']}/dst"], c["width"]) for c in golden.meta("layout")]
    cases.append((3, [0, 0, 1, 1, 2, 2, 2], [1, 1, 1, 2, 2, 0, 0], 2))
    el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=12, edge_factor=8, seed=3)), True)
    cases.append((el.vertex_count, el.src, el.dst, 4))
    for n, src, dst, width in cases:
        g = _graph(wg, n, src, dst, None, width).device
        if g.nvec == 0:
            continue
        vs = torch.empty(g.vsrc.numel() + 64, dtype=torch.int32, device="cuda")[: g.vsrc.numel()]
        vs.copy_(g.vsrc)
        g2 = dv.DeviceGraph.from_lanes(g.n, g.width, g.edges, g.nvec, vs, None, g.vector_offsets())
        assert g2.entries == g.entries
        # the pipelined form (chunked index, falls back on parallel edges)
        host = {"vsrc": g.vsrc.cpu().pin_memory(), "voff": g.vector_offsets().cpu().pin_memory()}
        g2.vdst.zero_()
        g2.idx_pos.zero_()
        for chunks in (1, 3):
            assert g2.upload_rebuild(host, {"vsrc": g2.vsrc, "voff": torch.empty_like(host["voff"], device="cuda")},
                                     chunks=chunks) == g.entries
            assert np.array_equal(g2.vec_dst_np(), g.vec_dst_np())
            assert np.array_equal(g2.offsets_np(), g.offsets_np())
            assert np.array_equal(g2.positions_np(), g.positions_np())
            assert np.array_equal(g2.outdeg_np(), g.outdeg_np())
        # the bit-packed upload (lanes unpacked chunk by chunk)
        words, bits = g.pack_lanes()
        assert np.array_equal(words.cpu().numpy().view(np.uint32), _pack_np(g.vsrc.cpu().numpy().view(np.uint32), bits))
        hp = {"vsrc_bits": words.cpu().pin_memory(), "voff": host["voff"]}
        for chunks in (1, 3, 7):
            g2.vsrc.fill_(-7)
            g2.idx_pos.zero_()
            dp = {"vsrc_bits": torch.empty(words.numel() + 1, dtype=torch.int32, device="cuda")[: words.numel()],
                  "voff": torch.empty_like(host["voff"], device="cuda")}
            assert g2.upload_rebuild(hp, dp, chunks=chunks) == g.entries
            assert torch.equal(g2.vsrc, g.vsrc)
            assert np.array_equal(g2.positions_np(), g.positions_np())
        # the delta-coded upload (blocks decoded chunk by chunk)
        enc = g.encode_lanes()
        hc = {k: v.cpu().pin_memory() for k, v in enc.items()}
        hc["voff"] = host["voff"]
        assert _decode_np(hc, g.vec_dst_np(), g.width).tobytes() == g.vsrc.cpu().numpy().tobytes()
        for chunks, counted in ((1, False), (2, False), (5, False), (1, True), (3, True)):
            g2.vsrc.fill_(-7)
            g2.idx_pos.zero_()
            g2.outdeg.zero_()
            h = dict(hc, outdeg=g.outdeg[: g.n].cpu().pin_memory()) if counted else hc
            dc = {k: torch.empty(v.numel() + 1, dtype=v.dtype, device="cuda")[: v.numel()] for k, v in h.items()}
            # placed (degrees given): same lists up to their order; parallel
            # edges make it fall back to the sorted builder
            assert g2.upload_rebuild(h, dc, chunks=chunks) == g.entries
            assert torch.equal(g2.vsrc, g.vsrc)
            assert np.array_equal(g2.offsets_np(), g.offsets_np())
            assert np.array_equal(g2.outdeg_np(), g.outdeg_np())
            if counted:  # same lists, order inside each list unspecified
                assert np.array_equal(_sorted_lists(g2.offsets_np(), g2.positions_np()), g.positions_np())
            else:
                assert np.array_equal(g2.positions_np(), g.positions_np())
        # the compact host format: degrees as bytes + large ones, voff rebuilt
        # from the in-degrees; a symmetric claim ships no out-degrees (a false
        # claim fails the placement check and falls back to the sorted build)
        for sym in (False, True):
            hf = g.host_format(symmetric=sym)
            df = {k: torch.empty(v.numel() + 1, dtype=v.dtype, device="cuda")[: v.numel()].view(v.shape)
                  for k, v in hf.items()}
            g2.vsrc.fill_(-7)
            g2.vdst.fill_(-7)
            g2.idx_pos.zero_()
            g2.outdeg.zero_()
            assert g2.upload_rebuild(hf, df, chunks=3, outdeg_is_indeg=sym) == g.entries
            assert torch.equal(g2.vsrc, g.vsrc) and np.array_equal(g2.vec_dst_np(), g.vec_dst_np())
            assert np.array_equal(g2.offsets_np(), g.offsets_np())
            assert np.array_equal(g2.outdeg_np(), g.outdeg_np())
            assert np.array_equal(_sorted_lists(g2.offsets_np(), g2.positions_np()), g.positions_np())
        # placed over raw uint32 lanes too
        g2.idx_pos.zero_()
        assert g2.upload_rebuild(dict(host, outdeg=g.outdeg[: g.n].cpu().pin_memory()),
                                 {"vsrc": g2.vsrc, "voff": torch.empty_like(host["voff"], device="cuda")},
                                 chunks=2) == g.entries
        assert np.array_equal(_sorted_lists(g2.offsets_np(), g2.positions_np()), g.positions_np())
        assert np.array_equal(g2.vec_dst_np(), g.vec_dst_np())
        assert np.array_equal(g2.offsets_np(), g.offsets_np())
        assert np.array_equal(g2.outdeg_np(), g.outdeg_np())
        assert g2.lens_are_degrees == g.lens_are_degrees


# ------------------------------------------------- backend protocol (Tier 1)
@pytest.mark.parametrize("kind", ["pull_full", "pull_wedge", "transform"])
def test_backend_protocol_bit_exact(wg, golden, kind):
    """Every golden case of pkg/tests/test_kernels_backends.py:24-94 style,
    through B200Backend on a reference-layout topology (as the unmodified
    reference engine would call it)."""
    be = wg.B200Backend()
    for c in (c for c in golden.meta("kernels") if c["kind"] == kind):
        g = golden.kernel_case(c)
        n, width = c["n"], c["width"]
        topo = oracle.build_pull_topology(n, g["src"], g["dst"], g["w"], width)
        if kind == "transform":
            idx = oracle.build_edge_index(topo)
            ww = np.zeros_like(g["wedge"])
            v = be.transform(g["frontier"], n, idx.offsets, idx.positions, c["shift"], ww, 16, 1)
            assert v == c["visited"], c["id"]
            assert np.array_equal(ww, g["wedge"]), c["id"]
            continue
        kern = oracle.kern_of(c["app"])
        prev = g["prev"].copy()
        nxt = prev.copy()
        out = np.zeros_like(g["out"])
        if kind == "pull_full":
            t = be.pull_full(topo, prev, nxt, out, kern, UNREACHED, 1)
        else:
            t = be.pull_wedge(topo, g["wedge"], c["shift"], c["groups"], prev, nxt, out, kern, UNREACHED, 1)
        assert t == c["touched"], c["id"]
        assert np.array_equal(nxt, g["nxt"]), c["id"]
        assert np.array_equal(out, g["out"]), c["id"]


def test_backend_protocol_random_states_vs_oracle(wg):
    """Larger random graphs and states: B200Backend == oracle, all W, shifts."""
    be = wg.B200Backend()
    port = oracle.PortBackend(4)
    rng = np.random.default_rng(123)
    for trial in range(6):
        n = int(rng.integers(500, 5000))
        m = int(rng.integers(1000, 60000))
        src = rng.integers(0, n, m)
        dst = np.minimum((rng.pareto(0.8, m) * 5).astype(np.int64), n - 1) if trial % 2 else rng.integers(0, n, m)
        w = rng.integers(1, 1000, m)
        for width in (1, 2, 4, 8):
            topo = oracle.build_pull_topology(n, src, dst, w, width)
            idx = oracle.build_edge_index(topo)
            for app in ("bfs", "cc", "sssp"):
                kern = oracle.kern_of(app)
                prev = rng.integers(0, n + 2, n).astype(np.int64)
                prev[rng.random(n) < 0.3] = UNREACHED
                a_n, b_n = prev.copy(), prev.copy()
                a_o = np.zeros((n + 63) // 64, np.uint64)
                b_o = a_o.copy()
                ta = be.pull_full(topo, prev, a_n, a_o, kern, UNREACHED)
                tb = port.pull_full(topo, prev, b_n, b_o, kern, UNREACHED)
                assert ta == tb and np.array_equal(a_n, b_n) and np.array_equal(a_o, b_o)
                for shift in (0, 2, 3):
                    groups = (topo.vector_count + (1 << shift) - 1) >> shift
                    ww = np.zeros((groups + 63) // 64, np.uint64)
                    members = rng.choice(n, size=int(rng.integers(1, n // 4 + 2)), replace=False)
                    fw = np.zeros((n + 63) // 64, np.uint64)
                    oracle.set_bits(fw, members)
                    ww2 = ww.copy()
                    va = be.transform(fw, n, idx.offsets, idx.positions, shift, ww, 4096, 1)
                    vb = port.transform(fw, n, idx.offsets, idx.positions, shift, ww2, 4096, 1)
                    assert va == vb and np.array_equal(ww, ww2)
                    a_n, b_n = prev.copy(), prev.copy()
                    a_o[:] = 0
                    b_o[:] = 0
                    ta = be.pull_wedge(topo, ww, shift, groups, prev, a_n, a_o, kern, UNREACHED)
                    tb = port.pull_wedge(topo, ww, shift, groups, prev, b_n, b_o, kern, UNREACHED)
                    assert ta == tb and np.array_equal(a_n, b_n) and np.array_equal(a_o, b_o)


# ------------------------------------------------------ engine (Tier 2) ---
def _prep(wg, scale, app, width):
    el = wg.generate(wg.GenSpec("rmat", scale=scale, edge_factor=16, seed=1))
    el = wg.drop_self_loops_dedup(el, symmetric=True)
    if app == "sssp":
        el = wg.synthesize_weights(el, 255)
    topo = wg.build_pull_topology(el, width)
    return el, topo, wg.build_edge_index(topo), wg.compute_out_degrees(el)


def test_device_loop_matches_reference_runs(wg, golden):
    """Digest + every per-iteration stat (incl. work counters at equal W/vpg)
    + per-iteration frontiers, for all golden runs (RMAT s8-s12)."""
    zr = golden.npz("runs")
    cache = {}
    for r in golden.meta("runs"):
        key = (r["scale"], r["app"], r["width"])
        if key not in cache:
            cache[key] = _prep(wg, r["scale"], r["app"], r["width"])
        el, topo, idx, deg = cache[key]
        assert el.edge_count == r["E"]
        prog = wg.make_program(r["app"], None if r["app"] == "cc" else r["root"])
        cfg = wg.EngineConfig(threshold=wg.FullnessThreshold(Fraction(*r["thr"])),
                              precision=wg.FrontierPrecision(r["vpg"]), max_iterations=100000)
        flog = [] if r["scale"] <= 10 else None
        res = wg.run_until_convergence(topo, idx, prog, deg, cfg, frontier_log=flog)
        assert wg.result_digest(res.values) == r["digest"], r["name"]
        got = [[s.iteration, s.mode, s.active_edges, s.vectors_touched, s.frontier_out_size,
                s.covered_vectors, s.transform_entries] for s in res.stats]
        assert got == r["stats"], r["name"]
        assert res.converged == r["converged"]
        if flog is not None:
            assert [len(f) for f in flog] == zr[f"{r['name']}/flog_len"].tolist(), r["name"]
            cat = np.concatenate(flog) if flog else np.empty(0, np.int64)
            assert np.array_equal(cat, zr[f"{r['name']}/flog"]), r["name"]


def test_engine_known_answers(wg):
    """pkg/tests/test_engine.py:138-197 known answers on the device loop."""
    def built(edges, n, width=2):
        el = wg.EdgeList.from_pairs(edges, n)
        t = wg.build_pull_topology(el, width)
        return t, wg.build_edge_index(t), wg.compute_out_degrees(el)

    def cfg(threshold="0.2", vpg=1, max_iterations=200):
        return wg.EngineConfig(threshold=wg.FullnessThreshold.of(threshold),
                               precision=wg.FrontierPrecision(vpg), max_iterations=max_iterations)

    t, i, d = built(GT_EDGES, GT_VERTICES)
    r = wg.run_until_convergence(t, i, wg.bfs_program(0), d, cfg(threshold=1, vpg=1))
    assert r.values.tolist() == [0, 1, 1, 2, 3, 4] and r.converged
    assert r.stats[-1].frontier_out_size == 0 and all(s.mode == "Wedge" for s in r.stats)
    t, i, d = built([(0, 1), (1, 0), (2, 3), (3, 2)], 4)
    assert wg.run_until_convergence(t, i, wg.cc_program(), d, cfg()).values.tolist() == [0, 0, 2, 2]
    t, i, d = built([(0, 1, 5), (1, 2, 3)], 3)
    assert wg.run_until_convergence(t, i, wg.sssp_program(0), d, cfg()).values.tolist() == [0, 5, 8]
    t, i, d = built([(0, 1, 1), (0, 2, 4), (1, 2, 1)], 3)
    assert wg.run_until_convergence(t, i, wg.sssp_program(0), d, cfg()).values[2] == 2
    t, i, d = built([(0, 1), (1, 2), (2, 3)], 4)
    r = wg.run_until_convergence(t, i, wg.bfs_program(0), d, cfg(max_iterations=1))
    assert not r.converged and r.iterations == 1
    t, i, d = built([], 1)
    r = wg.run_until_convergence(t, i, wg.bfs_program(0), d, cfg())
    assert r.values.tolist() == [0] and r.iterations == 1 and r.converged
    t, i, d = built([(0, 1)], 2)
    r = wg.run_until_convergence(t, i, wg.bfs_program(1), d, cfg())
    assert r.values.tolist() == [UNREACHED, 0] and r.converged


def test_per_iteration_api_known_answers(wg):
    """pkg/tests/test_engine.py:58-130 through run_iteration_full/wedge."""
    el = wg.EdgeList.from_pairs(GT_EDGES, GT_VERTICES)
    t = wg.build_pull_topology(el, 2)
    i = wg.build_edge_index(t)
    d = wg.compute_out_degrees(el)
    buf = wg.ValueBuffers(np.array([0] + [UNREACHED] * 5), np.array([0] + [UNREACHED] * 5))
    fr, st = wg.run_iteration_full(t, buf, wg.bfs_program(0), d)
    assert buf.next.tolist() == [0, 1, 1, UNREACHED, UNREACHED, UNREACHED]
    assert fr.members().tolist() == [1, 2] and st.vectors_touched == t.vector_count
    buf = wg.ValueBuffers(np.array([0, 1, 1] + [UNREACHED] * 3), np.array([0, 1, 1] + [UNREACHED] * 3))
    _, st = wg.run_iteration_full(t, buf, wg.bfs_program(0), d)
    assert st.vectors_touched == t.vector_count - 2
    wedge = wg.WedgeFrontier.from_groups([0, 1], t.vector_count, wg.FrontierPrecision(1))
    buf = wg.ValueBuffers(np.array([0] + [UNREACHED] * 5), np.array([0] + [UNREACHED] * 5))
    fr, st = wg.run_iteration_wedge(t, wedge, buf, wg.bfs_program(0), d)
    assert buf.next.tolist() == [0, 1, 1, UNREACHED, UNREACHED, UNREACHED] and st.vectors_touched == 2
    f = wg.VertexFrontier.from_vertices([5], d, GT_VERTICES)
    w = wg.transform_frontier(f, i, wg.FrontierPrecision(4))
    assert w.bits.indices().tolist() == [0]
    f = wg.VertexFrontier.from_vertices([1, 2], d, GT_VERTICES)
    w = wg.transform_frontier(f, i, wg.FrontierPrecision(1))
    assert w.bits.indices().tolist() == [2] and w.entries_visited == 2
    f = wg.VertexFrontier.from_vertices([0], d, GT_VERTICES)
    assert wg.transform_frontier(f, i, wg.FrontierPrecision(1)).bits.indices().tolist() == [0, 1]
    assert wg.transform_frontier(f, i, wg.FrontierPrecision(2)).bits.indices().tolist() == [0]
    w = wg.WedgeFrontier.from_groups([2], 5, wg.FrontierPrecision(2))
    assert wg.wedge_covered_vectors(w, 5).tolist() == [4]


def test_generators_bit_identical(wg, golden):
    z = golden.npz("gen")
    el = wg.generate(wg.GenSpec("rmat", scale=8, edge_factor=16, seed=1))
    assert np.array_equal(el.src, z["rmat8_src"]) and np.array_equal(el.dst, z["rmat8_dst"])
    el = wg.generate(wg.GenSpec("rmat", scale=11, edge_factor=4, seed=7))
    assert np.array_equal(el.src, z["rmat11_s7_src"]) and np.array_equal(el.dst, z["rmat11_s7_dst"])
    sym = wg.drop_self_loops_dedup(el, symmetric=True)
    assert np.array_equal(sym.src, z["rmat11_s7_sym_src"]) and np.array_equal(sym.dst, z["rmat11_s7_sym_dst"])
    wt = wg.synthesize_weights(sym, 255)
    assert np.array_equal(wt.weight, z["rmat11_s7_sym_w255"])
    h = wg.synthesize_weights(wg.EdgeList(1 << 26, z["hash_src"], z["hash_dst"]), 1000)
    assert np.array_equal(h.weight, z["hash_w1000"])


def test_grid_generator_matches_oracle(wg):
    el = wg.grid_graph(37, 53, seed=2)
    n, s, d, w = oracle.grid_edges(37, 53, seed=2)
    a = np.lexsort((el.dst, el.src))
    b = np.lexsort((d, s))
    assert np.array_equal(el.src[a], s[b]) and np.array_equal(el.dst[a], d[b])
    assert np.array_equal(el.weight[a], w[b])


def test_pagerank_hot_layout_is_a_stable_degree_order(wg):
    """wg_pagerank_hot_layout: slots = vertices by descending out-degree
    (stable), one slot per vertex with out-edges first; the hot lanes map
    back to the original sources lane for lane; the hot and the plain
    PageRank agree (same lane order -> same sums; only the dangling-mass
    summation order differs) and the hot run is bit-reproducible."""
    from paper_1903_07754_b200 import device as dv
    el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=14, edge_factor=16, seed=3)),
                                  symmetric=False)
    topo = wg.build_pull_topology(el, 4)
    g = topo.device
    n, lanes = g.n, g.nvec * g.width
    lay = dv.PageRankLayout(g)
    order = lay.order.cpu().numpy().view(np.uint32).astype(np.int64)
    od = g.outdeg_np().astype(np.int64)
    assert np.array_equal(np.sort(order), np.arange(n))
    assert lay.nsrc == int((od > 0).sum())
    od_sorted = od[order]
    assert np.all(np.diff(od_sorted) <= 0)
    assert np.all(np.diff(order)[np.diff(od_sorted) == 0] > 0)  # stable: ids ascend within a degree
    assert np.array_equal(lay.od_hot.cpu().numpy().view(np.uint32).astype(np.int64), od_sorted)
    vs = g.vsrc[:lanes].cpu().numpy().view(np.uint32).astype(np.int64)
    vh = lay.vsrc_hot[:lanes].cpu().numpy().view(np.uint32).astype(np.int64)
    real = vs != 0xFFFFFFFF
    assert np.array_equal(vh[~real], vs[~real])
    assert vh[real].max() < lay.nsrc and np.array_equal(order[vh[real]], vs[real])
    a = dv.pagerank(g, 20, 0.85, hot=True).clone()
    b = dv.pagerank(g, 20, 0.85, hot=True).clone()
    c = dv.pagerank(g, 20, 0.85, hot=False).clone()
    assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes()
    assert float((a.double() - c.double()).abs().max()) <= 1e-9
    ref = oracle.pagerank_numpy(el.vertex_count, el.src, el.dst, 20, 0.85)
    assert np.max(np.abs(a.cpu().numpy().astype(np.float64) - ref)) <= 1e-6


def test_pagerank_pull_writes_every_vertex_of_its_range(wg):
    """Gap fill (pagerank.cu): prep no longer clears acc between iterations --
    the pull writes the sum of every vertex up to its last destination,
    in-degree 0 included (zeros between sparse destinations, long runs without
    in-edges), and never a zero over a real sum."""
    import torch
    from paper_1903_07754_b200 import device as dv
    rng = np.random.default_rng(11)
    n = 3000
    # destinations only on multiples of 7 and a long run without in-edges
    dst = rng.choice(np.arange(0, 2000, 7), 12000)
    src = rng.integers(0, n, 12000)
    keep = src != dst
    el = wg.drop_self_loops_dedup(wg.EdgeList(n, src[keep], dst[keep]), symmetric=False)
    topo = wg.build_pull_topology(el, 4)
    g = topo.device
    ref = oracle.pagerank_numpy(el.vertex_count, el.src, el.dst, 20, 0.85)
    for hot in (True, False):
        bufs = (torch.empty(n, dtype=torch.float32, device="cuda"),
                torch.full((n,), 123.0, dtype=torch.float32, device="cuda"),  # poisoned acc
                torch.full((n,), 7.0, dtype=torch.float32, device="cuda"),
                torch.zeros(4, dtype=torch.float64, device="cuda"))
        r = dv.pagerank(g, 20, 0.85, bufs=bufs, hot=hot).cpu().numpy()
        assert np.max(np.abs(r.astype(np.float64) - ref)) <= 1e-6, hot


def test_pagerank_tiny_and_odd_sizes(wg):
    """Edge sizes of the PageRank path: a 5-vertex graph with an isolated
    vertex and a dangling one, and vertex counts that are not multiples of 4
    (scalar tail of the vectorised prep) or of 32."""
    cases = [(5, [0, 1, 2, 3], [1, 2, 0, 0])]
    rng = np.random.default_rng(21)
    for n in (33, 127, 1001):
        m = 6 * n
        cases.append((n, rng.integers(0, n, m), rng.integers(0, max(1, n // 2), m)))
    for n, src, dst in cases:
        src, dst = np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64)
        keep = src != dst
        el = wg.drop_self_loops_dedup(wg.EdgeList(n, src[keep], dst[keep]), symmetric=False)
        topo = wg.build_pull_topology(el, 4)
        r = wg.pagerank(topo, 20, 0.85)
        ref = oracle.pagerank_numpy(el.vertex_count, el.src, el.dst, 20, 0.85)
        assert r.shape == (n,)
        assert np.max(np.abs(r.astype(np.float64) - ref)) <= 1e-6, n


def test_pagerank_within_tolerance(wg):
    """|r_gpu - r_cpu| <= 1e-6 per vertex (north_star), float64 oracle."""
    for scale, ef, seed in ((10, 8, 1), (14, 16, 2)):
        el = wg.generate(wg.GenSpec("rmat", scale=scale, edge_factor=ef, seed=seed))
        el = wg.drop_self_loops_dedup(el, symmetric=False)
        topo = wg.build_pull_topology(el, 4)
        r = wg.pagerank(topo, 20, 0.85)
        ref = oracle.pagerank_numpy(el.vertex_count, el.src, el.dst, 20, 0.85)
        assert np.max(np.abs(r.astype(np.float64) - ref)) <= 1e-6
        assert abs(float(r.astype(np.float64).sum()) - 1.0) < 1e-4


def test_survey_digests_s16(wg):
    """Reference digests frozen in SURVEY §8(c) at RMAT s16 (BFS/CC/SSSP)."""
    want = {"bfs": ("591673cb243fad4e", 5), "cc": ("42bbdb18405bc729", 5), "sssp": ("7d2c2554722fbf74", 11)}
    defaults = {"bfs": (8, "0.01"), "cc": (4, "0.2"), "sssp": (4, "0.2")}
    for app, (dig, iters) in want.items():
        el, topo, idx, deg = _prep(wg, 16, app, 4)
        vpg, thr = defaults[app]
        cfg = wg.EngineConfig(threshold=wg.FullnessThreshold.of(thr), precision=wg.FrontierPrecision(vpg))
        res = wg.run_until_convergence(topo, idx, wg.make_program(app, None if app == "cc" else 0), deg, cfg)
        assert wg.result_digest(res.values) == dig, app
        assert res.iterations == iters, app


def test_u32_overflow_falls_back_exactly(wg):
    """Values beyond uint32 take the exact int64 device path."""
    el = wg.EdgeList(3, [0, 1], [1, 2], [4_000_000_000, 4_000_000_000])
    t = wg.build_pull_topology(el, 4)
    r = wg.run_until_convergence(t, wg.build_edge_index(t), wg.sssp_program(0), wg.compute_out_degrees(el),
                                 wg.EngineConfig())
    assert r.values.tolist() == [0, 4_000_000_000, 8_000_000_000]


def test_bottom_up_levels_follow_the_initial_value(wg):
    """Level-synchronous runs (WG_RUN_FIRST_HIT) with a non-zero common
    initial value and several roots: the bottom-up dense pulls must give
    base + hops, like the oracle's reference loop."""
    import dataclasses
    el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=14, edge_factor=16, seed=4)), True)
    n = el.vertex_count
    roots = np.array([0, 5, 77])
    base = 9

    def init(n_):
        v = np.full(n_, UNREACHED, np.int64)
        v[roots] = base
        return v
    prog = dataclasses.replace(wg.bfs_program(0), initial_value=lambda v: base if v in set(roots) else UNREACHED,
                               initial_frontier=lambda n_: tuple(roots), initial_values=init)
    topo = wg.build_pull_topology(el, 4)
    idx = wg.build_edge_index(topo)
    deg = wg.compute_out_degrees(el)
    cfg = wg.EngineConfig(threshold=wg.FullnessThreshold.of("0.01"), precision=wg.FrontierPrecision(8))
    res = wg.run_until_convergence(topo, idx, prog, deg, cfg)
    assert any(s.mode == wg.MODE_FULL for s in res.stats[1:])  # a bottom-up dense pull ran
    tp = oracle.build_pull_topology(n, el.src, el.dst, None, 4)
    ref = oracle.run_until_convergence(tp, oracle.build_edge_index(tp), oracle.compute_out_degrees(n, el.src),
                                       oracle.kern_of("bfs"), init(n), roots, Fraction(1, 100), 8)
    assert np.array_equal(res.values, ref.values)


# ------------------------------------------- host reference-layout ingest ---
def _oracle_graph(scale, app, sym=True):
    n, s, d = oracle.rmat_edges_fast(scale, 16, 1)
    s, d = oracle.prepare_unweighted(n, s, d, sym)
    w = oracle.synthesize_weights(s, d, 255) if app == "sssp" else None
    topo = oracle.build_pull_topology(n, s, d, w, 4)
    return n, topo, oracle.build_edge_index(topo), oracle.compute_out_degrees(n, s)


def _host_objects(wg, n, topo, idx):
    """The package's PullTopology / EdgeIndex over the reference's own host
    arrays (the reference constructors, graph.py:109-212)."""
    return (wg.PullTopology(n, topo.vector_width, topo.edge_count, topo.vec_dst, topo.lane_src,
                            topo.lane_weight, topo.lane_count),
            wg.EdgeIndex(n, topo.vector_count, idx.offsets, idx.positions))


@pytest.mark.parametrize("app", ["bfs", "cc", "sssp"])
def test_run_from_host_reference_layout(wg, app):
    """run_until_convergence on int64 host arrays: raw H2D + device narrowing
    (wg_ingest_*) + device value scan give the oracle's values and trace."""
    n, topo, idx, deg = _oracle_graph(12, app)
    ht, hi = _host_objects(wg, n, topo, idx)
    vpg, thr = (8, Fraction(1, 100)) if app == "bfs" else (4, Fraction(1, 5))
    cfg = wg.EngineConfig(threshold=wg.FullnessThreshold(thr), precision=wg.FrontierPrecision(vpg))
    be = wg.B200Backend(reupload=True)
    prog = wg.make_program(app, None if app == "cc" else 0)
    vals, front = oracle.initial_state(app, n, 0)
    want = oracle.run_until_convergence(topo, idx, deg, oracle.kern_of(app), vals, front, thr, vpg)
    for _ in range(2):  # the second call re-uploads into the cached buffers
        res = wg.run_until_convergence(ht, hi, prog, deg, cfg, backend=be)
        assert np.array_equal(res.values, want.values)
        assert wg.stats_signature(res.stats) == oracle.signature(want.stats)


def test_reupload_sees_arrays_changed_in_place(wg):
    n, topo, idx, deg = _oracle_graph(10, "sssp")
    ht, hi = _host_objects(wg, n, topo, idx)
    cfg = wg.EngineConfig()
    be = wg.B200Backend(reupload=True)
    prog = wg.make_program("sssp", 0)
    wg.run_until_convergence(ht, hi, prog, deg, cfg, backend=be)
    topo.lane_weight[topo.lane_weight > 0] += 7  # same objects, new weights
    res = wg.run_until_convergence(ht, hi, prog, deg, cfg, backend=be)
    vals, front = oracle.initial_state("sssp", n, 0)
    want = oracle.run_until_convergence(topo, idx, deg, oracle.SSSP, vals, front, Fraction(1, 5), 4)
    assert np.array_equal(res.values, want.values)


def test_ingest_rejects_out_of_range_ids(wg):
    n, topo, idx, deg = _oracle_graph(8, "cc")
    bad = topo.lane_src.copy()
    bad[0, 0] = n + 5
    ht = wg.PullTopology(n, 4, topo.edge_count, topo.vec_dst, bad, None, topo.lane_count)
    hi = wg.EdgeIndex(n, topo.vector_count, idx.offsets, idx.positions)
    with pytest.raises(ValueError, match="lane source"):
        wg.run_until_convergence(ht, hi, wg.cc_program(), deg, wg.EngineConfig(), backend=wg.B200Backend())


@pytest.mark.parametrize("app", ["bfs", "cc", "sssp"])
def test_value_log_matches_reference(wg, app):
    """value_log (engine.py:337-338, 381-385): one value snapshot per
    iteration, equal to the reference loop's, with frontier_log beside it."""
    n, topo, idx, deg = _oracle_graph(10, app)
    ht, hi = _host_objects(wg, n, topo, idx)
    cfg = wg.EngineConfig(threshold=wg.FullnessThreshold(Fraction(1, 5)), precision=wg.FrontierPrecision(4))
    vlog, flog = [], []
    res = wg.run_until_convergence(ht, hi, wg.make_program(app, None if app == "cc" else 0), deg, cfg,
                                   frontier_log=flog, value_log=vlog)
    want_v, want_f = [], []
    vals, front = oracle.initial_state(app, n, 0)
    want = oracle.run_until_convergence(topo, idx, deg, oracle.kern_of(app), vals, front, Fraction(1, 5), 4,
                                        frontier_log=want_f, value_log=want_v)
    assert len(vlog) == len(want_v) == len(res.stats) == len(want.stats)
    for got, exp in zip(vlog, want_v):
        assert got.dtype == np.int64 and np.array_equal(got, exp)
    for got, exp in zip(flog, want_f):
        assert np.array_equal(got, exp)
    assert np.array_equal(vlog[-1], res.values)


@pytest.mark.parametrize("case", ["cc_floor", "bfs_bottom_up", "bfs_bottom_up_i64", "bfs_level_base"])
def test_plain_dense_kernels_from_iteration_2(wg, monkeypatch, case):
    """floor_pull_kernel (CC floor skipping) and bottom_up_pull_kernel (BFS)
    normally start at iteration 3 (WG_FLOOR_FROM); forced from iteration 2
    on a small graph they must still give the oracle's values and work
    counters -- including the int64 path (values >= 2^32) and a non-zero
    level base.  Both loop drivers (graph / per-iteration launches)."""
    import dataclasses
    monkeypatch.setenv("WG_FLOOR_FROM", "2")
    app = "cc" if case.startswith("cc") else "bfs"
    n, topo, idx, deg = _oracle_graph(12, app)
    ht, hi = _host_objects(wg, n, topo, idx)
    prog = wg.make_program(app, None if app == "cc" else 0)
    vals, front = oracle.initial_state(app, n, 0)
    base = {"bfs_bottom_up_i64": 5_000_000_000, "bfs_level_base": 7}.get(case)
    if base is not None:
        vals = vals.copy()
        vals[0] = base
        prog = dataclasses.replace(prog, initial_values=lambda k, v=vals: v.copy())
    thr = Fraction(1, 5)  # dense iterations early enough to reach the plain kernels
    want = oracle.run_until_convergence(topo, idx, deg, oracle.kern_of(app), vals, front, thr, 4)
    assert sum(s.mode == "FullScan" for s in want.stats[1:]) >= 1
    for graph in ("1", "0"):
        monkeypatch.setenv("WG_GRAPH", graph)
        cfg = wg.EngineConfig(threshold=wg.FullnessThreshold(thr), precision=wg.FrontierPrecision(4))
        res = wg.run_until_convergence(ht, hi, prog, deg, cfg, backend=wg.B200Backend())
        assert np.array_equal(res.values, want.values), (case, graph)
        assert wg.stats_signature(res.stats) == oracle.signature(want.stats), (case, graph)


def test_pagerank_deterministic_and_hub_split(wg):
    """No float atomics: two runs are bit-identical, also on a graph whose
    hubs' in-vectors span many warp ranges (pr_fixup adds the pieces in
    order); and within 1e-6 of the float64 oracle there too."""
    rng = np.random.default_rng(5)
    n = 5000
    # two hubs with thousands of in-edges + random edges
    src = np.concatenate([rng.integers(0, n, 40000), rng.integers(0, n, 9000), rng.integers(0, n, 20000)])
    dst = np.concatenate([np.full(40000, 7), np.full(9000, 4000), rng.integers(0, n, 20000)])
    keep = src != dst
    el = wg.drop_self_loops_dedup(wg.EdgeList(n, src[keep], dst[keep]), symmetric=False)
    topo = wg.build_pull_topology(el, 4)
    a = wg.pagerank(topo, 20, 0.85).copy()
    b = wg.pagerank(topo, 20, 0.85).copy()
    assert a.tobytes() == b.tobytes()
    ref = oracle.pagerank_numpy(el.vertex_count, el.src, el.dst, 20, 0.85)
    assert np.max(np.abs(a.astype(np.float64) - ref)) <= 1e-6
    el2 = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=16, edge_factor=16, seed=9)),
                                   symmetric=False)
    t2 = wg.build_pull_topology(el2, 4)
    x = wg.pagerank(t2, 20, 0.85).copy()
    y = wg.pagerank(t2, 20, 0.85).copy()
    assert x.tobytes() == y.tobytes()
    ref2 = oracle.pagerank_numpy(el2.vertex_count, el2.src, el2.dst, 20, 0.85)
    assert np.max(np.abs(x.astype(np.float64) - ref2)) <= 1e-6
