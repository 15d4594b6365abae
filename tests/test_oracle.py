"""Pin the CPU oracle (oracle/) to the reference: every golden vector in
tests/golden/ (produced from the reference package itself) must be
reproduced by the oracle's C restatement and numpy driver.  When the
reference's own compiled kernels exist (oracle/_ref), they are checked too.
CPU only."""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import GT_EDGES, GT_VERTICES


def _topo(case, n, width):
    return oracle.build_pull_topology(n, case["src"], case["dst"], case["w"], width)


def _backends():
    bes = [oracle.PortBackend(1), oracle.PortBackend(4)]
    if oracle.ref_kernels() is not None:
        bes.append(oracle.RefBackend(1))
    return bes


@pytest.mark.parametrize("kind", ["pull_full", "pull_wedge", "transform"])
def test_oracle_kernels_match_golden(golden, kind):
    cases = [c for c in golden.meta("kernels") if c["kind"] == kind]
    assert cases
    for be in _backends():
        for c in cases:
            g = golden.kernel_case(c)
            n, width = c["n"], c["width"]
            topo = _topo(g, n, width)
            if kind == "transform":
                index = oracle.build_edge_index(topo)
                ww = np.zeros_like(g["wedge"])
                visited = be.transform(g["frontier"], n, index.offsets, index.positions, c["shift"],
                                       ww, 16, 1)
                assert visited == c["visited"], (be.name, c["id"])
                assert np.array_equal(ww, g["wedge"]), (be.name, c["id"])
                continue
            kern = oracle.kern_of(c["app"])
            prev = g["prev"].copy()
            nxt = prev.copy()
            out = np.zeros_like(g["out"])
            if kind == "pull_full":
                t = be.pull_full(topo, prev, nxt, out, kern, oracle.UNREACHED, 1)
            else:
                t = be.pull_wedge(topo, g["wedge"], c["shift"], c["groups"], prev, nxt, out, kern,
                                  oracle.UNREACHED, 1)
            assert t == c["touched"], (be.name, c["id"])
            assert np.array_equal(nxt, g["nxt"]), (be.name, c["id"])
            assert np.array_equal(out, g["out"]), (be.name, c["id"])


def test_oracle_layout_matches_golden(golden):
    z = golden.npz("layout")
    for c in golden.meta("layout"):
        nm = c["name"]
        w = z[f"{nm}/w"] if c["weighted"] else None
        topo = oracle.build_pull_topology(c["n"], z[f"{nm}/src"], z[f"{nm}/dst"], w, c["width"])
        assert np.array_equal(topo.vec_dst, z[f"{nm}/vec_dst"]), nm
        assert np.array_equal(topo.lane_src, z[f"{nm}/lane_src"]), nm
        assert np.array_equal(topo.lane_count, z[f"{nm}/lane_count"]), nm
        if c["weighted"]:
            assert np.array_equal(topo.lane_weight, z[f"{nm}/lane_weight"]), nm
        idx = oracle.build_edge_index(topo)
        assert np.array_equal(idx.offsets, z[f"{nm}/offsets"]), nm
        assert np.array_equal(idx.positions, z[f"{nm}/positions"]), nm
        assert np.array_equal(oracle.compute_out_degrees(c["n"], z[f"{nm}/src"]), z[f"{nm}/degrees"]), nm


def test_gt_known_answers():
    """Known answers of pkg/tests/test_graph_core.py:39-44, 116-118, 136-140."""
    src = [e[0] for e in GT_EDGES]
    dst = [e[1] for e in GT_EDGES]
    topo = oracle.build_pull_topology(GT_VERTICES, src, dst, None, 2)
    vecs = [(int(topo.vec_dst[p]), [int(x) for x in topo.lane_src[p, : topo.lane_count[p]]])
            for p in range(topo.vector_count)]
    assert vecs == [(1, [0]), (2, [0]), (3, [1, 2]), (3, [5]), (4, [3]), (5, [4])]
    idx = oracle.build_edge_index(topo)
    got = {v: idx.positions[idx.offsets[v]: idx.offsets[v + 1]].tolist() for v in range(GT_VERTICES)}
    assert got == {0: [0, 1], 1: [2], 2: [2], 3: [4], 4: [5], 5: [3]}
    assert oracle.compute_out_degrees(GT_VERTICES, src).tolist() == [2, 1, 1, 1, 1, 1]


def test_oracle_runs_match_golden(golden):
    """Driver restatement: digest + every per-iteration stat of the reference
    (runs.json), and per-iteration frontiers where recorded."""
    z = golden.npz("gen")
    runs = golden.meta("runs")
    zr = golden.npz("runs")
    graphs = {}
    for r in runs:
        if r["scale"] > 10:
            continue
        key = (r["scale"], r["app"], r["width"])
        if key not in graphs:
            n, s, d = oracle.rmat_edges(r["scale"], 16, 1)
            keep = s != d
            s, d, _ = oracle.symmetrize(s[keep], d[keep], None, dedup=True)
            w = oracle.synthesize_weights(s, d, 255) if r["app"] == "sssp" else None
            topo = oracle.build_pull_topology(n, s, d, w, r["width"])
            graphs[key] = (n, topo, oracle.build_edge_index(topo), oracle.compute_out_degrees(n, s))
        n, topo, idx, deg = graphs[key]
        assert topo.edge_count == r["E"]
        vals, front = oracle.initial_state(r["app"], n, r["root"])
        flog = []
        out = oracle.run_until_convergence(topo, idx, deg, oracle.kern_of(r["app"]), vals, front,
                                           Fraction(*r["thr"]), r["vpg"], frontier_log=flog)
        assert oracle.result_digest(out.values) == r["digest"], r["name"]
        got = [[s.iteration, s.mode, s.active_edges, s.vectors_touched, s.frontier_out_size,
                s.covered_vectors, s.transform_entries] for s in out.stats]
        assert got == r["stats"], r["name"]
        assert np.array_equal(out.values, zr[f"{r['name']}/values"])
        lens = zr[f"{r['name']}/flog_len"]
        assert [len(f) for f in flog] == lens.tolist()
        assert np.array_equal(np.concatenate(flog) if flog else np.empty(0), zr[f"{r['name']}/flog"])


def test_oracle_generators_match_golden(golden):
    z = golden.npz("gen")
    n, s, d = oracle.rmat_edges(8, 16, 1)
    assert np.array_equal(s, z["rmat8_src"]) and np.array_equal(d, z["rmat8_dst"])
    n, s, d = oracle.rmat_edges(11, 4, 7, chunk=1000)  # chunked stream == one-shot stream
    assert np.array_equal(s, z["rmat11_s7_src"]) and np.array_equal(d, z["rmat11_s7_dst"])
    keep = s != d
    ss, dd, _ = oracle.symmetrize(s[keep], d[keep], None, dedup=True)
    assert np.array_equal(ss, z["rmat11_s7_sym_src"]) and np.array_equal(dd, z["rmat11_s7_sym_dst"])
    assert np.array_equal(oracle.synthesize_weights(ss, dd, 255), z["rmat11_s7_sym_w255"])
    assert np.array_equal(oracle.synthesize_weights(z["hash_src"], z["hash_dst"], 1000), z["hash_w1000"])
    # frozen known answer (pkg/tests/test_io.py:151-154)
    assert oracle.synthesize_weights(np.array([0]), np.array([1]), 128).tolist() == [56]


def test_oracle_pagerank_forms_agree():
    n, s, d = oracle.rmat_edges(9, 8, 3)
    s, d = oracle.dedup_directed(s, d)
    topo = oracle.build_pull_topology(n, s, d, None, 4)
    deg = oracle.compute_out_degrees(n, s)
    a = oracle.pagerank(topo, deg, 20, 0.85)
    b = oracle.pagerank_numpy(n, s, d, 20, 0.85)
    assert np.max(np.abs(a - b)) < 1e-12
    assert abs(a.sum() - 1.0) < 1e-9


def test_survey_digests_s16_bfs():
    """SURVEY §8(c) froze reference digests at RMAT s16; the oracle must
    reproduce the BFS one (the others run in the GPU suite)."""
    n, s, d = oracle.rmat_edges(16, 16, 1)
    keep = s != d
    s, d, _ = oracle.symmetrize(s[keep], d[keep], None, dedup=True)
    assert len(s) == 1_817_684
    topo = oracle.build_pull_topology(n, s, d, None, 4)
    idx = oracle.build_edge_index(topo)
    deg = oracle.compute_out_degrees(n, s)
    assert int(np.argmax(deg)) == 0
    vals, front = oracle.initial_state("bfs", n, 0)
    out = oracle.run_until_convergence(topo, idx, deg, oracle.BFS, vals, front, Fraction(1, 100), 8,
                                       backend=oracle.PortBackend(4))
    assert oracle.result_digest(out.values) == "591673cb243fad4e"
    assert len(out.stats) == 5


def test_threaded_input_prep_matches_golden(golden):
    """The reference arm's fast input preparation (orc_rmat + radix-sort
    dedup) reproduces the reference generators' golden outputs."""
    z = golden.npz("gen")
    n, s, d = oracle.rmat_edges_fast(8, 16, 1)
    assert np.array_equal(s, z["rmat8_src"]) and np.array_equal(d, z["rmat8_dst"])
    n, s, d = oracle.rmat_edges_fast(11, 4, 7)
    assert np.array_equal(s, z["rmat11_s7_src"]) and np.array_equal(d, z["rmat11_s7_dst"])
    ss, dd = oracle.prepare_unweighted(n, s, d, True)
    assert np.array_equal(ss, z["rmat11_s7_sym_src"]) and np.array_equal(dd, z["rmat11_s7_sym_dst"])
    keep = s != d
    a, b = oracle.dedup_directed(s[keep], d[keep])
    ss, dd = oracle.prepare_unweighted(n, s, d, False)
    assert np.array_equal(ss, a) and np.array_equal(dd, b)
