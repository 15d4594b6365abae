"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package `wedgegraph` from /root/reference/pkg/src
(read-only; nothing is copied) and, when oracle/_ref holds the reference's
compiled Cython kernels, injects them as `wedgegraph._kernels` so both the
`native` and `python` backends are available.  Every fixture records the
reference's own outputs on seeded inputs:

* kernels.npz  — backend protocol cases (pull_full / pull_wedge / transform)
                 in the style of pkg/tests/test_kernels_backends.py:24-94.
* layout.npz   — build_pull_topology / build_edge_index / compute_out_degrees
                 outputs (graph.py:220-301) for small graphs.
* runs.npz + runs.json — run_until_convergence results (values, per-iteration
                 stats, per-iteration frontiers) for BFS/CC/SSSP on RMAT
                 graphs prepared like SURVEY §8(d).
* gen.npz      — generator outputs (graph_io.py:87-221).

The GPU box never reads /root/reference: only these committed fixtures.
"""

from __future__ import annotations

import importlib.util
import json
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
ROOT = OUT.parent.parent
REF_SRC = Path("/root/reference/pkg/src")


def import_reference():
    sys.path.insert(0, str(REF_SRC))
    cands = sorted((ROOT / "oracle" / "_ref").glob("_kernels*.so"))
    if cands:
        spec = importlib.util.spec_from_file_location("wedgegraph._kernels", cands[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules["wedgegraph._kernels"] = mod
    import wedgegraph  # noqa: E402
    return wedgegraph


wg = import_reference()
from wedgegraph.bitmask import Bitmask  # noqa: E402

UNREACHED = wg.UNREACHED


def random_edge_tuples(rng, max_vertices=64, max_edges=256, weighted=False):
    n = int(rng.integers(2, max_vertices + 1))
    m = int(rng.integers(1, max_edges + 1))
    src = rng.integers(0, n, size=m)
    dst = rng.integers(0, n, size=m)
    wgt = rng.integers(1, 101, size=m) if weighted else None
    return n, src.astype(np.int64), dst.astype(np.int64), (None if wgt is None else wgt.astype(np.int64))


def random_state(rng, n):
    prev = rng.integers(0, n + 2, size=n).astype(np.int64)
    prev[rng.random(n) < 0.3] = UNREACHED
    return prev


def build(n, src, dst, w, width):
    el = wg.EdgeList(n, src, dst, w)
    topo = wg.build_pull_topology(el, width)
    return el, topo, wg.build_edge_index(topo), wg.compute_out_degrees(el)


PROGRAMS = {"bfs": lambda: wg.bfs_program(0), "cc": wg.cc_program, "sssp": lambda: wg.sssp_program(0)}


def skewed_edges(rng, n, m):
    """Heavy-tailed destinations so some destinations span many warps."""
    src = rng.integers(0, n, size=m)
    dst = np.minimum((rng.pareto(0.7, size=m) * 3).astype(np.int64), n - 1)
    return src.astype(np.int64), dst.astype(np.int64)


def make_kernels():
    be = wg.get_backend("native" if "native" in wg.available_backends() else "python")
    store = {}
    meta = []

    graphs = {}

    def put(prefix, **arrs):
        # graphs are stored once (int32) and referenced by id; nxt as a diff
        src, dst, w = arrs.pop("src"), arrs.pop("dst"), arrs.pop("w", None)
        key = (src.tobytes(), dst.tobytes(), None if w is None else w.tobytes())
        if key not in graphs:
            gid = f"g{len(graphs)}"
            graphs[key] = gid
            store[f"{gid}/src"] = src.astype(np.int32)
            store[f"{gid}/dst"] = dst.astype(np.int32)
            if w is not None:
                store[f"{gid}/w"] = w.astype(np.int32)
        store[f"{prefix}/graph"] = np.array(graphs[key])
        if "nxt" in arrs:
            prev, nxt = arrs["prev"], arrs.pop("nxt")
            ch = np.nonzero(prev != nxt)[0]
            store[f"{prefix}/chg_idx"] = ch.astype(np.int32)
            store[f"{prefix}/chg_val"] = nxt[ch]
        for k, v in arrs.items():
            if v is not None:
                store[f"{prefix}/{k}"] = np.asarray(v)

    cid = 0
    # pull_full: test_kernels_backends.py:24-43 style + larger skewed graphs
    specs = [(s, w, 32, 120) for s in range(15) for w in (1, 2, 4)]
    specs += [(100 + s, w, 2000, 16000) for s in range(4) for w in (1, 2, 4, 8)]
    for seed, width, maxv, maxe in specs:
        rng = np.random.default_rng(seed)
        if maxv > 100:
            n = maxv
            src, dst = skewed_edges(rng, n, maxe)
            w = rng.integers(1, 101, size=maxe).astype(np.int64)
        else:
            n, src, dst, w = random_edge_tuples(rng, maxv, maxe, weighted=True)
        _, topo, index, deg = build(n, src, dst, w, width)
        for app, mk in PROGRAMS.items():
            prog = mk()
            prev = random_state(rng, n)
            nxt = prev.copy()
            out = Bitmask(n)
            touched = be.pull_full(topo, prev, nxt, out.words, prog.kernel, UNREACHED, 1)
            p = f"c{cid}"
            put(p, src=src, dst=dst, w=w, prev=prev, nxt=nxt, out=out.words)
            meta.append(dict(id=p, kind="pull_full", n=n, width=width, app=app, touched=int(touched)))
            cid += 1

    # pull_wedge: test_kernels_backends.py:46-72 style
    specs = [(1000 + s, 2, 32, 120) for s in range(15)] + [(1100 + s, 4, 2000, 16000) for s in range(4)]
    for seed, width, maxv, maxe in specs:
        rng = np.random.default_rng(seed)
        if maxv > 100:
            n = maxv
            src, dst = skewed_edges(rng, n, maxe)
            w = rng.integers(1, 101, size=maxe).astype(np.int64)
        else:
            n, src, dst, w = random_edge_tuples(rng, maxv, maxe, weighted=True)
        _, topo, index, deg = build(n, src, dst, w, width)
        nvec = topo.vector_count
        for shift in (0, 1, 2, 3, 4):
            groups = (nvec + (1 << shift) - 1) >> shift
            ww = np.zeros((groups + 63) >> 6, dtype=np.uint64)
            picks = rng.integers(0, groups, size=max(1, groups // (2 if maxv < 100 else 7)))
            for g in picks:
                ww[g >> 6] |= np.uint64(1) << np.uint64(g & 63)
            for app, mk in PROGRAMS.items():
                prog = mk()
                prev = random_state(rng, n)
                nxt = prev.copy()
                out = Bitmask(n)
                touched = be.pull_wedge(topo, ww, shift, groups, prev, nxt, out.words, prog.kernel,
                                        UNREACHED, 1)
                p = f"c{cid}"
                put(p, src=src, dst=dst, w=w, prev=prev, nxt=nxt, out=out.words, wedge=ww)
                meta.append(dict(id=p, kind="pull_wedge", n=n, width=width, app=app, shift=shift,
                                 groups=groups, touched=int(touched)))
                cid += 1

    # transform: test_kernels_backends.py:75-94 style
    specs = [(2000 + s, 2, 70, 250) for s in range(10)] + [(2100 + s, 4, 2000, 16000) for s in range(4)]
    for seed, width, maxv, maxe in specs:
        rng = np.random.default_rng(seed)
        if maxv > 100:
            n = maxv
            src, dst = skewed_edges(rng, n, maxe)
            src, dst = dst, src  # skewed sources: hub out-lists span many warps
        else:
            n, src, dst, _ = random_edge_tuples(rng, maxv, maxe)
        _, topo, index, deg = build(n, src, dst, None, width)
        members = rng.choice(n, size=int(rng.integers(0, n + 1)), replace=False).astype(np.int64)
        fw = Bitmask.from_indices(n, members).words
        nvec = topo.vector_count
        for shift in (0, 2, 3):
            groups = max(0, (nvec + (1 << shift) - 1) >> shift)
            ww = np.zeros((groups + 63) >> 6, dtype=np.uint64)
            visited = be.transform(fw, n, index.offsets, index.positions, shift, ww, 16, 1)
            p = f"c{cid}"
            put(p, src=src, dst=dst, w=None, frontier=fw, wedge=ww)
            meta.append(dict(id=p, kind="transform", n=n, width=width, shift=shift, groups=groups,
                             visited=int(visited)))
            cid += 1
    np.savez_compressed(OUT / "kernels.npz", **store)
    (OUT / "kernels.json").write_text(json.dumps(meta, indent=0))
    print("kernels:", cid, "cases")


def make_layout():
    store, meta = {}, []
    GT = [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4), (4, 5), (5, 3)]
    cases = [("gt_w2", 6, np.array([e[0] for e in GT]), np.array([e[1] for e in GT]), None, 2)]
    rng = np.random.default_rng(77)
    for width in (1, 2, 4, 8):
        n, src, dst, w = random_edge_tuples(rng, 200, 3000, weighted=True)
        cases.append((f"rand_w{width}", n, src, dst, w, width))
    el = wg.generate(wg.GenSpec("rmat", scale=10, edge_factor=16, seed=1))
    for width in (1, 4):
        cases.append((f"rmat10_w{width}", el.vertex_count, el.src, el.dst, None, width))
    for name, n, src, dst, w, width in cases:
        e, topo, index, deg = build(n, np.asarray(src, np.int64), np.asarray(dst, np.int64), w, width)
        store[f"{name}/src"] = e.src
        store[f"{name}/dst"] = e.dst
        if w is not None:
            store[f"{name}/w"] = e.weight
            store[f"{name}/lane_weight"] = topo.lane_weight
        store[f"{name}/vec_dst"] = topo.vec_dst
        store[f"{name}/lane_src"] = topo.lane_src
        store[f"{name}/lane_count"] = topo.lane_count
        store[f"{name}/offsets"] = index.offsets
        store[f"{name}/positions"] = index.positions
        store[f"{name}/degrees"] = deg
        meta.append(dict(name=name, n=int(n), width=width, weighted=w is not None))
    np.savez_compressed(OUT / "layout.npz", **store)
    (OUT / "layout.json").write_text(json.dumps(meta, indent=0))
    print("layout:", len(meta), "cases")


def prepared(scale, ef, app, seed=1):
    """SURVEY §8(d) pipeline: RMAT -> drop self-loops -> symmetrize(dedup) for cc/bfs;
    sssp: symmetrized + hash weights (max 255)."""
    el = wg.generate(wg.GenSpec("rmat", scale=scale, edge_factor=ef, seed=seed))
    keep = el.src != el.dst
    el = wg.EdgeList(el.vertex_count, el.src[keep], el.dst[keep])
    el = wg.symmetrize(el, dedup=True)
    if app == "sssp":
        el = wg.synthesize_weights(el, 255)
    return el


def make_runs():
    store, meta = {}, []
    be = wg.get_backend("native" if "native" in wg.available_backends() else "python")
    cfgs = {"bfs": (8, Fraction(1, 100)), "cc": (4, Fraction(1, 5)), "sssp": (4, Fraction(1, 5))}
    for scale in (8, 10, 12):
        for app in ("bfs", "cc", "sssp"):
            el = prepared(scale, 16, app)
            deg = wg.compute_out_degrees(el)
            root = int(np.argmax(deg))
            for width in (4,) if scale > 8 else (1, 4):
                topo = wg.build_pull_topology(el, width)
                index = wg.build_edge_index(topo)
                vpg0, thr0 = cfgs[app]
                for vpg, thr in ((vpg0, thr0), (1, Fraction(1)), (16, Fraction(1, 2)), (4, Fraction(0))):
                    prog = wg.make_program(app, None if app == "cc" else root)
                    cfg = wg.EngineConfig(threshold=wg.FullnessThreshold(thr),
                                          precision=wg.FrontierPrecision(vpg), max_iterations=100000)
                    flog = []
                    res = wg.run_until_convergence(topo, index, prog, deg, cfg, backend=be,
                                                   frontier_log=flog)
                    name = f"s{scale}_{app}_w{width}_v{vpg}_t{thr.numerator}_{thr.denominator}"
                    stats = [[s.iteration, s.mode, s.active_edges, s.vectors_touched, s.frontier_out_size,
                              s.covered_vectors, s.transform_entries] for s in res.stats]
                    if scale <= 10:
                        store[f"{name}/values"] = np.asarray(res.values)
                        lens = np.array([len(f) for f in flog], np.int64)
                        store[f"{name}/flog_len"] = lens
                        store[f"{name}/flog"] = (np.concatenate(flog) if flog else np.empty(0, np.int64))
                    meta.append(dict(name=name, scale=scale, app=app, width=width, vpg=vpg,
                                     thr=[thr.numerator, thr.denominator], root=root,
                                     digest=wg.result_digest(res.values), converged=res.converged,
                                     stats=stats, V=el.vertex_count, E=el.edge_count))
    # the GT worked example (conftest.py:21-22) at W=2
    np.savez_compressed(OUT / "runs.npz", **store)
    (OUT / "runs.json").write_text(json.dumps(meta))
    print("runs:", len(meta))


def make_gen():
    store = {}
    el = wg.generate(wg.GenSpec("rmat", scale=8, edge_factor=16, seed=1))
    store["rmat8_src"], store["rmat8_dst"] = el.src, el.dst
    el = wg.generate(wg.GenSpec("rmat", scale=11, edge_factor=4, seed=7))
    store["rmat11_s7_src"], store["rmat11_s7_dst"] = el.src, el.dst
    keep = el.src != el.dst
    sym = wg.symmetrize(wg.EdgeList(el.vertex_count, el.src[keep], el.dst[keep]), dedup=True)
    store["rmat11_s7_sym_src"], store["rmat11_s7_sym_dst"] = sym.src, sym.dst
    w = wg.synthesize_weights(sym, 255)
    store["rmat11_s7_sym_w255"] = w.weight
    rng = np.random.default_rng(5)
    s = rng.integers(0, 1 << 26, 4096)
    d = rng.integers(0, 1 << 26, 4096)
    store["hash_src"], store["hash_dst"] = s, d
    store["hash_w1000"] = wg.synthesize_weights(wg.EdgeList(1 << 26, s, d), 1000).weight
    np.savez_compressed(OUT / "gen.npz", **store)
    print("gen done")


if __name__ == "__main__":
    print("backends:", wg.available_backends())
    make_kernels()
    make_layout()
    make_runs()
    make_gen()
