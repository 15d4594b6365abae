"""Frontier-density sweep (BASELINE.json configs[4]): on the
directed RMAT s25 ef32 graph, seeded random frontiers whose out-degree sum is
f*|E|; for each f one forced Wedge iteration (transform + group compaction +
pull) and one forced dense iteration are timed with the library's CUDA-event
timers (median of --reps).  The crossover tells where the Wedge gate should
switch on B200 (the reference default threshold is 1/5, cli.py:52-56).

usage: python tools/density_sweep.py [--scale 25] [--ef 32] [--reps 5] [--out profiles/x.json]
"""
from __future__ import annotations

import argparse
import json
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

FRACTIONS = [0.0001, 0.0003, 0.001, 0.003, 0.01, 0.03, 0.1, 0.2, 0.3, 0.5, 1.0]


def frontier_for(deg: np.ndarray, f: float, rng) -> np.ndarray:
    """Random vertices (with out-edges) until their out-degree sum reaches f*E."""
    E = int(deg.sum())
    if f >= 1.0:
        return np.arange(deg.size, dtype=np.int64)
    cand = np.flatnonzero(deg > 0)
    perm = rng.permutation(cand)
    cum = np.cumsum(deg[perm])
    k = int(np.searchsorted(cum, f * E, side="left")) + 1
    return np.sort(perm[: min(k, perm.size)])


def time_iteration(loop, g, init, members, kern, thr, reps, timer):
    from paper_1903_07754_b200 import device as dv
    words = dv.initial_words(g.n, members)
    res = []
    recs = None
    for r in range(reps + 1):
        p = loop.seed(init, words, kern, thr)
        timer.reset()
        p.timer = timer.handle
        loop.enqueue(p, 1, 1)
        recs = loop._read(1, 1)
        rows = timer.read()
        if r == 0:
            continue  # warm-up
        by = {}
        for kind, it, ms in rows:
            by[kind] = by.get(kind, 0.0) + ms
        res.append(by)
    rec = recs[0]
    med = {k: float(np.median([b.get(k, 0.0) for b in res])) for k in (1, 2, 3, 4)}
    return med, rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=25)
    ap.add_argument("--ef", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib, device as dv

    el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=args.scale, edge_factor=args.ef, seed=1)),
                                  symmetric=False)
    topo = wg.build_pull_topology(el, 4)
    g = topo.device
    deg = g.outdeg_np()
    E = int(g.edges)
    kern = wg.cc_program().kernel  # min-label propagation: every pulled destination can update
    init = dv.encode_values(np.arange(g.n, dtype=np.int64), _lib.WG_VAL_U32)
    loop = dv.DeviceLoop(g, 2, _lib.WG_VAL_U32)  # 4 vectors per group
    timer = _lib.EventTimer(64)
    rng = np.random.default_rng(7)
    rows = []
    for f in FRACTIONS:
        members = frontier_for(deg, f, rng)
        act = int(deg[members].sum())
        row = {"f": f, "frontier": int(members.size), "active_edges": act, "active_fraction": act / E}
        if act < E:  # forced Wedge: threshold 1 (wedge iff sum < E)
            med, rec = time_iteration(loop, g, init, members, kern, Fraction(1), args.reps, timer)
            assert int(rec[0]) == 2, rec[0]
            row["wedge"] = {"transform_ms": round(med[1], 4), "pull_ms": round(med[2], 4),
                            "end_ms": round(med[3] + med[4], 4),
                            "total_ms": round(med[1] + med[2] + med[3] + med[4], 4),
                            "covered_vectors": int(rec[7]), "transform_entries": int(rec[8]),
                            "vectors_touched": int(rec[2])}
        else:
            row["wedge"] = None
        med, rec = time_iteration(loop, g, init, members, kern, Fraction(0), args.reps, timer)
        assert int(rec[0]) == 1, rec[0]
        row["dense"] = {"pull_ms": round(med[2], 4), "end_ms": round(med[3] + med[4], 4),
                        "total_ms": round(med[1] + med[2] + med[3] + med[4], 4), "vectors_touched": int(rec[2])}
        if row["wedge"]:
            row["wedge_speedup"] = round(row["dense"]["total_ms"] / row["wedge"]["total_ms"], 3)
        rows.append(row)
        print(json.dumps(row), flush=True)
    cross = None
    for r in rows:
        if r["wedge"] and r["wedge"]["total_ms"] >= r["dense"]["total_ms"]:
            cross = r["f"]
            break
    out = {"graph": f"RMAT s{args.scale} ef{args.ef} directed dedup (BASELINE configs[4])", "V": g.n, "E": E,
           "W": 4, "vpg": 4, "kernel": "min-label (CC) min-plus", "reps": args.reps,
           "timing": "median of CUDA-event timers around each launch group, one iteration, hot L2",
           "first_fraction_where_dense_wins": cross, "rows": rows}
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
