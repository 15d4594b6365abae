"""Cross-check the device paths on a large config and certify the result.
usage: python tools/validate_large.py sssp26"""
import os, sys
from fractions import Fraction
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv
from paper_1903_07754_b200.engine import _initial_values

name = sys.argv[1] if len(sys.argv) > 1 else "sssp26"
wl = bench.WORKLOADS[name]
el, topo = bench.make_graph(wl)
g = topo.device
app = wl["app"]
prog = wg.make_program(app, None if app == "cc" else 0)
shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
init = dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32)
words = dv.all_words(g.n) if app == "cc" else dv.initial_words(g.n, np.array([0]))
res = {}
for label, kw in (("graph+persistent", dict(graph=True)), ("no-graph sorted", dict(graph=False))):
    loop = dv.DeviceLoop(g, shift, _lib.WG_VAL_U32)
    p = loop.seed(init, words, prog.kernel, Fraction(wl["thr"]))
    recs, conv, last = loop.drive(p, g.n + 16, **kw)
    vals = loop.values_after(last).clone()
    dig = wg.result_digest(dv.values_to_int64(vals, _lib.WG_VAL_U32))
    res[label] = (dig, [(r.mode[0], r.active_edges, r.frontier_out_size) for r in recs], vals)
    print(label, dig, len(recs), "".join(r.mode[0] for r in recs), flush=True)
a, b = res["graph+persistent"], res["no-graph sorted"]
for i, (x, y) in enumerate(zip(a[1], b[1])):
    if x != y:
        print("first trace difference at iteration", i + 1, x, y)
        break
# certificate on the GPU: d[v] <= d[u] + w for every edge; every reached v != root is tight
s, d, w = el.device_arrays()
s = s.to(torch.int64) & 0xFFFFFFFF; d = d.to(torch.int64) & 0xFFFFFFFF
wt = (w.to(torch.int64) & 0xFFFFFFFF) if w is not None else torch.ones_like(s)
inc = 1 if app == "bfs" else 0
for label in res:
    v = res[label][2].to(torch.int64) & 0xFFFFFFFF
    INF = 0xFFFFFFFF
    fin = v[s] != INF
    cand = v[s] + (wt if app == "sssp" else inc)
    viol = (fin & (cand < v[d])).sum().item()
    tight = torch.zeros(g.n, dtype=torch.bool, device="cuda")
    tight[d[fin & (cand == v[d])]] = True
    reached = v != INF
    reached[0] = False
    untight = (reached & ~tight).sum().item()
    print(label, "violations", viol, "untight reached vertices", untight, "reached", int(reached.sum()), flush=True)
