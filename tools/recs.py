"""Print per-iteration records (mode, active edge fraction, frontier size) of a workload."""
import sys
from fractions import Fraction
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv
from paper_1903_07754_b200.engine import _initial_values
wl = bench.WORKLOADS[sys.argv[1]]
el, topo = bench.make_graph(wl)
g = topo.device
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
loop = dv.DeviceLoop(g, {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]], _lib.WG_VAL_U32)
init = dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32)
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
p = loop.seed(init, words, prog.kernel, Fraction(wl["thr"]))
recs, conv, last = loop.drive(p, g.n + 16)
for r in recs[:40]:
    print(r.iteration, r.mode, f"active {r.active_edges / g.edges:.4f}", "frontier_out", r.frontier_out_size,
          "touched", r.vectors_touched, "covered", r.covered_vectors)
