"""Small driver for ncu captures: build one BASELINE workload and run it once
(or twice) through the device loop.  Usage: python tools/prof_run.py cc22 [runs]"""
import sys
from fractions import Fraction
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_1903_07754_b200 import _lib, device as dv
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200.engine import _initial_values

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cc22"]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
el, topo = bench.make_graph(wl)
g = topo.device
if wl["app"] == "pr":
    for _ in range(runs):
        dv.pagerank(g, 20, 0.85)
    torch.cuda.synchronize()
    sys.exit(0)
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
loop = dv.DeviceLoop(g, shift, _lib.WG_VAL_U32)
dinit = dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32)
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
for _ in range(runs):
    p = loop.seed(dinit, words, prog.kernel, Fraction(wl["thr"]), first_hit=(wl["app"] == "bfs"),
                  identity_init=(wl["app"] == "cc"))
    recs, conv, last = loop.drive(p, g.n + 16)
torch.cuda.synchronize()
print("iterations", len(recs), "converged", conv)
