"""Host-side profile (cProfile) of bench steps on a small workload: where the
time outside the kernels goes.  usage: python tools/host_prof.py [bfs16]"""
import cProfile
import pstats
import sys
import time
from fractions import Fraction
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv
from paper_1903_07754_b200.engine import _initial_values

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "bfs16"]
el, topo = bench.make_graph(wl)
g = topo.device
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
init = _initial_values(prog, g.n)
loop = dv.DeviceLoop(g, {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]], _lib.WG_VAL_U32)
dinit = dv.encode_values(init, _lib.WG_VAL_U32)
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
fh = dv.first_hit_ok(prog.kernel, init, None if wl["app"] == "cc" else np.array([0]))
lvl = dv.first_hit_level(init) if fh else 0
ident = dv.identity_values(init)


def step():
    p = loop.seed(dinit, words, prog.kernel, Fraction(wl["thr"]), first_hit=fh, level_base=lvl, identity_init=ident)
    return loop.drive(p, g.n + 16)


for _ in range(50):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    step()
torch.cuda.synchronize()
print(f"wall per step {1000 * (time.perf_counter() - t0) / 200:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
