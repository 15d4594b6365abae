"""Marginal cost of each iteration inside the real loop graph: TTS with the
iteration cap at k = 1..K (CUDA events, best of R), differenced.
Usage: python tools/iter_cost.py cc22 [reps]"""
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
R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
el, topo = bench.make_graph(wl)
g = topo.device
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
loop = dv.DeviceLoop(g, shift, _lib.WG_VAL_U32)
init = _initial_values(prog, g.n)
iv = dv.prepare_initial_values(init, prog.kernel, None if wl["app"] == "cc" else np.array([0]))
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
thr = Fraction(wl["thr"])


def run(cap):
    p = loop.seed(iv.seed(_lib.WG_VAL_U32), words, prog.kernel, thr, first_hit=iv.first_hit,
                  level_base=iv.level_base, identity_init=iv.identity, defer=True)
    return loop.drive(p, cap)


recs, _, _ = run(g.n + 16)
K = len(recs)
stream = torch.cuda.current_stream()
tts = []
for cap in range(0, K + 1):
    best = 1e9
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        if cap:
            run(cap)
        else:
            loop.seed(iv.seed(_lib.WG_VAL_U32), words, prog.kernel, thr, first_hit=iv.first_hit,
                      level_base=iv.level_base, identity_init=iv.identity, defer=True)
        b.record(stream)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    tts.append(best)
print(f"{wl['desc']}: {K} iterations, TTS {tts[-1]:.4f} ms (seed {tts[0]:.4f} ms)")
for k in range(1, K + 1):
    r = recs[k - 1]
    print(f"  it {k:2d} {r.mode:8s} +{(tts[k] - tts[k - 1]) * 1e3:8.1f} us  active_edges={r.active_edges} "
          f"frontier_out={r.frontier_out_size} touched={r.vectors_touched}")
