import sys, time
from fractions import Fraction
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv
from paper_1903_07754_b200.engine import _initial_values
import ctypes
wl = bench.WORKLOADS["sssp_grid"]
el, topo = bench.make_graph(wl)
g = topo.device
prog = wg.sssp_program(0)
loop = dv.DeviceLoop(g, 2, _lib.WG_VAL_U32)
init = dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32)
words = dv.initial_words(g.n, np.array([0]))
p = loop.seed(init, words, prog.kernel, Fraction(1, 5))
L = _lib.load()
exe = loop._graph_for(p)
it = 1
for launch in range(4):
    limit = it - 1 + loop.ring - 2
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _lib.check(L.wg_run_loop_launch(exe, ctypes.byref(loop.bufs), limit, _lib.stream_ptr()))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    c = loop.ctrl.cpu().tolist()
    rows = loop._read(it, 8)
    print("launch", launch, "it", it, "limit", limit, "ctrl", c, "ms", round((t1 - t0) * 1e3, 2),
          "variants", [int(r[15 - 4]) if False else int(r[11]) for r in rows], "modes", [int(r[0]) for r in rows], flush=True)
    it = min(c[0], limit) + 1
