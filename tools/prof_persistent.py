"""Launch the persistent Wedge loop directly (no graph) on a workload, for ncu.
usage: python tools/prof_persistent.py sssp_grid [iterations]"""
import ctypes, sys
from fractions import Fraction
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv
from paper_1903_07754_b200.engine import _initial_values
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "sssp_grid"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
skip_to = int(sys.argv[3]) if len(sys.argv) > 3 else 0
el, topo = bench.make_graph(wl)
g = topo.device
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
loop = dv.DeviceLoop(g, {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]], _lib.WG_VAL_U32)
init = dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32)  # noqa
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
p = loop.seed(init, words, prog.kernel, Fraction(wl["thr"]))
L = _lib.load()
ts = torch.zeros(4 * 20000, dtype=torch.int64, device="cuda")
_lib.check(L.wg_debug_phase_buffer(ts.data_ptr(), 20000))
if skip_to:
    _lib.check(L.wg_run_persistent(ctypes.byref(g.struct()), ctypes.byref(loop.bufs), ctypes.byref(p), skip_to, _lib.stream_ptr()))
    torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
_lib.check(L.wg_run_persistent(ctypes.byref(g.struct()), ctypes.byref(loop.bufs), ctypes.byref(p), skip_to + iters, _lib.stream_ptr()))
b.record(); b.synchronize()
print("ctrl", loop.ctrl.cpu().tolist(), "ms", a.elapsed_time(b), "us/iter", 1000 * a.elapsed_time(b) / max(1, int(loop.ctrl[0]) - skip_to))

t = ts.view(-1, 4).cpu().numpy()[1: int(loop.ctrl[0]) + 1]
t = t[t[:, 0] > 0]
d = np.diff(t, axis=1) / 1000.0
nxt = (t[1:, 0] - t[:-1, 3]) / 1000.0
print("iterations stamped", len(t))
for name, col in (("transform", d[:, 0]), ("pull", d[:, 1]), ("finalize+sync", d[:, 2])):
    print(f"{name:14s} us: mean {col.mean():8.2f}  p50 {np.median(col):8.2f}  p90 {np.percentile(col, 90):8.2f}")
print(f"between iters  us: mean {nxt.mean():8.2f}")
