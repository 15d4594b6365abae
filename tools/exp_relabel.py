"""Experiment: effect of degree-ordered vertex relabelling on the dense pull."""
import sys, time
from fractions import Fraction
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv

el = wg.generate(wg.GenSpec("rmat", scale=22, edge_factor=16, seed=1))
el = wg.drop_self_loops_dedup(el, symmetric=True)
s, d, _ = el.device_arrays()
n = el.vertex_count
s64 = s.to(torch.int64); d64 = d.to(torch.int64)
deg = torch.bincount(s64, minlength=n)

def run(src, dst, label):
    g = dv.DeviceGraph.build(n, src, dst, None, 4)
    loop = dv.DeviceLoop(g, 2, _lib.WG_VAL_U32)
    init = dv.encode_values(np.arange(n), _lib.WG_VAL_U32)
    words = dv.all_words(n)
    prog = wg.cc_program()
    for _ in range(3):
        p = loop.seed(init, words, prog.kernel, Fraction(1, 5)); loop.drive(p, n + 16)
    timer = _lib.EventTimer(64)
    p = loop.seed(init, words, prog.kernel, Fraction(1, 5)); p.timer = timer.handle
    recs, conv, last = loop.drive(p, n + 16)
    torch.cuda.synchronize()
    rows = timer.read()
    pulls = [ms for k, it, ms in rows if k == 2]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); p = loop.seed(init, words, prog.kernel, Fraction(1, 5)); loop.drive(p, n + 16); b.record(); b.synchronize()
    print(label, "pull ms per iteration", [round(x, 3) for x in pulls], "total", round(a.elapsed_time(b), 3), flush=True)
    return dv.values_to_int64(loop.values_after(last), _lib.WG_VAL_U32)

v0 = run(s, d, "reference order")
order = torch.argsort(-deg, stable=True)          # old ids by decreasing degree
new_of_old = torch.empty_like(order); new_of_old[order] = torch.arange(n, device=order.device)
s2 = new_of_old[s64].to(torch.int32); d2 = new_of_old[d64].to(torch.int32)
v1 = run(s2, d2, "degree relabelled (labels = new ids, not comparable)")
