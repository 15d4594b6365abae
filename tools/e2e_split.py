"""Split the e2e step of bench.py into H2D, on-device rebuild and loop (CUDA
events; median of 5).  usage: python tools/e2e_split.py [cc22]"""
import sys
from fractions import Fraction
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv
from paper_1903_07754_b200.engine import _initial_values

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cc22"]
el, topo = bench.make_graph(wl)
g = topo.device
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
host = {"vsrc": g.vsrc.cpu().pin_memory(), "voff": g.vector_offsets().cpu().pin_memory()}
if g.vw is not None:
    host["vw"] = g.vw.cpu().pin_memory()
dev = {k: torch.empty(v.numel() + 64, dtype=v.dtype, device="cuda")[: v.numel()] for k, v in host.items()}
for k, v in host.items():
    dev[k].copy_(v)
scratch = torch.empty(int(_lib.load().wg_index_scratch_bytes(g.nvec * g.width, g.n)), dtype=torch.uint8,
                      device="cuda")
g2 = dv.DeviceGraph.from_lanes(g.n, g.width, g.edges, g.nvec, dev["vsrc"], dev.get("vw"), dev["voff"], scratch)
shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
loop = dv.DeviceLoop(g2, shift, _lib.WG_VAL_U32)
init = dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32)
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
out_host = torch.empty(g.n, dtype=torch.int32).pin_memory()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


rows = []
for rep in range(6):
    e0 = ev()
    for k, v in host.items():
        dev[k].copy_(v, non_blocking=True)
    e1 = ev()
    g2.rebuild_derived(dev["voff"], scratch)
    e2 = ev()
    p = loop.seed(init, words, prog.kernel, Fraction(wl["thr"]))
    recs, conv, last = loop.drive(p, g.n + 16)
    e3 = ev()
    out_host.copy_(loop.values_after(last), non_blocking=True)
    e4 = ev()
    e4.synchronize()
    if rep:
        rows.append([e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3), e3.elapsed_time(e4)])
r = np.median(np.array(rows), axis=0)
h2d = sum(v.numel() * v.element_size() for v in host.values())
print(f"{wl['desc']}: H2D {r[0]:.3f} ms ({h2d / r[0] / 1e6:.1f} GB/s)  rebuild {r[1]:.3f} ms  loop {r[2]:.3f} ms  "
      f"D2H {r[3]:.3f} ms  total {r.sum():.3f} ms")
