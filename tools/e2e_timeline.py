"""Timeline of one e2e step (CUDA events): per-chunk copy end, decode end,
index-chunk end, index finish, loop end, D2H end, relative to the start.
usage: python tools/e2e_timeline.py [workload] [format coded|bits|raw] [chunks]"""
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
fmt = sys.argv[2] if len(sys.argv) > 2 else "coded"
el, topo = bench.make_graph(wl)
g = topo.device
chunks = int(sys.argv[3]) if len(sys.argv) > 3 else max(1, min(8, (g.nvec * g.width) >> 22))
placed = len(sys.argv) > 4 and sys.argv[4] == "placed"
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
kw = {}
if fmt == "compact":  # bench.py's default host format
    host = g.host_format(symmetric=bool(wl.get("sym") or "grid" in wl))
    kw["outdeg_is_indeg"] = bool(wl.get("sym") or "grid" in wl)
    placed = False
else:
    host = {"voff": g.vector_offsets().cpu().pin_memory()}
if fmt == "compact":
    pass
elif fmt == "coded":
    host.update({k: v.cpu().pin_memory() for k, v in g.encode_lanes().items()})
elif fmt == "bits":
    host["vsrc_bits"] = g.pack_lanes()[0].cpu().pin_memory()
else:
    host["vsrc"] = g.vsrc.cpu().pin_memory()
if placed:
    host["outdeg"] = g.outdeg[: g.n].cpu().pin_memory()
if g.vw8 is not None:
    host["vw8"] = g.vw8[: g.nvec * g.width].cpu().pin_memory()
dev = {k: torch.empty(v.numel() + 64, dtype=v.dtype, device="cuda")[: v.numel()].view(v.shape) for k, v in host.items()}
for k, v in host.items():
    dev[k].copy_(v)
dev["vsrc"] = torch.empty(g.nvec * g.width + 64, dtype=torch.int32, device="cuda")[: g.nvec * g.width]
dev["vsrc"].copy_(g.vsrc)
vw = None
if g.vw8 is not None:
    vw = torch.empty(g.nvec * g.width + 64, dtype=torch.int32, device="cuda")[: g.nvec * g.width]
    vw.copy_(g.vw)
g2 = dv.DeviceGraph.from_lanes(g.n, g.width, g.edges, g.nvec, dev["vsrc"], vw,
                               dev["voff"] if "voff" in dev else g.vector_offsets())
if g.vw8 is not None:
    g2.vw8 = dev["vw8"]
    g2._struct = None
shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
loop = dv.DeviceLoop(g2, shift, _lib.WG_VAL_U32)
init = dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32)
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
out_host = torch.empty(g.n, dtype=torch.int32).pin_memory()
iv = _initial_values(prog, g.n)
members = None if wl["app"] == "cc" else np.array([0])
fh = dv.first_hit_ok(prog.kernel, iv, members)
flags = dict(first_hit=fh, level_base=dv.first_hit_level(iv) if fh else 0, identity_init=dv.identity_values(iv))
cs = torch.cuda.Stream()
h2d = sum(v.numel() * v.element_size() for v in host.values())


def ev(label, tr):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    tr.append((label, e))


rows = []
for rep in range(5):
    tr = []
    ev("start", tr)
    g2.upload_rebuild(host, dev, chunks=chunks, copy_stream=cs, trace=tr, **kw)
    ev("rebuilt", tr)
    p = loop.seed(init, words, prog.kernel, Fraction(wl["thr"]), **flags)
    recs, conv, last = loop.drive(p, g.n + 16)
    ev("loop", tr)
    out_host.copy_(loop.values_after(last), non_blocking=True)
    ev("d2h", tr)
    p = loop.seed(init, words, prog.kernel, Fraction(wl["thr"]), **flags)
    loop.drive(p, g.n + 16)
    ev("loop again", tr)
    torch.cuda.synchronize()
    t0 = tr[0][1]
    rows.append([(lab, t0.elapsed_time(e)) for lab, e in tr])
print(f"{wl['desc']} format={fmt} chunks={chunks} placed={placed} H2D bytes={h2d}")
last = rows[-1]
for i, (lab, _) in enumerate(last):
    print(f"  {lab:>12s} {np.median([r[i][1] for r in rows[1:]]):8.3f} ms")
