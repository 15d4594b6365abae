"""GPU timeline of the loop graph's kernels, per iteration (%globaltimer
stamps, wg_debug_kernel_timeline).  Usage: python tools/timeline.py cc22 [runs]
Prints, per iteration, each kernel's start offset and duration (us) relative
to the run's first stamped kernel; the last run of `runs` is reported."""
import ctypes
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

NAMES = ["decide", "sparse_gate", "transform", "group_count", "group_list", "pull_wedge", "pull_sparse",
         "dense_dst", "dense_tma", "bottom_up", "floor", "ident", "fcount", "flist", "finalize", "step",
         "seed", "persistent"]
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cc22"]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
el, topo = bench.make_graph(wl)
g = topo.device
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
loop = dv.DeviceLoop(g, shift, _lib.WG_VAL_U32)
iv = dv.prepare_initial_values(_initial_values(prog, g.n), prog.kernel,
                               None if wl["app"] == "cc" else np.array([0]))
words = dv.all_words(g.n) if wl["app"] == "cc" else dv.initial_words(g.n, np.array([0]))
L = _lib.load()
K = int(L.wg_debug_kernel_ids())
CAP = 64
buf = torch.empty(CAP * K * 2, dtype=torch.int64, device="cuda")
phases = torch.zeros(CAP * 4, dtype=torch.int64, device="cuda")  # persistent-loop phase stamps
for r in range(runs):
    v = buf.view(CAP, K, 2)
    v[:, :, 0] = -1  # ~0 as uint64
    v[:, :, 1] = 0
    torch.cuda.synchronize()
    _lib.check(L.wg_debug_kernel_timeline(buf.data_ptr() if r == runs - 1 else None, CAP))
    phases.zero_()
    _lib.check(L.wg_debug_phase_buffer(phases.data_ptr() if r == runs - 1 else None, CAP))
    p = loop.seed(iv.seed(_lib.WG_VAL_U32), words, prog.kernel, Fraction(wl["thr"]), first_hit=iv.first_hit,
                  level_base=iv.level_base, identity_init=iv.identity, defer=True)
    recs, conv, last = loop.drive(p, g.n + 16)
    torch.cuda.synchronize()
_lib.check(L.wg_debug_kernel_timeline(None, 0))
_lib.check(L.wg_debug_phase_buffer(None, 0))
ph = phases.view(CAP, 4).cpu().numpy()
a = buf.view(CAP, K, 2).cpu().numpy().view(np.uint64)
stamped = a[:, :, 1] > 0
t0 = a[:, :, 0][stamped].min()
print(f"{wl['desc']}: {len(recs)} iterations; us relative to the first stamped kernel")
prev_end = t0
for it in range(0, min(len(recs) + 2, CAP)):
    row = [(NAMES[k], (int(a[it, k, 0]) - t0) / 1e3, (int(a[it, k, 1]) - int(a[it, k, 0])) / 1e3)
           for k in range(K) if a[it, k, 1] > 0]
    if not row:
        continue
    row.sort(key=lambda x: x[1])
    end = max(s + d for _, s, d in row)
    mode = recs[it - 1].mode if it - 1 < len(recs) else "-"
    print(f"it {it:3d} {mode:8s} [{row[0][1]:8.1f} .. {end:8.1f}] = {end - row[0][1]:7.1f} us")
    for nme, s, d in row:
        print(f"      {nme:12s} start {s:8.1f}  dur {d:7.1f}")

print("persistent-loop phases (stamps 0..3 per iteration, us relative to the first stamped kernel):")
for it in range(1, CAP):
    if ph[it, 0] == 0:
        continue
    st = [(int(x) - int(t0)) / 1e3 for x in ph[it]]
    print(f"it {it:3d} " + "  ".join(f"{x:8.1f}" for x in st) + "   deltas " +
          "  ".join(f"{st[i + 1] - st[i]:6.1f}" for i in range(3)))
