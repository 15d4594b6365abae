"""Host-side breakdown of one bench step (seeded loop-graph launch + record
read-back): where the wall time of a small run goes.
usage: python tools/step_breakdown.py bfs16 [steps]"""
import ctypes
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
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
thr = Fraction(wl["thr"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()


def step():
    p = loop.seed(dinit, words, prog.kernel, thr, first_hit=fh, level_base=lvl, identity_init=ident, defer=True)
    return loop.drive(p, g.n + 16)


for _ in range(50):
    step()
torch.cuda.synchronize()

# (1) back-to-back steps, no flush: wall per step and GPU event per step
t0 = time.perf_counter()
for _ in range(steps):
    step()
torch.cuda.synchronize()
print(f"wall per step, back to back: {1e6 * (time.perf_counter() - t0) / steps:.1f} us")

# (2) the bench's own measurement (flush + events around the step)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for k in range(steps):
    flush.fill_(k & 0xFF)
    ev[k][0].record(stream)
    step()
    ev[k][1].record(stream)
torch.cuda.synchronize()
ms = np.array([a.elapsed_time(b) for a, b in ev])
print(f"bench-style event time per step (L2 flushed): mean {1e3 * ms.mean():.1f} us  p50 {1e3 * np.median(ms):.1f} us")

# (3) the same with the flush finished before the step starts (host not hidden)
for k in range(steps):
    flush.fill_(k & 0xFF)
    torch.cuda.synchronize()
    ev[k][0].record(stream)
    step()
    ev[k][1].record(stream)
torch.cuda.synchronize()
ms = np.array([a.elapsed_time(b) for a, b in ev])
print(f"event time per step, flush synchronised first: mean {1e3 * ms.mean():.1f} us  p50 {1e3 * np.median(ms):.1f} us")

# (4) host phases of a step (perf_counter, us): seed / launch / sync+copy / parse
L = _lib.load()
acc = np.zeros(4)
for k in range(steps):
    a = time.perf_counter()
    p = loop.seed(dinit, words, prog.kernel, thr, first_hit=fh, level_base=lvl, identity_init=ident, defer=True)
    b = time.perf_counter()
    pending = loop._pending
    loop._pending = None
    init_values, init_words, counts = pending
    exe0 = loop._graph_for(p, None, seeded=("all" if counts is not None else "words", counts))
    sv, sw = loop._seed_buffers(init_words.numel())
    _lib.check(L.wg_run_loop_launch_seeded(exe0, ctypes.byref(loop.bufs), g.n + 16, dv._ptr(init_values), dv._ptr(sv),
                                           g.n * init_values.element_size(), dv._ptr(init_words), dv._ptr(sw),
                                           min(init_words.numel(), sw.numel()) * 4, _lib.stream_ptr(None)))
    c = time.perf_counter()
    head = 4 + dv.HEAD_RECORDS * dv.REC_U64
    loop.host_state[:head].copy_(loop.state[:head], non_blocking=True)
    stream.synchronize()
    d = time.perf_counter()
    hs = loop._host_np
    done = int(hs[0])
    rows = hs[4:].reshape(loop.ring, dv.REC_U64)[1: 1 + done].tolist()
    recs = []
    loop._parse(rows, 1, recs, None)
    e = time.perf_counter()
    acc += [b - a, c - b, d - c, e - d]
print("host phases per step (us): seed %.1f  graph launch call %.1f  copies+sync (GPU run inside) %.1f  parse %.1f"
      % tuple(1e6 * acc / steps))
