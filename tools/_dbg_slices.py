import sys, ctypes
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from fractions import Fraction
import numpy as np, torch
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib
from paper_1903_07754_b200.distributed import DeviceShard, destination_bounds
import oracle
el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=13, edge_factor=16, seed=2)), True)
n = el.vertex_count; src, dst = el.src, el.dst
prog = wg.make_program("cc", None)
bounds = destination_bounds(np.bincount(dst, minlength=n), 4, 2)
init = prog.initial_values(n)
shards = [DeviceShard(n, src, dst, None, 4, bounds, r, prog.kernel, init, None, Fraction(1,5), 2, _lib.WG_VAL_U32) for r in range(2)]
for s in shards: s.seed()
topo = oracle.build_pull_topology(n, src, dst, None, 4); idx = oracle.build_edge_index(topo); deg = oracle.compute_out_degrees(n, src)
v0, front = oracle.initial_state("cc", n, 0)
vlog=[]; flog=[]
want = oracle.run_until_convergence(topo, idx, deg, oracle.CC, v0, front, Fraction(1,5), 4, value_log=vlog, frontier_log=flog)
print("want", [(s.mode, s.frontier_out_size) for s in want.stats])
L = _lib.load()
prev_sum = shards[0].initial_edge_sum()
for it in range(1, 8):
    dense = shards[0].gate_dense(prev_sum)
    for r, s in enumerate(shards):
        s.step(it)
    torch.cuda.synchronize()
    for r, s in enumerate(shards):
        lo, hi = bounds[r], bounds[r+1]
        loc = s.loop.vals[it & 1][lo:hi].cpu().numpy().view(np.uint32).astype(np.int64)
        print(f"it{it} shard{r} local owned values ok:", np.array_equal(loc, vlog[it-1][lo:hi]))
    if not dense:
        print("wedge; stop"); break
    for r, s in enumerate(shards):
        _lib.check(L.wg_exchange_slice_pack(ctypes.byref(s.g.struct()), ctypes.byref(s.loop.bufs), ctypes.byref(s.p), it, bounds[r], bounds[r+1], s.slice_send.data_ptr(), _lib.stream_ptr()))
    recv = torch.cat([s.slice_send for s in shards])
    rs = [s.apply_slices(it, recv, overflow_any=False) for s in shards]
    for r, s in enumerate(shards):
        v = s.loop.vals[it & 1].cpu().numpy().view(np.uint32).astype(np.int64)
        w = s.loop.vals[(it-1) & 1].cpu().numpy().view(np.uint32).astype(np.int64)
        print(f"  shard{r} after apply: vals ok {np.array_equal(v, vlog[it-1])} other ok {np.array_equal(w, vlog[it-1])} rec {rs[r]}")
    prev_sum = rs[0].out_edge_sum
