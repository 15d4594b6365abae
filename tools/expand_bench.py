"""Time wg_expand_destinations on the CC s22 layout."""
import sys, torch, numpy as np
sys.path.insert(0,'/root/repo')
import bench
from paper_1903_07754_b200 import _lib
wl = bench.WORKLOADS["cc22"]
el, topo = bench.make_graph(wl)
g = topo.device
L = _lib.load()
voff = g.vector_offsets()
out = torch.empty_like(g.vdst)
scr = torch.empty(int(L.wg_expand_scratch_bytes(g.nvec)), dtype=torch.uint8, device="cuda")
for rep in range(5):
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(L.wg_expand_destinations(g.n, voff.data_ptr(), g.nvec, out.data_ptr(), scr.data_ptr(), scr.numel(),
                                         _lib.stream_ptr()))
    b.record(); torch.cuda.synchronize()
    print("expand ms", a.elapsed_time(b), torch.equal(out, g.vdst))
v = voff.cpu().numpy().astype(np.int64)
runs = np.diff(v)
print("max run", runs.max(), "argmax", runs.argmax())
