"""GPU-side time of the chunked index build on resident data (the host
enqueue is hidden behind a sleep kernel), per chunk count.
usage: python tools/index_chunk_bench.py [workload]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_1903_07754_b200 import _lib, device as dv

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cc22"]
el, topo = bench.make_graph(wl)
g = topo.device
L = _lib.load()
W = g.width
enc = g.encode_lanes()
voff = g.vector_offsets()
for chunks in (1, 2, 4, 8, 16):
    align = _lib.WG_CODED_BLOCK_VECTORS
    cuts = [min(g.nvec, (g.nvec * c // chunks) // align * align) for c in range(chunks)] + [g.nvec]
    max_lanes = max(max(cuts[c + 1] - cuts[c] for c in range(chunks)) * W, 1)
    need = max(int(L.wg_index_chunked_scratch_bytes(g.nvec * W, max_lanes, g.n)),
               int(L.wg_index_scratch_bytes(g.nvec * W, g.n)))
    scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    gs = ctypes.byref(g.struct())
    res = []
    for rep in range(4):
        torch.cuda.synchronize()
        torch.cuda._sleep(100_000_000)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(chunks + 2)]
        e[0].record()
        for c in range(chunks):
            _lib.check(L.wg_index_chunk_coded(gs, enc["lane_stream"].data_ptr(), enc["lane_widths"].data_ptr(),
                                              enc["lane_blocks"].data_ptr(), cuts[c] // align,
                                              -(-cuts[c + 1] // align), c, max_lanes, scratch.data_ptr(),
                                              scratch.numel(), _lib.stream_ptr()))
            e[c + 1].record()
        ent = ctypes.c_uint64(0)
        _lib.check(L.wg_index_finish(gs, max_lanes, g.idx_off.data_ptr(), g.idx_pos.data_ptr(), g.outdeg.data_ptr(),
                                     scratch.data_ptr(), scratch.numel(), ctypes.byref(ent), _lib.stream_ptr()))
        e[-1].record()
        torch.cuda.synchronize()
        res.append([e[0].elapsed_time(x) for x in e[1:]])
    r = np.median(np.array(res[1:]), axis=0)
    per = np.diff(np.r_[0, r[:-1]])
    print(f"chunks={chunks:2d} total {r[-1]:.3f} ms  per-chunk {np.round(per, 3).tolist()}  finish {r[-1] - r[-2]:.3f}")
