"""Per-phase timing of the packed sharded loop (run under torchrun, one
process per GPU): host time of step (loop kernels + wg_exchange_pack_all),
the all-gather, and apply (wg_exchange_apply_all + record read), each
followed by a synchronize.  usage: torchrun ... tools/shard_prof.py [cc22]"""
import os
import sys
import time
from fractions import Fraction
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import torch.distributed as dist

import bench
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, distributed as D

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cc22"]
el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=wl["scale"], edge_factor=wl["ef"], seed=1)),
                              wl["sym"])
s, d, w = el.device_arrays()
n = el.vertex_count
indeg = torch.bincount(d.to(torch.int64) & 0xFFFFFFFF, minlength=n).cpu().numpy()
bounds = D.destination_bounds(indeg, 4, world)
prog = wg.make_program(wl["app"], None if wl["app"] == "cc" else 0)
shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
sh = D.DeviceShard(n, s, d, w, 4, bounds, rank, prog.kernel, prog.initial_values(n),
                   None if wl["app"] == "cc" else np.array([0]), Fraction(wl["thr"]), shift, _lib.WG_VAL_U32)
rows = []
for rep in range(4):
    sh.seed()
    cap = sh.capacity
    per = []
    for it in range(1, 10000):
        t0 = time.perf_counter()
        sh.step(it)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        nb = sh.message_bytes(cap)
        recv = sh.recv[: world * nb]
        dist.all_gather_into_tensor(recv, sh.send[:nb])
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rec, maxc = sh.apply_packed(it, recv, world, cap)
        t3 = time.perf_counter()
        per.append((t1 - t0, t2 - t1, t3 - t2))
        cap = min(sh.capacity, max(D.PACKED_MIN_CAP, 2 * maxc))
        if rec.out_edge_sum == 0:
            break
    if rep:
        rows.append(np.array(per).sum(axis=0))
if rank == 0:
    r = np.median(np.array(rows), axis=0) * 1000
    print(f"{wl['desc']} world={world}: step {r[0]:.3f} ms, all-gather {r[1]:.3f} ms, apply+record {r[2]:.3f} ms, "
          f"iterations {it}")
    # the same step with no synchronisation in between (as run_sharded does)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.run_sharded(sh, n + 16, values=False)
    torch.cuda.synchronize()
    print(f"run_sharded wall {1000 * (time.perf_counter() - t0):.3f} ms")
dist.destroy_process_group()
