"""Per-phase host timing of the sharded loop (run under torchrun)."""
import os, sys, time
from fractions import Fraction
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch, torch.distributed as dist
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, distributed as D
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=22, edge_factor=16, seed=1)), True)
s, d, w = el.device_arrays()
n = el.vertex_count
indeg = torch.bincount(d.to(torch.int64) & 0xFFFFFFFF, minlength=n).cpu().numpy()
bounds = D.destination_bounds(indeg, 4, world)
prog = wg.cc_program()
sh = D.DeviceShard(n, s, d, w, 4, bounds, rank, prog.kernel, prog.initial_values(n), None, Fraction(1, 5), 2,
                   _lib.WG_VAL_U32)
tm = {"step": 0.0, "gather": 0.0, "apply": 0.0}
for rep in range(3):
    sh.seed()
    for it in range(1, 20):
        t0 = time.perf_counter(); v, x = sh.step(it); torch.cuda.synchronize(); t1 = time.perf_counter()
        av = D.all_gather_var(v); ax = D.all_gather_var(x); torch.cuda.synchronize(); t2 = time.perf_counter()
        r = sh.apply(it, av, ax); torch.cuda.synchronize(); t3 = time.perf_counter()
        if rep == 2:
            tm["step"] += t1 - t0; tm["gather"] += t2 - t1; tm["apply"] += t3 - t2
        if r.out_edge_sum == 0:
            break
if rank == 0:
    print({k: round(v * 1000, 3) for k, v in tm.items()}, "iterations", it)
dist.destroy_process_group()
