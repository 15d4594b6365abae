import sys
from fractions import Fraction
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
import paper_1903_07754_b200 as wg
wl = bench.WORKLOADS["sssp_grid"]
el, topo = bench.make_graph(wl)
idx = wg.build_edge_index(topo)
deg = wg.compute_out_degrees(el)
cfg = wg.EngineConfig(threshold=wg.FullnessThreshold.of("0.2"), precision=wg.FrontierPrecision(4), max_iterations=100000)
r = wg.run_until_convergence(topo, idx, wg.sssp_program(0), deg, cfg)
a = np.array([s.active_edges for s in r.stats]); f = np.array([s.frontier_out_size for s in r.stats])
t = np.array([s.vectors_touched for s in r.stats])
print("iters", len(a), "device_ms", r.device_ms)
for q in (0, 10, 25, 50, 75, 90, 99, 100):
    print(q, "active_edges", int(np.percentile(a, q)), "frontier", int(np.percentile(f, q)), "touched", int(np.percentile(t, q)))
print("sum active", a.sum(), "sum touched", t.sum())
