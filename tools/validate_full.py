"""Full-size reference results, independent of the product: the UNMODIFIED
reference driver (wedgegraph.run_until_convergence, engine.py:330-388, native
backend, every host core) from baseline/_ref on inputs built by the oracle's
restated generators and layout builders (oracle/, pinned against the
reference's own outputs by tests/test_oracle.py) -- no device code involved.
Records each workload's result digest and per-iteration trace
(iteration, mode, active_edges, frontier_out) into the JSON file given as
argv[1] (the committed copy is tests/golden/full_size.json), which
tests/test_gpu_large.py checks the device engine against.

Runs on the GPU box's host (196 GB RAM, 16 cores); s26 needs ~40 GB.
usage: python tools/validate_full.py out.json cc22 bfs26 sssp26 [sssp_grid]
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402  (workload table + reference-arm helpers; imports no product code)

out_path = Path(sys.argv[1])
which = sys.argv[2:] or ["cc22", "bfs26", "sssp26"]
res = json.loads(out_path.read_text()) if out_path.exists() else {}
ref, why = bench.import_reference()
if ref is None:
    sys.exit(f"reference unavailable: {why}")
threads = os.cpu_count() or 1
for name in which:
    wl = bench.WORKLOADS[name]
    t0 = time.perf_counter()
    n, E, tp, idx, deg, _ = bench.prepare_reference_input(wl)
    prep = time.perf_counter() - t0
    topo = ref.PullTopology(n, 4, E, tp.vec_dst, tp.lane_src, tp.lane_weight, tp.lane_count)
    index = ref.EdgeIndex(n, tp.vector_count, idx.offsets, idx.positions)
    prog = ref.make_program(wl["app"], None if wl["app"] == "cc" else 0)
    cfg = ref.EngineConfig(threshold=ref.FullnessThreshold.of(wl["thr"]),
                           precision=ref.FrontierPrecision(wl["vpg"]), workers=threads, max_iterations=n + 16)
    t1 = time.perf_counter()
    out = ref.run_until_convergence(topo, index, prog, deg, cfg, backend="native")
    run = time.perf_counter() - t1
    res[name] = {
        "reference_digest": ref.result_digest(out.values), "iterations": len(out.stats),
        "converged": out.converged, "V": n, "E": E,
        "trace": [[s.iteration, s.mode, int(s.active_edges), int(s.frontier_out_size)] for s in out.stats],
        "vectors_touched": [int(s.vectors_touched) for s in out.stats],
        "source": "stock reference driver (baseline/_ref wedgegraph.run_until_convergence, native backend, "
                  f"workers={threads}) on oracle-built inputs (tools/validate_full.py)",
        "input_prep_s": round(prep, 1), "reference_seconds": round(run, 1),
    }
    print(name, res[name]["reference_digest"], len(out.stats), f"prep {prep:.0f}s run {run:.0f}s", flush=True)
    del topo, index, tp, idx, deg, out
    out_path.write_text(json.dumps(res, indent=1))
