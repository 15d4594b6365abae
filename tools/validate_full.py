"""Full-size parity against the reference's own compiled kernels (oracle/_ref,
16 host threads, the restated reference driver) for the BASELINE configs the
bench checks only by certificate: the 4096^2 grid SSSP (configs[2]) and the
s25 PageRank (configs[4], float64 oracle, |r_gpu - r_cpu| <= 1e-6).  Writes
the reference digests / PR error to the JSON file given as argv[1] (the
committed copy is tests/golden/full_size.json).  ~20 min of host CPU.

usage: python tools/validate_full.py out.json [grid] [pr25]
"""
import json
import os
import sys
import time
from fractions import Fraction
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
import oracle
import paper_1903_07754_b200 as wg
from paper_1903_07754_b200 import _lib, device as dv
from paper_1903_07754_b200.engine import _initial_values

out_path = sys.argv[1]
which = sys.argv[2:] or ["grid", "pr25"]
threads = os.cpu_count() or 1
res = json.loads(Path(out_path).read_text()) if Path(out_path).exists() else {}

if "grid" in which:
    wl = bench.WORKLOADS["sssp_grid"]
    el, topo = bench.make_graph(wl)
    g = topo.device
    prog = wg.make_program("sssp", 0)
    loop = dv.DeviceLoop(g, 2, _lib.WG_VAL_U32)
    p = loop.seed(dv.encode_values(_initial_values(prog, g.n), _lib.WG_VAL_U32), dv.initial_words(g.n, np.array([0])),
                  prog.kernel, Fraction(wl["thr"]))
    recs, conv, last = loop.drive(p, g.n + 16)
    gpu = dv.values_to_int64(loop.values_after(last), _lib.WG_VAL_U32)
    tp, idx, deg = bench.host_reference_layout(g)
    be = oracle.RefBackend(threads) if oracle.ref_kernels() is not None else oracle.PortBackend(threads)
    init, front = oracle.initial_state("sssp", g.n, 0)
    t0 = time.perf_counter()
    ref = oracle.run_until_convergence(tp, idx, deg, oracle.kern_of("sssp"), init, front, Fraction(wl["thr"]),
                                       wl["vpg"], g.n + 16, backend=be)
    t = time.perf_counter() - t0
    trace_ok = [(r.mode, r.active_edges, r.frontier_out_size) for r in recs] == \
               [(s[1], s[2], s[3]) for s in oracle.trace(ref.stats)]
    res["sssp_grid"] = {"reference_digest": oracle.result_digest(ref.values), "gpu_digest": wg.result_digest(gpu),
                        "equal": bool(np.array_equal(ref.values, gpu)), "iterations": len(ref.stats),
                        "trace_equal": bool(trace_ok), "reference_seconds": round(t, 1),
                        "backend": type(be).__name__, "threads": threads}
    print("grid", res["sssp_grid"], flush=True)
    Path(out_path).write_text(json.dumps(res, indent=1))

if "pr25" in which:
    wl = bench.WORKLOADS["pr25"]
    el, topo = bench.make_graph(wl)
    g = topo.device
    r = dv.pagerank(g, 20, 0.85).cpu().numpy().astype(np.float64)
    tp, idx, deg = bench.host_reference_layout(g)
    t0 = time.perf_counter()
    ref = oracle.pagerank(tp, deg, 20, 0.85, threads)
    t = time.perf_counter() - t0
    err = float(np.max(np.abs(r - ref)))
    res["pr25"] = {"max_abs_error": err, "tolerance": 1e-6, "ok": err <= 1e-6, "sum_gpu": float(r.sum()),
                   "oracle": "oracle.pagerank (float64 C port)", "oracle_seconds": round(t, 1)}
    print("pr25", res["pr25"], flush=True)
    Path(out_path).write_text(json.dumps(res, indent=1))
