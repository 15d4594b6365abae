"""Benchmark of the B200 Wedge-Frontier pull engine (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload cc22|bfs16|sssp_grid|pr25|bfs26|sssp26]

Default workload (BASELINE.json configs[1], the metric's reference config):
Connected Components on RMAT scale 22, edge factor 16, (a,b,c,d) =
(.57,.19,.19,.05), seed 1, self-loops removed, symmetrised + de-duplicated,
W=4 vectors, Wedge precision 4 vectors/bit, fullness threshold 1/5 (the
reference CLI defaults, cli.py:52-56).  Inputs are generated on the device with
the reference's own PCG64 stream (bit-identical, tests/test_gpu_parity.py).

A step = one run to convergence (time-to-solution, TTS) with the graph
resident in HBM; value = GTEPS = |E| / TTS.  The graph (>= 600 MB) is larger
than the 126 MB L2 and L2 is additionally flushed (256 MB write) between
timed steps.  e2e = the same run through the C ABI with the layout in pinned
host memory: H2D of the layout + loop + D2H of the labels, per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from fractions import Fraction
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "cc22": dict(app="cc", scale=22, ef=16, sym=True, vpg=4, thr="0.2", weights=None,
                 desc="CC on symmetrized RMAT s22 ef16 (BASELINE configs[1])",
                 expect_digest="a9b4aaec4bde3218"),
    "bfs16": dict(app="bfs", scale=16, ef=16, sym=True, vpg=8, thr="0.01", weights=None,
                  desc="BFS on symmetrized RMAT s16 ef16 (BASELINE configs[0])",
                  expect_digest="591673cb243fad4e"),
    "sssp16": dict(app="sssp", scale=16, ef=16, sym=True, vpg=4, thr="0.2", weights=255,
                   desc="SSSP on symmetrized RMAT s16 ef16, hash weights <= 255",
                   expect_digest="7d2c2554722fbf74"),
    # expected digests of the full-size configs: the reference's own kernels
    # on the same inputs (tests/golden/full_size.json)
    "sssp_grid": dict(app="sssp", grid=(4096, 4096), vpg=4, thr="0.2", iterations=8627, ref_iteration_cap=64,
                      desc="SSSP on 4096x4096 grid, p=0.9, w in [1,1000] (BASELINE configs[2])",
                      expect_digest="3895390ac91e5500"),
    "bfs26": dict(app="bfs", scale=26, ef=16, sym=False, vpg=8, thr="0.01", weights=None,
                  desc="BFS on directed dedup RMAT s26 ef16 (BASELINE configs[3])",
                  expect_digest="8494a0a1f8a0196d"),
    "sssp26": dict(app="sssp", scale=26, ef=16, sym=False, vpg=4, thr="0.2", weights=255,
                   desc="SSSP on directed dedup RMAT s26 ef16, w<=255 (BASELINE configs[3])",
                   expect_digest="184036ba61690aac"),
    "pr25": dict(app="pr", scale=25, ef=32, sym=False, desc="PageRank 20 it on directed dedup RMAT s25 ef32 "
                 "(BASELINE configs[4])"),
}
GRID_SEED = 2
METRIC = "GTEPS"
DATA_DESC = "synthetic (seeded RMAT on the reference's PCG64 stream / fixed-seed grid)"
L2_NOTE = "inputs larger than L2 + 256 MB L2 flush between timed steps"


def workload_config(wl, n, E):
    """The `config` object, identical in both arms (static workload keys only;
    run-specific figures go to `run`)."""
    return {"workload": wl["desc"], "app": wl["app"], "V": int(n), "E": int(E), "W": 4,
            "vpg": wl.get("vpg"), "threshold": wl.get("thr"), "l2": L2_NOTE}


def rle_modes(recs) -> str:
    """Mode sequence, run-length encoded: e.g. "F3W3" (FullScan x3, Wedge x3)."""
    out, prev, cnt = [], None, 0
    for r in recs:
        m = "W" if r.mode == "Wedge" else "F"
        if m == prev:
            cnt += 1
        else:
            if prev:
                out.append(f"{prev}{cnt}")
            prev, cnt = m, 1
    if prev:
        out.append(f"{prev}{cnt}")
    return "".join(out)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    (sub-millisecond queries, a sample every ~1 ms) with an nvidia-smi
    fallback (a sample every 0.2 s)."""

    # NVML clocks-event-reason bits (nvmlClocksEventReason*)
    NVML_REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                    "hw_thermal_slowdown": 0x40}
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, set of reasons)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((float(sm), float(mx), {k for k, b in self.NVML_REASONS.items() if bits & b}))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if out:
            r = [x.strip() for x in out.split(",")]
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            num = lambda x: float(x) if x.replace(".", "").isdigit() else None
            self.rows.append((num(r[0]), num(r[1]),
                              {names[i] for i in range(4) if len(r) > 3 + i and r[3 + i].lower() == "active"}))

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:
                pass
            # 20 ms: every NVML query takes driver locks that the timed steps' graph
            # launches also need (a 1 ms poll added ~0.1 ms to a 0.25 ms BFS s16
            # step); tick() samples between steps as well
            self._stop.wait(0.02 if self._nvml else 0.2)

    def tick(self, min_interval: float = 0.004):
        """Synchronous sample between timed steps (the timed region of a small
        workload is shorter than the sampler thread's period) -- at most one per
        min_interval: an NVML query idles the GPU for ~1 ms, and a step that
        starts on an idled GPU measured 0.33 ms where back-to-back steps take
        0.17 ms (BFS s16)."""
        now = time.perf_counter()
        if now - getattr(self, "_last_tick", 0.0) < min_interval:
            return
        self._last_tick = now
        try:
            if self._nvml:
                self._sample_nvml()
        except Exception:
            pass

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows if r[0] is not None]
        mx = [r[1] for r in self.rows if r[1] is not None]
        reasons = sorted(set().union(*(r[2] for r in self.rows)))
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self._nvml else "nvidia-smi"}


# -------------------------------------------------------------- workload --
def gather_peak():
    """Measured ceiling of one-gather-per-edge kernels (tools/microbench_sector.cu,
    profiles/gather_peak.json): random 4-byte gathers per second when every
    gather needs its own 32-byte sector from L2 -- an SM's L1 sends about one
    sector request per cycle to the crossbar, whatever the table size."""
    try:
        return float(json.loads((ROOT / "profiles" / "gather_peak.json").read_text())["l2_resident_gathers_per_s"])
    except Exception:
        return 148 * 1.965e9


def gather_roofline(gathers, ms):
    """Second roofline of a pull: its random gathers against gather_peak()."""
    pk = gather_peak()
    rate = gathers / (ms * 1e-3) if ms else 0.0
    return {"bound": "L1->crossbar sector requests (one 4-byte gather per 32-byte sector)",
            "gathers_per_launch": int(gathers), "achieved_ggathers_s": round(rate / 1e9, 1),
            "peak_ggathers_s": round(pk / 1e9, 1), "frac": round(rate / pk, 4),
            "peak_source": "measured, tools/microbench_sector.cu (profiles/r02_microbench_sector.txt)",
            "hbm_equivalent": "at 4 useful bytes per 32-byte sector this ceiling is %.2f of the HBM copy peak"
                              % (4 * pk / 1e9 / peaks()[0])}


def make_graph(wl, width=4):
    import paper_1903_07754_b200 as wg
    if "grid" in wl:
        el = wg.grid_graph(wl["grid"][0], wl["grid"][1], GRID_SEED, 0.9, 1000)
    else:
        el = wg.generate(wg.GenSpec("rmat", scale=wl["scale"], edge_factor=wl["ef"], seed=1))
        el = wg.drop_self_loops_dedup(el, symmetric=wl["sym"])
        if wl.get("weights"):
            el = wg.synthesize_weights(el, wl["weights"])
    topo = wg.build_pull_topology(el, width)
    return el, topo


def run_b200(args, wl):
    import torch
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib, device as dv
    from paper_1903_07754_b200.engine import _initial_values

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if world > 1 or args.sharded:
        return run_b200_sharded(args, wl, rank, world, local)

    t0 = time.perf_counter()
    el, topo = make_graph(wl)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    g = topo.device
    n, E = g.n, g.edges
    log(f"[bench] built {wl['desc']}: V={n} E={E} nvec={g.nvec} entries={g.entries} in {build_s:.1f}s "
        f"({g.memory_bytes() / 1e9:.2f} GB layout)")

    if wl["app"] == "pr":
        return run_pagerank(args, wl, el, topo, build_s)

    app = wl["app"]
    root = 0
    prog = wg.make_program(app, None if app == "cc" else root)
    kern = prog.kernel
    thr = Fraction(wl["thr"])
    shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
    init = _initial_values(prog, n)
    loop = dv.DeviceLoop(g, shift, _lib.WG_VAL_U32)
    dinit = dv.encode_values(init, _lib.WG_VAL_U32)
    words = dv.all_words(n) if app == "cc" else dv.initial_words(n, np.array([root]))
    max_it = n + 16  # cli.py:162
    # BFS is level-synchronous: first-hit early exit in the filtered pulls
    fh = dv.first_hit_ok(kern, init, None if app == "cc" else np.array([root]))
    lvl = dv.first_hit_level(init) if fh else 0
    ident = dv.identity_values(init)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step(timer=None):
        # deferred: the seed runs as the loop graph's prologue (one launch per run)
        p = loop.seed(dinit, words, kern, thr, first_hit=fh, level_base=lvl, identity_init=ident, defer=True)
        if timer is not None:
            p.timer = timer.handle
        return loop.drive(p, max_it)

    # clock ramp: small workloads (C1: 0.4 ms per step) would otherwise time
    # steps taken before the SMs leave their idle clocks; untimed, like the
    # warm-up steps that follow
    t_ramp = time.perf_counter()
    while time.perf_counter() - t_ramp < float(os.environ.get("WG_RAMP_S", "1.0")):
        step()
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        recs, conv, last = step()
    torch.cuda.synchronize()
    values = dv.values_to_int64(loop.values_after(last), _lib.WG_VAL_U32)
    digest = wg.result_digest(values)
    cert = certificate(el, values, app)
    iters = len(recs)
    modes = rle_modes(recs)
    log(f"[bench] {iters} iterations ({modes}), converged={conv}, digest={digest}")

    # ---- timed region: K steps, events per step, L2 flushed in between ----
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            clk.tick()
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    launches = _lib.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    gteps = E * world / (ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (pull), CUDA events per launch ----
    timer = _lib.EventTimer(8 * (iters + 8))
    flush.fill_(1)
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    recs_t, _, _ = step(timer)
    torch.cuda.synchronize()
    kernels_per_step = _lib.launch_count() - l0  # launched one by one here (no graph)
    rows = timer.read()
    roof = roofline(rows, recs_t, n, E, g.weighted(), kern.filter_unvisited, wl)

    out = {
        "metric": METRIC, "value": round(gteps, 4), "unit": "GTEPS (|E|/time-to-solution)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": DATA_DESC,
        "config": workload_config(wl, n, E),
        "run": {"iterations": iters, "modes": modes, "parallelism": "1 GPU", "build_s": round(build_s, 2),
                "tts_ms": round(ms, 4)},
        "parity": {"digest": digest, "expected": wl.get("expect_digest"),
                   "ok": (digest == wl["expect_digest"]) if wl.get("expect_digest") else cert["ok"],
                   "certificate": cert},
        "gpu_launches": int(launches),
        "gpu_launches_note": ("host-side launches in the timed region: per step the seed kernels and ONE "
                              "conditional CUDA graph launch; the graph then runs the loop's kernels "
                              f"({int(kernels_per_step)} per step when launched one by one, "
                              "early-exiting ones included)"),
        "timed_wall_s": round(wall, 3),
        "roofline": roof,
    }
    clocks = clk.summary()
    out["clocks"] = clocks
    if rank == 0 and not args.no_e2e:
        out["e2e"] = e2e_api(args, wl, g, prog, values)
        if args.e2e_compact:
            out["e2e_compact"] = e2e_b200(args, wl, g, loop, dinit, words, kern, thr, max_it, fh, lvl, ident)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, args)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_b200_sharded(args, wl, rank, world, local):
    """N GPUs: destination-range shards of the same graph (strong scaling),
    per-iteration exchange of updated values by NCCL all-gather; the time of
    a step is the max over ranks (CUDA events on each rank's stream)."""
    import torch
    import torch.distributed as dist
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib
    from paper_1903_07754_b200.distributed import DeviceShard, destination_bounds, run_sharded
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    t0 = time.perf_counter()
    app = wl["app"]
    local_edges = None
    from paper_1903_07754_b200 import device as dv
    if "grid" in wl or app == "pr":
        if "grid" in wl:
            el = wg.grid_graph(wl["grid"][0], wl["grid"][1], GRID_SEED, 0.9, 1000)
        else:
            el = wg.drop_self_loops_dedup(wg.generate(wg.GenSpec("rmat", scale=wl["scale"], edge_factor=wl["ef"],
                                                                 seed=1)), symmetric=wl["sym"])
        s, d, w = el.device_arrays()
        n, E = el.vertex_count, el.edge_count
        indeg = torch.bincount(d.to(torch.int64) & 0xFFFFFFFF, minlength=n).cpu().numpy()
        bounds = destination_bounds(indeg, 4, world)
    else:
        # partitioned ingest: each rank generates 1/N of the edge stream and
        # receives the edges of its destination range (no rank holds all E)
        from paper_1903_07754_b200.distributed import rmat_partitioned
        n, E, bounds, s, d, outdeg = rmat_partitioned(wl["scale"], wl["ef"], 1, wl["sym"])
        w = None
        if wl.get("weights"):
            w = dv.weights_hash(s, d, wl["weights"])  # synthesize_weights (graph_io.py:205-221) per edge
        local_edges = (E, outdeg)
    if app == "pr":
        return run_pagerank_sharded_bench(args, wl, rank, world, local, n, E, s, d, bounds, t0)
    prog = wg.make_program(app, None if app == "cc" else 0)
    shift = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[wl["vpg"]]
    shard = DeviceShard(n, s, d, w, 4, bounds, rank, prog.kernel, prog.initial_values(n),
                        None if app == "cc" else np.array([0]), Fraction(wl["thr"]), shift, _lib.WG_VAL_U32,
                        local=local_edges)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    max_it = n + 16
    for _ in range(args.warmup):
        vals, recs, conv = run_sharded(shard, max_it)
    digest = wg.result_digest(vals)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    stream = torch.cuda.current_stream()
    ts = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)  # L2 flush between timed steps, like the single-GPU path
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _, recs, conv = run_sharded(shard, max_it, values=False)
            b.record(stream)
            clk.tick()
            b.synchronize()
            ts.append(a.elapsed_time(b))
    dist.barrier()
    launches = _lib.launch_count() - launches0
    t = torch.tensor([float(np.mean(ts))], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    out = {
        "metric": METRIC, "value": round(E / (ms * 1e-3) / 1e9, 4), "unit": "GTEPS (|E|/time-to-solution)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (device RMAT, reference PCG64 stream)",
        "config": {"workload": wl["desc"], "app": app, "V": n, "E": E, "W": 4, "vpg": wl["vpg"],
                   "threshold": wl["thr"], "iterations": len(recs), "parallelism": f"dst-shard x{world}",
                   "bounds": bounds, "build_s": round(build_s, 2), "l2": L2_NOTE},
        "parity": {"digest": digest, "expected": wl.get("expect_digest"),
                   "ok": (digest == wl["expect_digest"]) if wl.get("expect_digest") else None},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def run_pagerank_sharded_bench(args, wl, rank, world, local, n, E, s, d, bounds, t0):
    """PageRank over destination shards: per iteration one NCCL all-gather of
    the padded per-rank sum slices (paper_1903_07754_b200.distributed)."""
    import torch
    import torch.distributed as dist
    from paper_1903_07754_b200 import _lib
    from paper_1903_07754_b200.distributed import DevicePageRankShard, run_pagerank_sharded
    shard = DevicePageRankShard(n, s, d, 4, bounds, rank)
    del s, d
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        r = run_pagerank_sharded(shard, 20)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    stream = torch.cuda.current_stream()
    ts = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r = run_pagerank_sharded(shard, 20)
            b.record(stream)
            clk.tick()
            b.synchronize()
            ts.append(a.elapsed_time(b))
    dist.barrier()
    launches = _lib.launch_count() - launches0
    t = torch.tensor([float(np.mean(ts))], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    out = {
        "metric": METRIC, "value": round(20 * E / (ms * 1e-3) / 1e9, 4), "unit": "GTEPS (20*|E|/time, PageRank)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl["desc"], "V": n, "E": E, "W": 4, "parallelism": f"dst-shard x{world}",
                   "bounds": bounds, "build_s": round(build_s, 2), "l2": "inputs larger than L2"},
        "parity": {"rank_sum": float(r.double().sum().item()), "sum_ok": abs(float(r.double().sum()) - 1) < 1e-3},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def certificate(el, values, app):
    """Size-independent correctness certificate of the final values on the GPU.
    BFS/SSSP: d[v] <= d[u] + w(u,v) on every edge and every reached vertex
    except the root has a tight in-edge.  CC: labels agree across every edge,
    label(v) <= v and every label is its own label (a component minimum)."""
    import torch
    s, d, w = el.device_arrays()
    s = s.to(torch.int64) & 0xFFFFFFFF
    d = d.to(torch.int64) & 0xFFFFFFFF
    v = torch.from_numpy(np.ascontiguousarray(values)).cuda()
    if app == "cc":
        ids = torch.arange(v.numel(), device="cuda")
        bad = int((v[s] != v[d]).sum()) + int((v > ids).sum()) + int((v[v] != v).sum())
        return {"kind": "cc-labels", "violations": bad, "ok": bad == 0}
    INF = 1 << 62
    fin = v[s] != INF
    step = (w.to(torch.int64) & 0xFFFFFFFF) if app == "sssp" else torch.ones_like(s)
    cand = v[s] + step
    viol = int((fin & (cand < v[d])).sum())
    tight = torch.zeros(v.numel(), dtype=torch.bool, device="cuda")
    tight[d[fin & (cand == v[d])]] = True
    reached = v != INF
    reached[0] = False
    untight = int((reached & ~tight).sum())
    return {"kind": f"{app}-distances", "violated_edges": viol, "untight_vertices": untight,
            "reached": int(reached.sum()) + 1, "ok": viol == 0 and untight == 0}


def roofline(rows, recs, n, E, weighted, filt, wl):
    """Roofline of the dominant kernel: achieved = algorithmic bytes of its
    launches / their CUDA-event durations (per launch, on the launching
    stream: the library's timer, one iteration per launch group).

    Algorithmic bytes (uint32 ids/values, w = 1 if weighted):
    * destination-major dense pull (dense_dst_kernel; CC floor / BFS
      bottom-up): what that algorithm must touch -- prev[d], voff[d..d+1],
      nxt[d] and the next-frontier bit of every vertex (12V + V/8), the lanes
      it reads and the values / frontier bits it gathers (4 B each, device
      counters lanes_read / gathers) and the out-degree of each produced
      member (4U).  The 8(d) dense formula (every in-edge of every processed
      destination) does not describe it: a destination decided by its first
      lane (floor 0 / first frontier hit) provably needs none of its other
      lanes.
    * TMA dense pull: 4*E_p*(1+w) + 4V + 4U + V/8 (E_p = E, or the lanes of
      unvisited destinations when filtered).
    * Wedge iteration (transform + pull): 4A(1+w) + 4|F| + 4U + V/8 + [V/8 +
      8|F| + 4A]."""
    peak, peak_src = peaks()
    by_it = {}
    for kind, it, ms in rows:
        d = by_it.setdefault(it, {})
        d[kind] = d.get(kind, 0.0) + ms
    w = 1 if weighted else 0
    kern = {"dense_dst": [0.0, 0.0, 0], "dense_tma": [0.0, 0.0, 0], "wedge": [0.0, 0.0, 0]}
    step_t = 0.0
    prev_out = None
    per_iter = []
    for r in recs:
        t = by_it.get(r.iteration, {})
        pull_ms, prep_ms = t.get(2, 0.0), t.get(1, 0.0)
        fin_ms = t.get(3, 0.0) + t.get(4, 0.0)  # end of iteration (+ list build after a dense pull)
        step_t += pull_ms + prep_ms + fin_ms
        U = r.frontier_out_size
        if r.mode == "FullScan" and (r.lanes_read or r.gathers):
            name = "dense_dst"
            b = 12 * n + n / 8 + 4 * r.lanes_read + 4 * r.gathers + 4 * U
            kt = pull_ms
        elif r.mode == "FullScan":
            name = "dense_tma"
            ep = E if not filt else min(E, 4 * r.vectors_touched)
            b = 4 * ep * (1 + w) + 4 * n + 4 * U + n / 8
            kt = pull_ms
        else:
            name = "wedge"
            A = r.active_edges
            F = prev_out if prev_out is not None else 0
            b = 4 * A * (1 + w) + 4 * F + 4 * U + n / 8 + (n / 8 + 8 * F + 4 * A)
            kt = pull_ms + prep_ms
        kern[name][0] += b
        kern[name][1] += kt
        kern[name][2] += 1
        per_iter.append({"it": r.iteration, "mode": r.mode, "kernel": name, "pull_ms": round(pull_ms, 4),
                         "prep_ms": round(prep_ms, 4), "end_ms": round(fin_ms, 4), "alg_MB": round(b / 1e6, 2),
                         "lanes_read": r.lanes_read, "gathers": r.gathers})
        prev_out = U
    # dominant = the single kernel with the most time in a step (what an ncu
    # launch list ranks): a Wedge iteration is three kernels (K3 transform, K4
    # compaction, K5 pull), so it competes with its pull alone; its roofline is
    # still reported over the whole iteration (prep + pull)
    single = {"dense_dst": kern["dense_dst"][1], "dense_tma": kern["dense_tma"][1],
              "wedge": sum(x["pull_ms"] for x in per_iter if x["kernel"] == "wedge")}
    dom = max(single, key=lambda k: single[k])
    bts, ms, launches = kern[dom]
    ach = bts / (ms * 1e-3) / 1e9 if ms else 0.0
    desc = {"dense_dst": "dense_dst_kernel (destination-major dense pull%s)" % (
                ": bottom-up BFS" if filt else ": floor-probing min-label pull"),
            "dense_tma": "pull_dense_tma_kernel (K6, TMA-streamed dense pull)",
            "wedge": "transform + group compaction + wedge pull (K3+K4+K5)"}[dom]
    prof = ROOT / "profiles" / "traffic.json"
    measured_traffic = None
    if prof.exists():
        try:
            ent = json.loads(prof.read_text()).get(f"{wl['desc']}|{dom}")
            measured_traffic = ent.get("dram_bytes_per_launch") if isinstance(ent, dict) else ent
        except Exception:
            pass
    if dom == "dense_dst":
        dom_gathers = sum(r.gathers for r in recs if r.mode == "FullScan" and (r.lanes_read or r.gathers))
    elif dom == "dense_tma":
        dom_gathers = sum((E if not filt else min(E, 4 * r.vectors_touched)) for r in recs
                          if r.mode == "FullScan" and not (r.lanes_read or r.gathers))
    else:
        dom_gathers = sum(r.active_edges for r in recs if r.mode != "FullScan")
    other = {k: {"alg_MB": round(v[0] / 1e6, 2), "ms": round(v[1], 4), "launches": v[2],
                 "achieved_gbs": round(v[0] / (v[1] * 1e-3) / 1e9, 1) if v[1] else None}
             for k, v in kern.items() if v[2]}
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4), "traffic": measured_traffic, "kernel": desc,
            "peak_source": peak_src, "launches": launches,
            "algorithmic_bytes_per_launch": round(bts / max(1, launches), 1),
            "kernel_ms_per_launch": round(ms / max(1, launches), 4),
            "gather_roofline": gather_roofline(dom_gathers / max(1, launches), ms / max(1, launches)),
            "by_kernel": other, "kernel_sum_ms": round(step_t, 4),
            "per_iteration": per_iter if len(per_iter) <= 16 else per_iter[:8] + per_iter[-2:],
            "iterations_timed": len(per_iter)}


def e2e_api(args, wl, g, prog, expect_values):
    """`e2e`: the same metric through the public API call a reference user
    makes -- ``run_until_convergence(topology, index, program, degrees,
    config, backend=B200Backend(reupload=True))`` (engine.py:330-388 /
    kernels.py:137-151) -- on the reference's own host layout: int64
    PullTopology / EdgeIndex / out-degree arrays (graph.py:109-212) in pinned
    host memory.  Per step the backend copies every one of those arrays to the
    device raw (reupload: nothing cached between steps), narrows / validates
    them there (wg_ingest_*), uploads and scans the initial values, runs the
    loop and returns int64 values with the reference sentinel in host memory."""
    import torch
    import paper_1903_07754_b200 as wg

    def pinned(a):
        if a is None:
            return None
        t = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    lane_src, lane_w, lane_count = g.lanes_np()
    topo = wg.PullTopology(g.n, g.width, g.edges, pinned(g.vec_dst_np()), pinned(lane_src), pinned(lane_w),
                           pinned(lane_count))
    idx = wg.EdgeIndex(g.n, g.nvec, pinned(g.offsets_np()), pinned(g.positions_np()))
    deg = pinned(g.outdeg_np())
    del lane_src, lane_w, lane_count
    cfg = wg.EngineConfig(threshold=wg.FullnessThreshold.of(wl["thr"]),
                          precision=wg.FrontierPrecision(wl["vpg"]), max_iterations=g.n + 16)
    be = wg.B200Backend(reupload=True)
    arrays = [topo.vec_dst, topo.lane_src, topo.lane_weight, topo.lane_count, idx.offsets, idx.positions, deg]
    h2d = sum(a.nbytes for a in arrays if a is not None) + 8 * g.n  # + the int64 initial values
    d2h = 8 * g.n
    stream = torch.cuda.current_stream()
    res = None
    for _ in range(max(1, args.warmup)):
        res = wg.run_until_convergence(topo, idx, prog, deg, cfg, backend=be)
    ok = bool(np.array_equal(res.values, expect_values))
    ts, walls = [], []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        a.record(stream)
        res = wg.run_until_convergence(topo, idx, prog, deg, cfg, backend=be)
        b.record(stream)
        b.synchronize()
        walls.append(time.perf_counter() - w0)
        ts.append(a.elapsed_time(b))
    ms = float(np.mean(ts))
    ok = ok and bool(np.array_equal(res.values, expect_values))
    return {"value": round(g.edges / (ms * 1e-3) / 1e9, 4), "unit": "GTEPS (|E|/time-to-solution)",
            "ms_per_step": round(ms, 3), "wall_ms_per_step": round(1e3 * float(np.mean(walls)), 3),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "result_equal": ok,
            "device_loop_ms": round(float(res.device_ms), 4),
            "path": "wg.run_until_convergence(PullTopology(int64 host arrays), EdgeIndex(int64), program, "
                    "int64 degrees, EngineConfig, backend=B200Backend(reupload=True)): per step H2D of every "
                    "reference-layout array + initial values (pinned host memory, chunked behind the copy "
                    "engine), device narrowing/validation (wg_ingest_*, wg_values_scan), device loop, D2H of "
                    "int64 values"}


def e2e_b200(args, wl, g, loop, dinit, words, kern, thr, max_it, first_hit=False, level_base=0,
             identity_init=False):
    """`e2e_compact` (--e2e-compact): the loop through the C ABI with the graph in pinned HOST memory.
    Per step: H2D of the topology in its compact form -- the lane sources
    delta-coded per vector (wg_encode_lanes, ~15 bits per lane at s22), the
    per-destination vector offsets voff, weights as bytes when <= 255, and the
    out-degrees (the reference call's `degrees` input) -- in up to 8 chunks on
    a copy stream; on the compute stream vec_dst from voff
    (wg_expand_destinations), then per arrived chunk the lanes decoded and
    either placed into the edge index at offsets scanned from the degrees
    (wg_index_place_*, verified at the end) or sorted into it
    (wg_index_chunk_coded / wg_index_finish, for indexes over 1 GiB); then the
    device loop and the D2H of the values.
    """
    import torch
    from paper_1903_07754_b200 import _lib, device as dv

    p0 = loop.seed(dinit, words, kern, thr, first_hit=first_hit, level_base=level_base,
                   identity_init=identity_init)
    ref_vals = loop.values_after(loop.drive(p0, max_it)[2]).clone()
    # lane sources travel delta-coded (default), as wg_lane_bits(n)-bit fields
    # or as uint32 (WG_E2E_FORMAT = coded | bits | raw)
    fmt = os.environ.get("WG_E2E_FORMAT", "coded")
    if fmt == "bits" and g.lane_bits() >= 32:
        fmt = "raw"
    pack = fmt == "bits"
    # the out-degrees travel too (the reference call's `degrees` input): the
    # index is then placed chunk by chunk instead of sorted
    # (auto: while the index fits in ~8x L2; at s25/s26 its random slot writes
    # cost more than the chunk sorts, measured in profiles/r01_e2e_index.txt)
    mode = os.environ.get("WG_E2E_INDEX", "auto")
    placed = mode == "placed" or (mode == "auto" and g.edges * 4 <= (1 << 30))
    t_fmt = time.perf_counter()
    rebuild_kw = {}
    if fmt == "coded":
        # compact degrees (a byte per vertex + the large ones); a symmetric
        # input ships no out-degrees (= in-degrees, verified by the placement)
        symmetric = bool(wl.get("sym") or "grid" in wl)
        host = g.host_format(symmetric=symmetric)
        if not placed:
            host.pop("outdeg8", None)
            host.pop("outdeg_big", None)
        rebuild_kw["outdeg_is_indeg"] = symmetric and placed
    else:
        host = {"voff": g.vector_offsets().cpu().pin_memory()}
        if pack:
            host["vsrc_bits"] = g.pack_lanes()[0].cpu().pin_memory()
        else:
            host["vsrc"] = g.vsrc.cpu().pin_memory()
        if placed:
            host["outdeg"] = g.outdeg[: g.n].cpu().pin_memory()
    t_fmt = time.perf_counter() - t_fmt
    if g.vw8 is not None:  # weights <= 255 travel as bytes and are widened on the device
        host["vw8"] = g.vw8[: g.nvec * g.width].cpu().pin_memory()
    elif g.vw is not None:
        host["vw"] = g.vw.cpu().pin_memory()
    # device buffers with readable slack past the end (TMA tail rounding, wedge_b200.h)
    dev = {k: torch.empty(v.numel() + 64, dtype=v.dtype, device="cuda")[: v.numel()].view(v.shape)
           for k, v in host.items()}
    for k, v in host.items():
        dev[k].copy_(v)
    if fmt != "raw":
        dev["vsrc"] = torch.empty(g.nvec * g.width + 64, dtype=torch.int32, device="cuda")[: g.nvec * g.width]
        dev["vsrc"].copy_(g.vsrc)  # first build only; every timed step re-decodes it from the upload
    if "vw8" in dev:
        dev["vw"] = torch.empty(g.nvec * g.width + 64, dtype=torch.int32, device="cuda")[: g.nvec * g.width]
    lanes = g.nvec * g.width
    scratch = torch.empty(int(_lib.load().wg_index_scratch_bytes(g.nvec * g.width, g.n)), dtype=torch.uint8,
                          device="cuda")
    if "vw8" in dev:
        _lib.check(_lib.load().wg_widen_weights(lanes, dev["vw8"].data_ptr(), dev["vw"].data_ptr(),
                                                _lib.stream_ptr()))
    g2 = dv.DeviceGraph.from_lanes(g.n, g.width, g.edges, g.nvec, dev["vsrc"], dev.get("vw"),
                                   dev["voff"] if "voff" in dev else g.vector_offsets(), scratch)
    if "vw8" in dev:
        g2.vw8 = dev["vw8"]
        g2._struct = None
    assert g2.entries == g.entries and g2.lens_are_degrees == g.lens_are_degrees
    loop2 = dv.DeviceLoop(g2, loop.shift, loop.val_type)
    out_host = torch.empty(g.n, dtype=torch.int32).pin_memory()
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = out_host.numel() * 4
    stream = torch.cuda.current_stream()

    copy_stream = torch.cuda.Stream()

    # pipelined: each chunk's index sort overlaps the copy of the next (chunks
    # of >= 4M lanes; small graphs upload in one piece)
    chunks = int(os.environ.get("WG_E2E_CHUNKS", "0")) or max(1, min(8, (g.nvec * g.width) >> 22))

    def one():
        g2.upload_rebuild(host, dev, chunks=chunks, copy_stream=copy_stream, **rebuild_kw)
        p = loop2.seed(dinit, words, kern, thr, first_hit=first_hit, level_base=level_base,
                       identity_init=identity_init)
        recs, conv, last = loop2.drive(p, max_it)
        out_host.copy_(loop2.values_after(last), non_blocking=True)
        return last

    for _ in range(max(1, args.warmup)):
        one()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        one()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.mean(ts))
    # the last step's decoded layout and result equal the resident run's
    same = bool(torch.equal(g2.vsrc, g.vsrc)) and bool(torch.equal(out_host.cuda(), ref_vals))
    return {"value": round(g.edges / (ms * 1e-3) / 1e9, 4), "unit": "GTEPS (|E|/time-to-solution)",
            "ms_per_step": round(ms, 3), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "result_equal": same, "lane_format": fmt, "lane_bits_per_lane": round(
                8 * sum(host[k].numel() * host[k].element_size() for k in host if k.startswith(("lane_", "vsrc")))
                / max(1, g.nvec * g.width), 2),
            "host_format_build_s": round(t_fmt, 2), "index": "placed from the degrees" if placed else "chunked sort",
            "path": "pinned host topology (lane sources delta-coded per vector [wg_encode_lanes], in-degrees and out-degrees (none for a symmetric input) as a byte per vertex + the large ones[, weights as bytes when <= 255]) -> H2D in up to 8 chunks; wg_widen_degrees, wg_vector_offsets, wg_expand_destinations, per chunk wg_index_place_coded (decode + index slots; or wg_index_chunk_coded + wg_index_finish), wg_index_place_end, wg_widen_weights -> device loop -> D2H values"}


def host_reference_layout(g):
    """Reference-layout int64 arrays (graph.py:109-212) downloaded from the
    device build (input preparation for the CPU arm; parity of this layout
    with the reference's own builder is tested in tests/test_gpu_parity.py)."""
    import oracle
    lane_src, lane_w, lane_count = g.lanes_np()
    topo = oracle.RefTopology(g.n, g.width, g.edges, g.vec_dst_np(), lane_src, lane_w, lane_count)
    idx = oracle.RefIndex(g.n, g.nvec, g.offsets_np(), g.positions_np())
    return topo, idx, g.outdeg_np()


def cpu_baseline(wl, args):
    """The reference CPU path on this host, beside the GPU number: the
    reference arm (`--impl reference`: the stock reference driver and its
    compiled kernels from baseline/_ref, every host core, plus the workers=1
    best-of-3 figure) run in a child process -- so the reference never shares
    a process with the product library -- on a bounded sample of the same
    workload (2 timed runs after 1 warm-up)."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", args.workload,
           "--steps", "2", "--warmup", "1"]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:  # reported, never fatal to the GPU line
        return {"value": None, "unavailable": f"reference arm failed: {e!r}"}
    if "unavailable" in d:
        return {"value": None, "unavailable": d["unavailable"]}
    cb = dict(d["cpu_baseline"])
    cb["ms_per_step"] = d["ms_per_step"]
    if "parity" in d:
        cb["digest"] = d["parity"].get("digest")
    return cb


def pr_traffic(wl):
    """Measured DRAM bytes per pr_pull launch (one `ncu --set full` capture, profiles/traffic.json)."""
    try:
        ent = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(f"{wl['desc']}|pr_pull")
        return ent.get("dram_bytes_per_launch")
    except Exception:
        return None


def run_pagerank(args, wl, el, topo, build_s):
    import torch
    import paper_1903_07754_b200 as wg
    from paper_1903_07754_b200 import _lib, device as dv
    g = topo.device
    n, E = g.n, g.edges
    bufs = (torch.empty(n, dtype=torch.float32, device="cuda"), torch.empty(n, dtype=torch.float32, device="cuda"),
            torch.empty(n, dtype=torch.float32, device="cuda"), torch.zeros(4, dtype=torch.float64, device="cuda"))
    for _ in range(args.warmup):
        dv.pagerank(g, 20, 0.85, bufs=bufs)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ts = []
    launches0 = _lib.launch_count()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with ClockSampler(0) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dv.pagerank(g, 20, 0.85, bufs=bufs)
            b.record(stream)
            clk.tick()
            b.synchronize()
            ts.append(a.elapsed_time(b))
    ms = float(np.mean(ts))
    peak, src = peaks()
    alg = 20 * (4 * E + 20 * n)
    ach = alg / (ms * 1e-3) / 1e9
    out = {"metric": METRIC, "value": round(20 * E / (ms * 1e-3) / 1e9, 4),
           "unit": "GTEPS (20*|E|/time, PageRank)", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": wl["desc"], "V": n, "E": E, "build_s": round(build_s, 2)},
           "gpu_launches": int(_lib.launch_count() - launches0),
           "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                        "frac": round(ach / peak, 4), "traffic": pr_traffic(wl), "peak_source": src,
                        "kernel": "pr_prep_hot + pr_pull + pr_fixup (20 iterations)",
                        "algorithmic_bytes_per_launch": 4 * E + 20 * n,
                        "gather_roofline": gather_roofline(E, ms / 20)},
           "clocks": clk.summary()}
    if not args.no_e2e:
        out["e2e"] = e2e_pagerank(args, g, bufs)
    if not args.no_cpu_baseline:
        out["cpu_baseline"], out["parity"] = cpu_baseline_pagerank(g, bufs[0])
    print(json.dumps(out), flush=True)


def e2e_pagerank(args, g, bufs):
    """PageRank through the C ABI with the layout in pinned host memory: H2D
    of the compact topology (delta-coded lanes, per-destination vector
    offsets, out-degrees; PageRank reads no edge index) in chunks on a copy
    stream, decoded on the device as they land (wg_widen_degrees,
    wg_vector_offsets, wg_expand_destinations, wg_decode_lanes), 20
    iterations, D2H ranks."""
    import torch
    from paper_1903_07754_b200 import device as dv
    ref = dv.pagerank(g, 20, 0.85, bufs=bufs).clone()
    t_fmt = time.perf_counter()
    host = g.host_format(symmetric=False)
    t_fmt = time.perf_counter() - t_fmt
    dev = {k: torch.empty(v.numel() + 64, dtype=v.dtype, device="cuda")[: v.numel()].view(v.shape)
           for k, v in host.items()}
    lanes = g.nvec * g.width
    vsrc = torch.empty(lanes + 64, dtype=torch.int32, device="cuda")
    vdst = torch.empty(g.nvec + 64, dtype=torch.int32, device="cuda")
    outdeg = torch.empty(g.n + 64, dtype=torch.int32, device="cuda")
    g2 = dv.DeviceGraph(g.n, g.width, g.edges, g.nvec, g.entries, vsrc[:lanes], vdst[: g.nvec], None,
                        g.idx_off, g.idx_pos, outdeg[: g.n])
    out_host = torch.empty(g.n, dtype=torch.float32).pin_memory()
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    stream = torch.cuda.current_stream()
    copy_stream = torch.cuda.Stream()
    chunks = int(os.environ.get("WG_E2E_CHUNKS", "0")) or max(1, min(8, lanes >> 22))

    def one():
        g2.upload_rebuild(host, dev, chunks=chunks, copy_stream=copy_stream, index=False)
        r = dv.pagerank(g2, 20, 0.85, bufs=bufs)
        out_host.copy_(r, non_blocking=True)

    for _ in range(max(1, args.warmup)):
        one()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        one()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.mean(ts))
    same = bool(torch.equal(g2.vsrc, g.vsrc[:lanes])) and float((out_host.cuda() - ref).abs().max()) <= 1e-7
    return {"value": round(20 * g.edges / (ms * 1e-3) / 1e9, 4), "unit": "GTEPS (20*|E|/time, PageRank)",
            "ms_per_step": round(ms, 3), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": g.n * 4,
            "result_equal": same, "host_format_build_s": round(t_fmt, 2),
            "path": "pinned host topology (lane sources delta-coded per vector, in/out-degrees as bytes + large ones) -> H2D in "
                    "chunks; wg_expand_destinations, wg_decode_lanes per chunk -> wg_pagerank -> D2H ranks"}


def cpu_baseline_pagerank(g, ranks=None):
    """The float64 C restatement of the PR iteration (no reference PR exists,
    SURVEY 8(a) a17) on all host threads, 20 iterations; with the device ranks
    it also returns the parity (max |r_gpu - r_cpu| per vertex, tolerance 1e-6)."""
    import oracle
    threads = os.cpu_count() or 1
    topo, _, deg = host_reference_layout(g)
    t0 = time.perf_counter()
    ref = oracle.pagerank(topo, deg, 20, 0.85, threads)
    t = time.perf_counter() - t0
    out = {"value": round(20 * g.edges / t / 1e9, 5), "unit": "GTEPS (20*|E|/time, PageRank)", "cores": threads,
           "kind": "port", "seconds_per_run": round(t, 3), "sample": "1 full run of 20 iterations (float64)"}
    parity = None
    if ranks is not None:
        err = float(np.max(np.abs(ranks.cpu().numpy().astype(np.float64) - ref)))
        parity = {"max_abs_error": err, "tolerance": 1e-6, "ok": err <= 1e-6, "oracle": "float64 C port"}
    return out, parity


def import_reference():
    """The UNMODIFIED reference package installed in baseline/_ref
    (baseline/install_ref.sh), never the product package."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "wedgegraph" / "__init__.py").exists():
        return None, "baseline/_ref not installed (baseline/install_ref.sh)"
    sys.path.insert(0, str(ref_dir))
    import wedgegraph
    import wedgegraph.kernels as rk
    if not str(Path(wedgegraph.__file__).resolve()).startswith(str(ref_dir.resolve())):
        return None, f"wedgegraph resolved outside baseline/_ref: {wedgegraph.__file__}"
    if "native" not in rk.available_backends():
        return None, "reference native (Cython) backend not built in baseline/_ref"
    return wedgegraph, None


def prepare_reference_input(wl):
    """Seeded input of the workload in the reference layout (int64 host
    arrays), prepared with the oracle's restated generators / builders (the
    reference's own take minutes at s22; equality with them is pinned by
    tests/test_oracle.py).  Returns (n, E, topology_arrays, index_arrays, degrees)."""
    import oracle
    if "grid" in wl:
        n, s, d, w = oracle.grid_edges(wl["grid"][0], wl["grid"][1], GRID_SEED)
    else:
        n, s, d = oracle.rmat_edges_fast(wl["scale"], wl["ef"], 1)
        s, d = oracle.prepare_unweighted(n, s, d, wl["sym"])
        w = oracle.synthesize_weights(s, d, wl["weights"]) if wl.get("weights") else None
    tp = oracle.build_pull_topology(n, s, d, w, 4)
    idx = oracle.build_edge_index(tp)
    deg = oracle.compute_out_degrees(n, s)
    return n, len(s), tp, idx, deg, (s, d)


def run_reference(args, wl):
    """--impl reference: the reference's own CPU implementation of the path --
    the stock driver wedgegraph.run_until_convergence (engine.py:330-388) over
    its compiled native backend (kernels.py:72-125, _kernels.pyx) from
    baseline/_ref, workers = every host core -- on the same workload, config,
    metric and unit as the b200 arm.  Never imports the product package.
    Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if wl["app"] == "pr":
        return run_reference_pagerank(args, wl, threads)
    ref, why = import_reference()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return
    t0 = time.perf_counter()
    n, E, tp, idx, deg, _ = prepare_reference_input(wl)
    prep_s = time.perf_counter() - t0
    topo = ref.PullTopology(n, 4, E, tp.vec_dst, tp.lane_src, tp.lane_weight, tp.lane_count)
    index = ref.EdgeIndex(n, tp.vector_count, idx.offsets, idx.positions)
    app = wl["app"]
    prog = ref.make_program(app, None if app == "cc" else 0)
    # a bounded sample per step: runs longer than the cap (grid SSSP, ~8.6K
    # iterations at ~0.1 s each) time their first `cap` iterations, scaled
    cap = int(wl.get("ref_iteration_cap", n + 16))
    full_iters = wl.get("iterations")

    def cfg(workers):
        return ref.EngineConfig(threshold=ref.FullnessThreshold.of(wl["thr"]),
                                precision=ref.FrontierPrecision(wl["vpg"]), workers=workers,
                                max_iterations=cap)

    def timed(workers, k):
        ts, res = [], None
        for _ in range(k):
            a = time.perf_counter()
            res = ref.run_until_convergence(topo, index, prog, deg, cfg(workers), backend="native")
            ts.append(time.perf_counter() - a)
        return ts, res

    # warm-up + the timed steps on every host core (the reference's CLI
    # reads WEDGE_WORKERS, cli.py:149-153)
    for _ in range(args.warmup):
        timed(threads, 1)
    ts, res = timed(threads, args.steps)
    iters = len(res.stats)
    scale = (full_iters / iters) if (full_iters and iters < full_iters) else 1.0
    ms = float(np.mean(ts)) * 1e3 * scale
    best_ms = float(np.min(ts)) * 1e3 * scale
    # BASELINE.md protocol: also one worker, warm best-of-3
    one = None
    if not args.no_single_worker:
        t1, _ = timed(1, 3)
        one = {"workers": 1, "best_of_3_ms": round(min(t1) * 1e3 * scale, 3),
               "value": round(E / (min(t1) * scale) / 1e9, 6)}
    val = E / (ms * 1e-3) / 1e9
    digest = ref.result_digest(res.values)
    sample = (f"each step = 1 full run of the stock reference driver to convergence ({iters} iterations, "
              f"workers={threads})") if scale == 1.0 else (
              f"each step = the first {iters} of {full_iters} iterations of the stock reference driver "
              f"(workers={threads}), scaled by the iteration count")
    out = {
        "impl": "reference", "metric": METRIC, "value": round(val, 6),
        "unit": "GTEPS (|E|/time-to-solution)", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": DATA_DESC,
        "config": workload_config(wl, n, E),
        "parity": {"digest": digest, "expected": wl.get("expect_digest"),
                   "ok": digest == wl.get("expect_digest") if scale == 1.0 else None,
                   "trace": rle_modes(res.stats), "iterations": iters},
        "cpu_baseline": {"value": round(val, 6), "unit": "GTEPS (|E|/time-to-solution)", "cores": threads,
                         "kind": "reference", "sample": sample, "best_ms": round(best_ms, 3),
                         "single_worker": one, "host": host_cpu()},
        "e2e": {"value": round(val, 6), "unit": "GTEPS (|E|/time-to-solution)", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference": {"package": "wedgegraph " + getattr(ref, "__version__", "?"),
                      "path": str(Path(ref.__file__).resolve().parent.relative_to(ROOT)),
                      "driver": "wedgegraph.run_until_convergence (engine.py:330-388)",
                      "backend": "native (compiled _kernels.pyx)", "input_prep_s": round(prep_s, 1),
                      "input_prep": "oracle restated generators/builders (untimed)"},
        "loaded_so": loaded_native_libs(),
    }
    print(json.dumps(out), flush=True)


def run_reference_pagerank(args, wl, threads):
    """PageRank has no reference implementation (the reference
    rejects it, test_apps.py:167-169): the arm times the float64 C port of the
    a17 semantics on every host core (kind "port")."""
    import oracle
    n, E, tp, _, deg, _ = prepare_reference_input(wl)
    ts = []
    for i in range(args.warmup + args.steps):
        a = time.perf_counter()
        oracle.pagerank(tp, deg, 20, 0.85, threads)
        if i >= args.warmup:
            ts.append(time.perf_counter() - a)
    t = float(np.mean(ts))
    val = 20 * E / t / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": "GTEPS (20*|E|/time, PageRank)",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": DATA_DESC, "config": workload_config(wl, n, E),
        "cpu_baseline": {"value": round(val, 6), "unit": "GTEPS (20*|E|/time, PageRank)", "cores": threads,
                         "kind": "port", "sample": "each step = 20 iterations (no reference PR exists)",
                         "host": host_cpu()},
        "e2e": {"value": round(val, 6), "unit": "GTEPS (20*|E|/time, PageRank)", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def loaded_native_libs():
    """Shared objects under the repo mapped into this process."""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except Exception:
        return None
    root = str(ROOT.resolve())
    return sorted({ln.split()[-1][len(root) + 1:] for ln in maps
                   if ln.split()[-1].startswith(root) and ".so" in ln.split()[-1]})


def host_cpu() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return f"{line.split(':', 1)[1].strip()} x{os.cpu_count()}"
    except Exception:
        pass
    return f"x{os.cpu_count()}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--workload", default="cc22", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-compact", action="store_true",
                    help="also time the compact delta-coded upload format (encode time reported, untimed)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the multi-GPU sharded path even at N=1")
    ap.add_argument("--no-single-worker", action="store_true",
                    help="reference arm: skip the workers=1 best-of-3 figure")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_b200(args, wl)


if __name__ == "__main__":
    main()
