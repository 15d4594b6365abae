"""Dump the CC s22 pull layout lanes (vsrc) to <base>.vsrc for the microbenchmarks."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench

el, topo = bench.make_graph(bench.WORKLOADS[sys.argv[2] if len(sys.argv) > 2 else "cc22"])
g = topo.device
g.vsrc[: g.nvec * g.width].cpu().numpy().tofile(sys.argv[1] + ".vsrc")
