"""B200-native Wedge-Frontier pull engine with the `wedgegraph` API.

A drop-in for the reference package's hot path (wedgegraph 0.1.0): graph
construction, vertex / Wedge frontiers, the pull iterations and the
convergence driver for BFS / CC / SSSP, plus a PageRank entry point.  Compute
runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/wedge_b200.h (libwedge_b200.so, loaded with ctypes); PyTorch only
provides device memory and streams.

The reference's push engine is out of scope; the CLI is
mirrored as ``python -m paper_1903_07754_b200``.  ``B200Backend`` also plugs
into the reference's own engine via its ``backend=`` seam.
"""

from .apps import bfs_program, cc_program, make_program, pagerank, sssp_program
from .backend import B200Backend, available_backends, get_backend
from .engine import (MODE_FULL, MODE_WEDGE, UNREACHED, ApplicationProgram, EngineConfig,
                     IterationStats, MinPlusKernel, RunResult, ValueBuffers, result_digest,
                     run_iteration_full, run_iteration_wedge, run_until_convergence, stats_signature)
from .frontier import (Bitmask, FrontierPrecision, FullnessThreshold, VertexFrontier, WedgeFrontier,
                       should_transform, transform_frontier, wedge_covered_vectors)
from .generators import (GenSpec, ParseError, drop_self_loops_dedup, generate, grid_graph, load_edge_list,
                         parse_edge_list, save_edge_list_binary, serialize_edge_list, symmetrize,
                         synthesize_weights)
from .graph import (EdgeIndex, EdgeList, PullTopology, build_edge_index, build_pull_topology,
                    compute_out_degrees)

__version__ = "0.1.0"

__all__ = [
    "ApplicationProgram", "B200Backend", "Bitmask", "EdgeIndex", "EdgeList", "EngineConfig",
    "FrontierPrecision", "FullnessThreshold", "GenSpec", "IterationStats", "MODE_FULL",
    "MODE_WEDGE", "MinPlusKernel", "PullTopology", "RunResult", "UNREACHED", "ValueBuffers",
    "VertexFrontier", "WedgeFrontier", "available_backends", "bfs_program", "build_edge_index",
    "build_pull_topology", "cc_program", "compute_out_degrees", "drop_self_loops_dedup", "generate",
    "get_backend", "grid_graph", "load_edge_list", "make_program", "parse_edge_list", "ParseError",
    "save_edge_list_binary", "serialize_edge_list", "pagerank", "result_digest", "run_iteration_full",
    "run_iteration_wedge", "run_until_convergence", "should_transform", "sssp_program",
    "stats_signature", "symmetrize", "synthesize_weights", "transform_frontier",
    "wedge_covered_vectors",
]
