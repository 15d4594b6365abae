"""ctypes binding of the C ABI declared in include/wedge_b200.h.

The shared library ``libwedge_b200.so`` is built in-tree by
``paper_1903_07754_b200._build.build()`` (nvcc, sm_100a).  There is no CPU
fallback: if the library is missing or no CUDA device is visible, every entry
point raises, loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libwedge_b200.so"

WG_OK = 0
WG_EINVAL, WG_ECUDA, WG_ENOSPACE, WG_EOVERFLOW = -1, -2, -3, -4
WG_VAL_U32, WG_VAL_I64 = 0, 1
NO_LANE = 0xFFFFFFFF

c_u32, c_u64, c_i32, c_i64, c_vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p


class WgGraph(ctypes.Structure):
    _fields_ = [("n", c_u32), ("width", c_u32), ("nvec", c_u64), ("edges", c_u64),
                ("entries", c_u64), ("vsrc", c_vp), ("vdst", c_vp), ("vw", c_vp),
                ("idx_off", c_vp), ("idx_pos", c_vp), ("outdeg", c_vp), ("flags", c_u32), ("vw8", c_vp),
                ("voff", c_vp), ("vfirst", c_vp)]


WG_GRAPH_LENS_ARE_DEGREES = 1


class WgMinPlus(ctypes.Structure):
    _fields_ = [("filter_unvisited", c_i32), ("use_weight", c_i32), ("apply_increment", c_i64),
                ("sentinel", c_i64)]


REC_FIELDS = ["mode", "active_edges", "vectors_touched", "frontier_out", "out_edge_sum",
              "nz_packed", "z_count", "covered_vectors", "transform_entries", "groups", "overflow",
              "reserved0", "reserved1", "reserved2", "reserved3", "reserved4", "lanes_read", "gathers"]
REC_U64 = 32  # record size in uint64 words


class WgRunBufs(ctypes.Structure):
    _fields_ = [("vals", c_vp * 2), ("fbits", c_vp * 2), ("fvert", c_vp * 2), ("fpref", c_vp * 2),
                ("tstart", c_vp * 2), ("gbits", c_vp), ("glist", c_vp), ("bcount", c_vp), ("recs", c_vp),
                ("ctrl", c_vp), ("ring", c_u32), ("gbits_alt", c_vp),
                ("glist_alt", c_vp), ("work", c_vp)]


class WgRunParams(ctypes.Structure):
    _fields_ = [("val_type", c_i32), ("shift", c_i32), ("kern", WgMinPlus), ("wedge_limit", c_u64),
                ("timer", c_vp), ("flags", c_i32), ("level_base", c_i64)]


WG_RUN_FIRST_HIT = 1
WG_RUN_KEEP_LISTS = 2
WG_RUN_IDENTITY_INIT = 8
WG_RUN_FLOOR_SKIP = 16
WG_RUN_LOCAL_GATE = 32
WG_CODED_BLOCK_VECTORS = 1024
WG_INGEST_BAD_DST, WG_INGEST_BAD_SRC, WG_INGEST_BAD_COUNT, WG_INGEST_BAD_WEIGHT = 1, 2, 4, 8
WG_INGEST_BAD_POS, WG_INGEST_BAD_DEGREE, WG_INGEST_BAD_OFFSETS, WG_INGEST_LENS_DIFFER = 16, 32, 64, 128
WG_VALUES_NOT_U32, WG_VALUES_NOT_IDENTITY = 1, 2


EXPORTS = [
    "wg_last_error", "wg_abi_version", "wg_device_sm_count", "wg_vector_capacity",
    "wg_layout_scratch_bytes", "wg_build_layout", "wg_kernel_workspace_bytes", "wg_transform",
    "wg_pull_full", "wg_pull_wedge", "wg_covered_groups", "wg_run_buffer_sizes", "wg_run_init",
    "wg_run_enqueue", "wg_run_enqueue_counter", "wg_pagerank", "wg_rmat_edges",
    "wg_canonical_scratch_bytes", "wg_canonical_edges", "wg_weights_hash", "wg_grid_edges",
    "wg_timer_create", "wg_timer_destroy", "wg_timer_reset", "wg_timer_read", "wg_launch_count",
    "wg_exchange_pack", "wg_exchange_apply", "wg_run_graph_create", "wg_run_graph_launch",
    "wg_run_graph_destroy", "wg_run_loop_graph_create", "wg_run_loop_launch", "wg_run_persistent",
    "wg_debug_phase_buffer", "wg_index_scratch_bytes", "wg_build_index", "wg_expand_destinations",
    "wg_narrow_weights", "wg_widen_weights", "wg_exchange_bytes", "wg_exchange_pack_all",
    "wg_exchange_apply_all", "wg_index_chunked_scratch_bytes", "wg_index_chunk", "wg_index_finish",
    "wg_pagerank_prep", "wg_pagerank_pull", "wg_lane_bits", "wg_packed_lane_words", "wg_pack_lanes",
    "wg_unpack_lanes", "wg_coded_blocks", "wg_coded_max_words", "wg_coded_width_words", "wg_widen_degrees",
    "wg_vector_offsets_scratch_bytes", "wg_vector_offsets", "wg_coded_scratch_bytes", "wg_encode_lanes",
    "wg_decode_lanes", "wg_index_chunk_coded", "wg_expand_scratch_bytes", "wg_index_placed_scratch_bytes",
    "wg_index_place_begin", "wg_index_place_chunk", "wg_index_place_coded", "wg_index_place_end",
    "wg_ingest_vectors", "wg_ingest_u32", "wg_ingest_offsets", "wg_values_scan", "wg_vector_offsets_from_dst",
    "wg_run_seed", "wg_debug_kernel_timeline", "wg_debug_kernel_ids", "wg_first_lanes",
    "wg_pagerank_ws_bytes", "wg_pagerank_prep_ws_bytes", "wg_exchange_slice_pack", "wg_exchange_apply_slices",
    "wg_run_loop_graph_create_seeded", "wg_run_loop_launch_seeded",
    "wg_pagerank_hot_ws_bytes", "wg_pagerank_hot_layout", "wg_pagerank_hot",
]

_LIB = None


class WedgeError(RuntimeError):
    """A C-ABI call failed (the message comes from wg_last_error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"wedge_b200 error {code}: {msg}")
        self.code = code


class OverflowError32(WedgeError):
    pass


def load(path: os.PathLike | str | None = None):
    """Load libwedge_b200.so (no compute call is made)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else Path(os.environ.get("WG_LIB", LIB_PATH))  # WG_LIB: an experiment build
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 engine has no CPU fallback)")
    L = ctypes.CDLL(str(p))
    G = ctypes.POINTER(WgGraph)
    K = ctypes.POINTER(WgMinPlus)
    B = ctypes.POINTER(WgRunBufs)
    P = ctypes.POINTER(WgRunParams)
    u64p = ctypes.POINTER(c_u64)
    sig = {
        "wg_last_error": (ctypes.c_char_p, []),
        "wg_abi_version": (ctypes.c_int, []),
        "wg_device_sm_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
        "wg_vector_capacity": (c_u64, [c_u64, c_u32, c_u32]),
        "wg_layout_scratch_bytes": (ctypes.c_size_t, [c_u64, c_u32]),
        "wg_build_layout": (ctypes.c_int, [c_u32, c_u64, c_vp, c_vp, c_vp, c_u32, c_u64, c_vp, c_vp,
                                           c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, u64p, c_vp]),
        "wg_kernel_workspace_bytes": (ctypes.c_size_t, [G, ctypes.c_int]),
        "wg_transform": (ctypes.c_int, [G, c_vp, ctypes.c_int, c_vp, c_vp, ctypes.c_size_t, u64p, c_vp]),
        "wg_pull_full": (ctypes.c_int, [G, ctypes.c_int, c_vp, c_vp, c_vp, K, c_vp, ctypes.c_size_t,
                                        u64p, c_vp]),
        "wg_pull_wedge": (ctypes.c_int, [G, c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp, K, c_vp,
                                         ctypes.c_size_t, u64p, c_vp]),
        "wg_covered_groups": (ctypes.c_int, [c_vp, c_u64, c_vp, c_vp, ctypes.c_size_t, u64p, c_vp]),
        "wg_run_buffer_sizes": (ctypes.c_int, [G, ctypes.c_int, u64p]),
        "wg_run_init": (ctypes.c_int, [G, B, P, c_vp, c_vp]),
        "wg_run_enqueue": (ctypes.c_int, [G, B, P, c_u64, c_u32, c_vp]),
        "wg_run_enqueue_counter": (ctypes.c_int, [G, B, P, c_u32, c_vp]),
        "wg_pagerank_ws_bytes": (ctypes.c_size_t, [G]),
        "wg_exchange_slice_pack": (ctypes.c_int, [G, B, P, c_u64, c_u32, c_u32, c_vp, c_vp]),
        "wg_exchange_apply_slices": (ctypes.c_int, [G, B, P, c_u64, c_vp, c_vp, c_u32, c_u32, c_u64, c_vp]),
        "wg_pagerank": (ctypes.c_int, [G, ctypes.c_int, ctypes.c_double, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       ctypes.c_size_t, c_vp]),
        "wg_pagerank_hot_ws_bytes": (ctypes.c_size_t, [G]),
        "wg_pagerank_hot_layout": (ctypes.c_int, [G, c_vp, c_vp, c_vp, u64p, c_vp, ctypes.c_size_t, c_vp]),
        "wg_pagerank_hot": (ctypes.c_int, [G, c_vp, c_vp, c_vp, c_u64, ctypes.c_int, ctypes.c_double, c_vp, c_vp,
                                           c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp]),
        "wg_pagerank_prep_ws_bytes": (ctypes.c_size_t, [c_u32]),
        "wg_pagerank_prep": (ctypes.c_int, [c_u32, ctypes.c_int, ctypes.c_double, c_vp, c_vp, c_vp, c_vp,
                                            c_vp, c_vp, ctypes.c_size_t, c_vp]),
        "wg_pagerank_pull": (ctypes.c_int, [G, c_vp, c_vp, c_u32, c_vp, ctypes.c_size_t, c_vp]),
        "wg_lane_bits": (c_u32, [c_u32]),
        "wg_packed_lane_words": (c_u64, [c_u64, c_u32]),
        "wg_pack_lanes": (ctypes.c_int, [c_u64, c_vp, c_u32, c_vp, c_vp]),
        "wg_unpack_lanes": (ctypes.c_int, [c_vp, c_u32, c_u64, c_u64, c_vp, c_vp]),
        "wg_coded_blocks": (c_u64, [c_u64]),
        "wg_coded_max_words": (c_u64, [c_u64, c_u32]),
        "wg_coded_width_words": (c_u64, [c_u64]),
        "wg_widen_degrees": (ctypes.c_int, [c_u32, c_vp, c_vp, c_u64, c_vp, c_vp]),
        "wg_vector_offsets_scratch_bytes": (ctypes.c_size_t, [c_u32]),
        "wg_vector_offsets": (ctypes.c_int, [c_u32, c_vp, c_u32, c_vp, c_vp, ctypes.c_size_t, c_vp]),
        "wg_coded_scratch_bytes": (ctypes.c_size_t, [c_u64]),
        "wg_encode_lanes": (ctypes.c_int, [G, c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, u64p, c_vp]),
        "wg_decode_lanes": (ctypes.c_int, [c_u64, c_u32, c_vp, c_vp, c_vp, c_vp, c_u64, c_u64, c_vp, c_vp]),
        "wg_index_chunk_coded": (ctypes.c_int, [G, c_vp, c_vp, c_vp, c_u64, c_u64, c_u32, c_u64, c_vp,
                                                ctypes.c_size_t, c_vp]),
        "wg_rmat_edges": (ctypes.c_int, [c_u32, c_u64, c_u64, c_u64, c_u64, c_u64,
                                         ctypes.POINTER(ctypes.c_double), c_vp, c_vp, c_vp]),
        "wg_canonical_scratch_bytes": (ctypes.c_size_t, [c_u64]),
        "wg_canonical_edges": (ctypes.c_int, [c_u64, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_vp,
                                              ctypes.c_size_t, u64p, c_vp]),
        "wg_weights_hash": (ctypes.c_int, [c_u64, c_vp, c_vp, c_u32, c_vp, c_vp]),
        "wg_grid_edges": (ctypes.c_int, [c_u32, c_u32, c_u64, c_u32, c_u32, c_vp, c_vp, c_vp, c_vp,
                                         u64p, c_vp]),
        "wg_timer_create": (c_vp, [ctypes.c_int]),
        "wg_timer_destroy": (None, [c_vp]),
        "wg_timer_reset": (ctypes.c_int, [c_vp]),
        "wg_timer_read": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(c_i32),
                                         ctypes.POINTER(c_i64), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
        "wg_launch_count": (c_u64, []),
        "wg_exchange_pack": (ctypes.c_int, [G, B, P, c_u64, c_vp, c_vp, c_u64, u64p, c_vp]),
        "wg_exchange_apply": (ctypes.c_int, [G, B, P, c_u64, c_vp, c_vp, c_u64, c_vp]),
        "wg_run_graph_create": (c_vp, [G, B, P, c_u32, c_vp]),
        "wg_run_graph_launch": (ctypes.c_int, [c_vp, c_vp]),
        "wg_run_graph_destroy": (None, [c_vp]),
        "wg_run_loop_graph_create": (c_vp, [G, B, P, c_vp]),
        "wg_run_loop_launch": (ctypes.c_int, [c_vp, B, c_u64, c_vp]),
        "wg_run_loop_graph_create_seeded": (c_vp, [G, B, P, c_vp, c_vp, u64p, c_vp]),
        "wg_run_loop_launch_seeded": (ctypes.c_int, [c_vp, B, c_u64, c_vp, c_vp, ctypes.c_size_t, c_vp, c_vp,
                                                     ctypes.c_size_t, c_vp]),
        "wg_run_persistent": (ctypes.c_int, [G, B, P, c_u64, c_vp]),
        "wg_debug_phase_buffer": (ctypes.c_int, [c_vp, c_u64]),
        "wg_index_scratch_bytes": (ctypes.c_size_t, [c_u64, c_u32]),
        "wg_build_index": (ctypes.c_int, [G, c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, u64p, c_vp]),
        "wg_expand_destinations": (ctypes.c_int, [c_u32, c_vp, c_u64, c_vp, c_vp, ctypes.c_size_t, c_vp]),
        "wg_expand_scratch_bytes": (ctypes.c_size_t, [c_u64]),
        "wg_index_placed_scratch_bytes": (ctypes.c_size_t, [c_u32]),
        "wg_index_place_begin": (ctypes.c_int, [G, c_vp, c_vp, ctypes.c_size_t, c_vp]),
        "wg_index_place_chunk": (ctypes.c_int, [G, c_u64, c_u64, c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp]),
        "wg_index_place_coded": (ctypes.c_int, [G, c_vp, c_vp, c_vp, c_u64, c_u64, c_vp, c_vp, c_vp,
                                                ctypes.c_size_t, c_vp]),
        "wg_index_place_end": (ctypes.c_int, [G, c_vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_int), c_vp]),
        "wg_narrow_weights": (ctypes.c_int, [G, c_vp, ctypes.POINTER(ctypes.c_int), c_vp]),
        "wg_widen_weights": (ctypes.c_int, [c_u64, c_vp, c_vp, c_vp]),
        "wg_exchange_bytes": (c_u64, [c_u64, ctypes.c_int]),
        "wg_index_chunked_scratch_bytes": (ctypes.c_size_t, [c_u64, c_u64, c_u32]),
        "wg_index_chunk": (ctypes.c_int, [G, c_u64, c_u64, c_u32, c_u64, c_vp, ctypes.c_size_t, c_vp]),
        "wg_index_finish": (ctypes.c_int, [G, c_u64, c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, u64p, c_vp]),
        "wg_exchange_pack_all": (ctypes.c_int, [G, B, P, c_u64, c_vp, c_u64, c_vp]),
        "wg_exchange_apply_all": (ctypes.c_int, [G, B, P, c_u64, c_vp, c_u32, c_u64, c_vp, c_vp]),
        "wg_ingest_vectors": (ctypes.c_int, [c_u64, c_u32, c_u32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                             c_vp, c_vp]),
        "wg_ingest_u32": (ctypes.c_int, [c_u64, c_vp, c_i64, c_vp, c_u32, c_vp, c_vp]),
        "wg_ingest_offsets": (ctypes.c_int, [c_u32, c_vp, c_u64, c_vp, c_vp, c_vp]),
        "wg_values_scan": (ctypes.c_int, [c_u32, c_vp, c_i64, c_vp, c_vp, c_vp]),
        "wg_vector_offsets_from_dst": (ctypes.c_int, [G, c_vp, c_vp]),
        "wg_run_seed": (ctypes.c_int, [G, B, P, c_vp, c_vp, u64p, c_vp]),
        "wg_debug_kernel_timeline": (ctypes.c_int, [c_vp, c_u64]),
        "wg_debug_kernel_ids": (c_u32, []),
        "wg_first_lanes": (ctypes.c_int, [G, c_vp, c_vp, c_vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = L
    return L


def check(rc: int) -> None:
    if rc != WG_OK:
        msg = load().wg_last_error().decode(errors="replace")
        if rc == WG_EOVERFLOW:
            raise OverflowError32(rc, msg)
        raise WedgeError(rc, msg)


class EventTimer:
    """CUDA-event pairs recorded by the library around each launch group of
    the device loop (kind 1 Wedge prep, 2 pull, 3 end-of-iteration)."""

    def __init__(self, capacity: int = 4096):
        L = load()
        self.capacity = capacity
        self.handle = L.wg_timer_create(capacity)
        if not self.handle:
            raise WedgeError(WG_ECUDA, L.wg_last_error().decode())

    def reset(self):
        check(load().wg_timer_reset(self.handle))

    def read(self):
        n = ctypes.c_int(0)
        ms = (ctypes.c_float * self.capacity)()
        kind = (c_i32 * self.capacity)()
        it = (c_i64 * self.capacity)()
        check(load().wg_timer_read(self.handle, ms, kind, it, self.capacity, ctypes.byref(n)))
        return [(int(kind[i]), int(it[i]), float(ms[i])) for i in range(n.value)]

    def __del__(self):
        try:
            if self.handle:
                load().wg_timer_destroy(self.handle)
        except Exception:
            pass


def launch_count() -> int:
    return int(load().wg_launch_count())


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1903_07754_b200 needs a CUDA device (B200, sm_100a); none is visible")
    load()
    return torch


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
