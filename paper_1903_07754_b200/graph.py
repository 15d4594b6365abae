"""Graph structures of the drop-in API, backed by the device layout.

Mirrors the reference's graph core (graph.py:1-301): ``EdgeList``,
``PullTopology``, ``EdgeIndex``, ``build_pull_topology``,
``build_edge_index``, ``compute_out_degrees``.  Construction runs on the GPU
(``wg_build_layout``); the reference-layout int64 arrays (``vec_dst``,
``lane_src``, ``lane_weight``, ``lane_count``, ``offsets``, ``positions``) are
materialised on the host lazily, only when a caller asks for them, so a
PullTopology built here can also be handed to code written against the
reference (it has the same attributes).
"""

from __future__ import annotations

from typing import Iterator, Optional

import numpy as np

from .device import DeviceGraph, to_dev_u32


def _ids(values, n: int, what: str) -> np.ndarray:
    a = np.ascontiguousarray(values, dtype=np.int64)
    if a.size and (a.min() < 0 or a.max() >= n):
        raise ValueError(f"{what} id out of range [0, {n})")
    return a


class EdgeList:
    """Directed edges over ids [0, vertex_count); optional positive weights
    (same contract as graph.py:36-106).  Arrays may be host (numpy) or device
    (torch int32 holding uint32 ids, as produced by the device generators);
    the other side is materialised on demand."""

    def __init__(self, vertex_count: int, src, dst, weight=None, *, _device=None):
        if vertex_count < 0:
            raise ValueError("vertex_count must be non-negative")
        self.vertex_count = int(vertex_count)
        self._dev = _device  # (src, dst, weight|None) device tensors
        if _device is not None:
            self._src = self._dst = self._w = None
            self._m = int(_device[0].numel())
            self._weighted = _device[2] is not None
            return
        s = _ids(src, self.vertex_count, "source")
        d = _ids(dst, self.vertex_count, "destination")
        if s.shape != d.shape:
            raise ValueError("src/dst arrays differ in length")
        w = None
        if weight is not None:
            w = np.ascontiguousarray(weight, dtype=np.int64)
            if w.shape != s.shape:
                raise ValueError("weight array length mismatch")
            if w.size and w.min() < 1:
                raise ValueError("edge weights must be positive")
        self._src, self._dst, self._w = s, d, w
        self._m = int(s.shape[0])
        self._weighted = w is not None

    @classmethod
    def from_device(cls, vertex_count: int, src, dst, weight=None) -> "EdgeList":
        return cls(vertex_count, None, None, _device=(src, dst, weight))

    @classmethod
    def from_pairs(cls, pairs, vertex_count: Optional[int] = None) -> "EdgeList":
        pairs = list(pairs)
        cols = list(zip(*pairs)) if pairs else [(), ()]
        src, dst = cols[0], cols[1]
        wgt = cols[2] if pairs and len(pairs[0]) == 3 else None
        if vertex_count is None:
            vertex_count = int(max(max(src, default=-1), max(dst, default=-1)) + 1)
        return cls(vertex_count, src, dst, wgt)

    # host views
    def _host(self):
        if self._src is None:
            s, d, w = self._dev
            self._src = s.cpu().numpy().view(np.uint32).astype(np.int64)
            self._dst = d.cpu().numpy().view(np.uint32).astype(np.int64)
            self._w = None if w is None else w.cpu().numpy().view(np.uint32).astype(np.int64)

    @property
    def src(self) -> np.ndarray:
        self._host()
        return self._src

    @property
    def dst(self) -> np.ndarray:
        self._host()
        return self._dst

    @property
    def weight(self) -> Optional[np.ndarray]:
        self._host()
        return self._w

    def device_arrays(self):
        """(src, dst, weight|None) as device int32 tensors (uint32 bits)."""
        if self._dev is None:
            w = to_dev_u32(self._w) if self._w is not None else None
            self._dev = (to_dev_u32(self._src), to_dev_u32(self._dst), w)
        return self._dev

    @property
    def edge_count(self) -> int:
        return self._m

    def is_weighted(self) -> bool:
        return self._weighted

    def edges(self) -> Iterator[tuple]:
        cols = [self.src.tolist(), self.dst.tolist()]
        if self.weight is not None:
            cols.append(self.weight.tolist())
        return iter(zip(*cols))

    def __len__(self) -> int:
        return self._m

    def __eq__(self, other) -> bool:
        if not isinstance(other, EdgeList):
            return NotImplemented
        if self.vertex_count != other.vertex_count or self._weighted != other._weighted:
            return False
        ok = np.array_equal(self.src, other.src) and np.array_equal(self.dst, other.dst)
        return bool(ok and (not self._weighted or np.array_equal(self.weight, other.weight)))

    def __repr__(self) -> str:
        return f"EdgeList(|V|={self.vertex_count}, |E|={self._m}, {'weighted' if self._weighted else 'unweighted'})"


class PullTopology:
    """Destination-grouped W-lane vectors (graph.py:109-164).

    Two forms: ``PullTopology(device_graph)`` -- resident on the device (what
    build_pull_topology returns; reference-layout host arrays are then lazy
    downloads) -- or the reference's own constructor
    ``PullTopology(vertex_count, vector_width, edge_count, vec_dst, lane_src,
    lane_weight, lane_count)`` over host int64 arrays, which the backend
    uploads (and narrows on the device) when a run needs them."""

    def __init__(self, *args):
        self._lanes = None
        self._vec_dst = None
        self._valid = None
        if len(args) == 1 and isinstance(args[0], DeviceGraph):
            self.device = args[0]
            self._host = None
            return
        if len(args) != 7:
            raise TypeError("PullTopology(device_graph) or PullTopology(vertex_count, vector_width, "
                            "edge_count, vec_dst, lane_src, lane_weight, lane_count)")
        n, w, m, vec_dst, lane_src, lane_weight, lane_count = args
        self.device = None
        self._host = (int(n), int(w), int(m))
        self._vec_dst = vec_dst
        self._lanes = (lane_src, lane_weight, lane_count)

    vertex_count = property(lambda self: self._host[0] if self._host else self.device.n)
    vector_width = property(lambda self: self._host[1] if self._host else self.device.width)
    edge_count = property(lambda self: self._host[2] if self._host else self.device.edges)
    vector_count = property(lambda self: int(self._vec_dst.shape[0]) if self._host else self.device.nvec)

    def is_weighted(self) -> bool:
        return self._lanes[1] is not None if self._host else self.device.weighted()

    @property
    def vec_dst(self) -> np.ndarray:
        if self._vec_dst is None:
            self._vec_dst = self.device.vec_dst_np()
        return self._vec_dst

    def _lane_arrays(self):
        if self._lanes is None:
            self._lanes = self.device.lanes_np()
        return self._lanes

    lane_src = property(lambda self: self._lane_arrays()[0])
    lane_weight = property(lambda self: self._lane_arrays()[1])
    lane_count = property(lambda self: self._lane_arrays()[2])

    def lane_valid(self) -> np.ndarray:
        if self._valid is None:
            self._valid = self.lane_count[:, None] > np.arange(self.vector_width)[None, :]
        return self._valid

    def lanes(self) -> Iterator[tuple]:
        ls, lw, lc = self._lane_arrays()
        vd = self.vec_dst
        for p in range(self.vector_count):
            for k in range(int(lc[p])):
                yield p, int(ls[p, k]), int(vd[p]), (int(lw[p, k]) if lw is not None else None)

    def __repr__(self) -> str:
        return (f"PullTopology(|V|={self.vertex_count}, |E|={self.edge_count}, "
                f"vectors={self.vector_count}, W={self.vector_width}, {'host' if self._host else 'device'})")


class EdgeIndex:
    """Per-source ascending, de-duplicated vector positions (graph.py:190-212).

    ``EdgeIndex(device_graph)`` shares the topology's device graph;
    ``EdgeIndex(vertex_count, vector_count, offsets, positions)`` is the
    reference's constructor over host int64 arrays."""

    def __init__(self, *args):
        self._off = None
        self._pos = None
        if len(args) == 1 and isinstance(args[0], DeviceGraph):
            self.device = args[0]
            self._host = None
            return
        if len(args) != 4:
            raise TypeError("EdgeIndex(device_graph) or EdgeIndex(vertex_count, vector_count, offsets, positions)")
        self.device = None
        self._host = (int(args[0]), int(args[1]))
        self._off, self._pos = args[2], args[3]

    vertex_count = property(lambda self: self._host[0] if self._host else self.device.n)
    vector_count = property(lambda self: self._host[1] if self._host else self.device.nvec)

    @property
    def offsets(self) -> np.ndarray:
        if self._off is None:
            self._off = self.device.offsets_np()
        return self._off

    @property
    def positions(self) -> np.ndarray:
        if self._pos is None:
            self._pos = self.device.positions_np()
        return self._pos

    def positions_for(self, v: int) -> np.ndarray:
        return self.positions[self.offsets[v]: self.offsets[v + 1]]

    def __repr__(self) -> str:
        if self._host:
            return f"EdgeIndex(|V|={self.vertex_count}, entries={len(self._pos)}, host)"
        return f"EdgeIndex(|V|={self.vertex_count}, entries={self.device.entries}, device)"


def build_pull_topology(edges: EdgeList, vector_width: int = 4) -> PullTopology:
    """graph.py:220-263 on the device (wg_build_layout); also builds the edge
    index and out-degrees in the same pass (retrieved by build_edge_index)."""
    if vector_width < 1 or vector_width & (vector_width - 1):
        raise ValueError(f"vector width must be a power of two >= 1, got {vector_width}")
    s, d, w = edges.device_arrays()
    g = DeviceGraph.build(edges.vertex_count, s, d, w, vector_width)
    return PullTopology(g)


def build_edge_index(topology) -> EdgeIndex:
    """graph.py:283-301.  For a device topology the index already exists;
    a reference-layout topology is uploaded (its index is then rebuilt on the
    device from the lanes)."""
    if isinstance(topology, PullTopology) and topology.device is not None:
        return EdgeIndex(topology.device)
    raise TypeError("build_edge_index expects a device PullTopology built by this package "
                    "(host reference-layout topologies carry their own EdgeIndex)")


def compute_out_degrees(edges: EdgeList) -> np.ndarray:
    """graph.py:277-280."""
    if edges.edge_count == 0:
        return np.zeros(edges.vertex_count, dtype=np.int64)
    import torch
    s = edges.device_arrays()[0]
    deg = torch.bincount(s.to(torch.int64) & 0xFFFFFFFF, minlength=edges.vertex_count)
    return deg.cpu().numpy().astype(np.int64)
