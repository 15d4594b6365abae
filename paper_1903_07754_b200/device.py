"""Device runtime: the resident pull layout, the device loop driver, the
per-call kernels of the backend protocol, PageRank and the input generators.

PyTorch is used only as the device-memory / stream provider: every tensor
here is a raw buffer whose pointer is handed to the C ABI (include/wedge_b200.h).
uint32 device data is stored in ``torch.int32`` tensors (same bits).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (WG_VAL_I64, WG_VAL_U32, NO_LANE, REC_FIELDS, REC_U64, WgGraph, WgMinPlus,
                   WgRunBufs, WgRunParams, check)

UNREACHED = 1 << 62  # engine.py:43
SLACK = 16  # vectors of readable slack after vsrc / vdst / vw (TMA tail rounding)
U32_INF = 0xFFFFFFFF


def _torch():
    return _lib.require_cuda()


def _ptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


def _padded(t, extra: int):
    import torch
    out = torch.zeros(t.numel() + extra, dtype=t.dtype, device=t.device)
    out[: t.numel()].copy_(t)
    return out[: t.numel()]


WIDTH_WORDS = 160  # uint32 words of 5-bit vector widths per coded block (wg_coded_width_words)


def to_dev_u32(a, device="cuda"):
    """numpy / torch integer array -> device int32 tensor holding uint32 bits."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.int32:
            return a.to(device).contiguous()
        return (a.to(device=device, dtype=torch.int64) & 0xFFFFFFFF).to(torch.int32).contiguous()
    arr = np.ascontiguousarray(a)
    if arr.dtype != np.uint32:
        if arr.size and (arr.min() < 0 or arr.max() > 0xFFFFFFFF):
            raise ValueError("values do not fit in uint32")
        arr = arr.astype(np.uint32)
    return torch.from_numpy(arr.view(np.int32)).to(device)


def u32_to_np64(t) -> np.ndarray:
    """device int32 (uint32 bits) tensor -> host int64 numpy array."""
    return t.cpu().numpy().view(np.uint32).astype(np.int64)


_INGEST_FLAGS = {"vec_dst outside [0, n)": _lib.WG_INGEST_BAD_DST, "lane source outside [0, n)": _lib.WG_INGEST_BAD_SRC,
                 "lane_count outside [0, W]": _lib.WG_INGEST_BAD_COUNT,
                 "lane weight outside [0, 2^32)": _lib.WG_INGEST_BAD_WEIGHT,
                 "index position outside [0, vector_count)": _lib.WG_INGEST_BAD_POS,
                 "out-degree outside [0, 2^32)": _lib.WG_INGEST_BAD_DEGREE,
                 "index offsets not monotone from 0 to len(positions)": _lib.WG_INGEST_BAD_OFFSETS}


class _IngestStaging:
    """Two device staging slots (int64 chunks) + a copy stream, shared by
    every reference-layout upload on a device (DeviceGraph.from_reference)."""

    _cache = {}

    def __init__(self, device, chunk, width, weighted):
        torch = _torch()
        self.chunk, self.width, self.weighted = chunk, width, weighted
        self.copy = torch.cuda.Stream(device=device)
        self.copy_done = torch.cuda.Event()
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        self.slots = []
        for _ in range(2):
            sl = {"dst": torch.empty(chunk, dtype=torch.int64, device=device),
                  "cnt": torch.empty(chunk, dtype=torch.int64, device=device),
                  "src": torch.empty(chunk * width, dtype=torch.int64, device=device),
                  "w": torch.empty(chunk * width, dtype=torch.int64, device=device) if weighted else None,
                  "ready": torch.cuda.Event(), "free": torch.cuda.Event()}
            self.slots.append(sl)

    def slot(self, k):
        return self.slots[k & 1]

    @classmethod
    def get(cls, device, chunk, width, weighted):
        key = (str(device), chunk, width)
        st = cls._cache.get(key)
        if st is None or (weighted and not st.weighted):
            st = cls._cache[key] = cls(device, chunk, width, weighted)
        return st


# ---------------------------------------------------------------------------
# Device graph
# ---------------------------------------------------------------------------
class DeviceGraph:
    """The pull layout resident in HBM: W-lane vectors ordered by (dst, src),
    their destinations, optional lane weights, the per-source edge index and
    out-degrees.  Replaces PullTopology + EdgeIndex + out-degrees
    (graph.py:109-212) on the device."""

    def __init__(self, n, width, edges, nvec, entries, vsrc, vdst, vw, idx_off, idx_pos, outdeg,
                 lens_are_degrees: bool = False, vw8=None):
        self.n, self.width, self.edges = int(n), int(width), int(edges)
        self.nvec, self.entries = int(nvec), int(entries)
        self.vsrc, self.vdst, self.vw = vsrc, vdst, vw
        self.idx_off, self.idx_pos, self.outdeg = idx_off, idx_pos, outdeg
        # every index length equals the out-degree (WG_GRAPH_LENS_ARE_DEGREES)
        self.lens_are_degrees = bool(lens_are_degrees)
        self.vw8 = vw8  # byte copy of vw when every weight <= 255 (the dense pull streams it)
        self.voff = None  # [n+1] per-destination vector offsets (ensure_voff; destination-major pulls)
        self.vfirst = None  # [n] each destination's smallest source (ensure_voff)
        self._struct = None

    def narrow_weights(self, stream=None) -> bool:
        """Keep a byte copy of the lane weights when all fit (wg_narrow_weights)."""
        torch = _torch()
        if self.vw is None or self.nvec == 0:
            return False
        lanes = self.nvec * self.width
        buf = getattr(self, "_vw8_buf", None)  # reused across re-uploads (stable loop-graph pointers)
        if buf is None or buf.numel() != lanes + 64:
            buf = torch.empty(lanes + 64, dtype=torch.uint8, device=self.vw.device)  # TMA tail slack
            self._vw8_buf = buf
        fits = ctypes.c_int(0)
        check(_lib.load().wg_narrow_weights(ctypes.byref(self.struct()), _ptr(buf), ctypes.byref(fits),
                                            _lib.stream_ptr(stream)))
        self.vw8 = buf if fits.value else None
        self._struct = None
        return bool(fits.value)

    # -- construction ------------------------------------------------------
    @classmethod
    def build(cls, n: int, src, dst, weight=None, width: int = 4, stream=None) -> "DeviceGraph":
        """Build on device from an edge list (graph.py:220-301 via wg_build_layout)."""
        torch = _torch()
        L = _lib.load()
        if width not in (1, 2, 4, 8):
            raise ValueError(f"vector width must be one of 1, 2, 4, 8 on the B200 engine, got {width}")
        s = to_dev_u32(src)
        d = to_dev_u32(dst)
        w = to_dev_u32(weight) if weight is not None else None
        m = int(s.numel())
        if d.numel() != m or (w is not None and w.numel() != m):
            raise ValueError("src/dst/weight lengths differ")
        cap = int(L.wg_vector_capacity(m, n, width))
        dev = s.device
        # +SLACK vectors: TMA bulk copies of the last chunk round up to 16 bytes
        vsrc = torch.empty((cap + SLACK) * width, dtype=torch.int32, device=dev)
        vdst = torch.empty(cap + SLACK, dtype=torch.int32, device=dev)
        vw = torch.empty((cap + SLACK) * width, dtype=torch.int32, device=dev) if w is not None else None
        idx_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        idx_pos = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        outdeg = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        scratch = torch.empty(int(L.wg_layout_scratch_bytes(m, n)), dtype=torch.uint8, device=dev)
        counts = (ctypes.c_uint64 * 2)()
        check(L.wg_build_layout(n, m, _ptr(s), _ptr(d), _ptr(w), width, cap, _ptr(vsrc), _ptr(vdst),
                                _ptr(vw), _ptr(idx_off), _ptr(idx_pos), _ptr(outdeg), _ptr(scratch),
                                scratch.numel(), counts, _lib.stream_ptr(stream)))
        del scratch
        nvec, entries = int(counts[0]), int(counts[1])
        # the built out-degrees count edges and index lengths never exceed
        # them, so equal totals mean equal per vertex
        g = cls(n, width, m, nvec, entries, vsrc[: max(nvec * width, 1)], vdst[: max(nvec, 1)],
                vw[: max(nvec * width, 1)] if vw is not None else None, idx_off,
                idx_pos[: max(entries, 1)], outdeg, lens_are_degrees=(entries == m))
        if vw is not None:
            g.narrow_weights(stream)
        return g

    @classmethod
    def from_reference(cls, topology, index, degrees, device="cuda", into=None, stream=None,
                       chunk_vectors: int = 1 << 22) -> "DeviceGraph":
        """Upload a reference-layout PullTopology / EdgeIndex / degrees
        (int64 host arrays, graph.py:109-212) into the device layout.

        The caller's int64 arrays travel raw, in chunks of `chunk_vectors`
        vectors (index entries / degrees in chunks of as many lanes) through
        two device staging slots: the copy engine moves chunk k+1 while the
        compute stream narrows and validates chunk k (wg_ingest_*), so nothing
        is converted on the host.  `into`: a graph of the same shape whose
        buffers are refilled (the caller's arrays may have changed in place).
        Raises ValueError when an id, weight, degree or offset does not fit
        the layout (a reference kernel would read out of bounds there)."""
        torch = _torch()
        L = _lib.load()
        n, width = int(topology.vertex_count), int(topology.vector_width)
        if width not in (1, 2, 4, 8):
            raise ValueError(f"vector width {width} is not supported by the B200 engine (1, 2, 4, 8)")
        nvec = int(topology.vector_count)
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
        h_dst = i64(topology.vec_dst).reshape(-1)
        h_cnt = i64(topology.lane_count).reshape(-1)
        h_src = i64(topology.lane_src).reshape(-1)
        h_w = None if topology.lane_weight is None else i64(topology.lane_weight).reshape(-1)
        h_off = i64(index.offsets).reshape(-1)
        h_pos = i64(index.positions).reshape(-1)
        h_deg = i64(degrees).reshape(-1)
        entries = int(h_pos.size)
        if h_src.size != nvec * width or h_cnt.size != nvec or (h_w is not None and h_w.size != nvec * width):
            raise ValueError("lane arrays do not match vector_count x vector_width")
        if h_off.size != n + 1 or h_deg.size != n:
            raise ValueError("index offsets / degrees do not match vertex_count")
        weighted = h_w is not None
        shape = (n, width, nvec, entries, weighted)
        g = into if (into is not None and getattr(into, "_ingest_shape", None) == shape) else None
        if g is None:
            vsrc = torch.empty(max(nvec, 1) * width + SLACK * width, dtype=torch.int32, device=device)
            vdst = torch.empty(max(nvec, 1) + SLACK, dtype=torch.int32, device=device)
            vw = torch.empty(max(nvec, 1) * width + SLACK * width, dtype=torch.int32, device=device) if weighted else None
            g = cls(n, width, int(topology.edge_count), nvec, entries,
                    vsrc[: max(nvec * width, 1)], vdst[: max(nvec, 1)],
                    vw[: max(nvec * width, 1)] if weighted else None,
                    torch.empty(n + 1, dtype=torch.int64, device=device),
                    torch.empty(max(entries, 1), dtype=torch.int32, device=device),
                    torch.empty(max(n, 1), dtype=torch.int32, device=device))
            if nvec == 0:
                vsrc.fill_(-1)
            g._ingest_shape = shape
        g.edges = int(topology.edge_count)
        comp = stream or torch.cuda.current_stream()
        st = _IngestStaging.get(device, chunk_vectors, width, weighted)
        st.copy.wait_stream(comp)  # `into`'s buffers may still be read by earlier work
        err = st.err
        err.zero_()
        tens = lambda a: torch.from_numpy(a)
        p = _ptr
        sp = _lib.stream_ptr(comp)

        def run_chunks(total, per, stage, kernel):
            for k, lo in enumerate(range(0, total, per)):
                hi = min(total, lo + per)
                slot = st.slot(k)
                st.copy.wait_event(slot["free"])
                with torch.cuda.stream(st.copy):
                    stage(slot, lo, hi)
                    slot["ready"].record(st.copy)
                comp.wait_event(slot["ready"])
                kernel(slot, lo, hi)
                slot["free"].record(comp)

        # vectors: vdst, vsrc (padding from lane_count), vw
        C = st.chunk

        def stage_vec(slot, lo, hi):
            slot["dst"][: hi - lo].copy_(tens(h_dst[lo:hi]), non_blocking=True)
            slot["cnt"][: hi - lo].copy_(tens(h_cnt[lo:hi]), non_blocking=True)
            slot["src"][: (hi - lo) * width].copy_(tens(h_src[lo * width: hi * width]), non_blocking=True)
            if weighted:
                slot["w"][: (hi - lo) * width].copy_(tens(h_w[lo * width: hi * width]), non_blocking=True)

        def ingest_vec(slot, lo, hi):
            check(L.wg_ingest_vectors(hi - lo, width, n, p(slot["dst"]), p(slot["cnt"]), p(slot["src"]),
                                      p(slot["w"]) if weighted else None, p(g.vdst) + 4 * lo,
                                      p(g.vsrc) + 4 * lo * width, (p(g.vw) + 4 * lo * width) if weighted else None,
                                      p(err), sp))
        run_chunks(nvec, C, stage_vec, ingest_vec)

        # index positions and degrees through the lane slot
        def stage_lin(arr):
            return lambda slot, lo, hi: slot["src"][: hi - lo].copy_(tens(arr[lo:hi]), non_blocking=True)

        run_chunks(entries, C * width, stage_lin(h_pos),
                   lambda slot, lo, hi: check(L.wg_ingest_u32(hi - lo, p(slot["src"]), nvec, p(g.idx_pos) + 4 * lo,
                                                              _lib.WG_INGEST_BAD_POS, p(err), sp)))
        run_chunks(n, C * width, stage_lin(h_deg),
                   lambda slot, lo, hi: check(L.wg_ingest_u32(hi - lo, p(slot["src"]), 1 << 32, p(g.outdeg) + 4 * lo,
                                                              _lib.WG_INGEST_BAD_DEGREE, p(err), sp)))
        with torch.cuda.stream(st.copy):
            g.idx_off.copy_(tens(h_off), non_blocking=True)
            st.copy_done.record(st.copy)
        comp.wait_event(st.copy_done)
        check(L.wg_ingest_offsets(n, p(g.idx_off), entries, p(g.outdeg), p(err), sp))
        bits = int(err.item())  # the one synchronisation of the upload
        bad = bits & ~_lib.WG_INGEST_LENS_DIFFER
        if bad:
            raise ValueError(f"reference layout does not fit the device layout (wg_ingest flags 0x{bad:x}): "
                             + ", ".join(k for k, b in _INGEST_FLAGS.items() if bad & b))
        g.lens_are_degrees = not (bits & _lib.WG_INGEST_LENS_DIFFER)
        g._struct = None
        if g.voff is not None:
            g.ensure_voff(comp, refresh=True)
        g._degrees_src = degrees  # the out-degrees this graph holds (engine._with_degrees)
        g._all_counts = None
        g.vw8 = None
        if weighted:
            g.narrow_weights(comp)
        return g

    # -- compact upload form -------------------------------------------------
    def vector_offsets(self):
        """Per-destination vector offsets voff [n+1] (uint32): the run-length
        form of vdst (vec_dst of graph.py:240-243)."""
        torch = _torch()
        cnt = torch.bincount(self.vdst[: self.nvec].to(torch.int64) & 0xFFFFFFFF, minlength=self.n)
        off = torch.zeros(self.n + 1, dtype=torch.int64, device=self.vdst.device)
        off[1:] = torch.cumsum(cnt, 0)
        return off.to(torch.int32)

    @classmethod
    def from_lanes(cls, n: int, width: int, edges: int, nvec: int, vsrc, vw, voff, scratch=None,
                   stream=None) -> "DeviceGraph":
        """Rebuild a layout from its lanes and per-destination vector offsets
        (device tensors): vdst by wg_expand_destinations, the edge index and
        out-degrees by wg_build_index.  vsrc needs SLACK vectors of readable
        slack past nvec*width (TMA tail rounding); so does the vdst made here."""
        torch = _torch()
        L = _lib.load()
        dev = vsrc.device
        vdst = torch.empty(nvec + SLACK, dtype=torch.int32, device=dev)
        idx_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        idx_pos = torch.empty(max(edges, 1), dtype=torch.int32, device=dev)
        outdeg = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        g = cls(n, width, edges, nvec, 0, vsrc, vdst[: max(nvec, 1)], vw, idx_off, idx_pos, outdeg)
        g.rebuild_derived(voff, scratch, stream)
        return g

    def lane_bits(self) -> int:
        """Bit width of one lane in the packed upload format (wg_lane_bits)."""
        return int(_lib.load().wg_lane_bits(self.n))

    def pack_lanes(self, stream=None):
        """vsrc as fixed-width bit fields (wg_pack_lanes): (int32 words, bits)."""
        torch = _torch()
        L = _lib.load()
        bits = self.lane_bits()
        lanes = self.nvec * self.width
        words = int(L.wg_packed_lane_words(lanes, bits))
        out = torch.empty(max(words, 1), dtype=torch.int32, device=self.vsrc.device)
        check(L.wg_pack_lanes(lanes, _ptr(self.vsrc), bits, _ptr(out), _lib.stream_ptr(stream)))
        return out[:words], bits

    def encode_lanes(self, stream=None) -> dict:
        """vsrc in the delta-coded upload format (wg_encode_lanes): device
        tensors "lane_stream" (int32 words), "lane_widths" (int32 words, 5
        bits per vector, WIDTH_WORDS per block) and "lane_blocks" (int64 block
        bit offsets, blocks + 1)."""
        torch = _torch()
        L = _lib.load()
        dev = self.vsrc.device
        nb = int(L.wg_coded_blocks(self.nvec))
        words = torch.empty(max(int(L.wg_coded_max_words(self.nvec, self.width)), 1), dtype=torch.int32, device=dev)
        widths = torch.empty(max(int(L.wg_coded_width_words(self.nvec)), 1), dtype=torch.int32, device=dev)
        blocks = torch.empty(nb + 1, dtype=torch.int64, device=dev)
        scratch = torch.empty(int(L.wg_coded_scratch_bytes(self.nvec)), dtype=torch.uint8, device=dev)
        used = ctypes.c_uint64(0)
        check(L.wg_encode_lanes(ctypes.byref(self.struct()), _ptr(words), _ptr(widths), _ptr(blocks), _ptr(scratch),
                                scratch.numel(), ctypes.byref(used), _lib.stream_ptr(stream)))
        return {"lane_stream": words[: int(used.value)], "lane_widths": widths[: int(L.wg_coded_width_words(self.nvec))],
                "lane_blocks": blocks}

    def in_degrees(self):
        """Real lanes per destination (device int32 [n])."""
        torch = _torch()
        lanes = self.vsrc[: self.nvec * self.width].view(self.nvec, self.width)
        real = (lanes != -1).sum(1).to(torch.int32)
        deg = torch.zeros(self.n, dtype=torch.int32, device=self.vsrc.device)
        return deg.index_add_(0, self.vdst[: self.nvec].to(torch.int64) & 0xFFFFFFFF, real)

    @staticmethod
    def compact_degrees(deg):
        """(min(deg, 255) as uint8, int32 [k, 2] (vertex, degree) for the rest)
        -- the upload form wg_widen_degrees reads (a tensor op on deg's device)."""
        import torch
        big = torch.nonzero(deg >= 255).flatten()
        pairs = torch.stack([big.to(torch.int32), deg[big].to(torch.int32)], 1).contiguous()
        return deg.clamp(max=255).to(torch.uint8), pairs

    def host_format(self, symmetric: bool = False) -> dict:
        """The compact host-resident topology of the e2e upload (pinned):
        delta-coded lanes, in-degrees (from which voff is rebuilt) and, unless
        the caller declares the graph symmetric (out-degrees = in-degrees,
        verified on the device by the placed index), the out-degrees, both as
        a byte per vertex plus the larger ones as (vertex, degree) pairs."""
        host = {k: v.cpu().pin_memory() for k, v in self.encode_lanes().items()}
        d8, big = self.compact_degrees(self.in_degrees())
        host["indeg8"], host["indeg_big"] = d8.cpu().pin_memory(), big.cpu().pin_memory()
        if not symmetric:
            o8, obig = self.compact_degrees(self.outdeg[: self.n])
            host["outdeg8"], host["outdeg_big"] = o8.cpu().pin_memory(), obig.cpu().pin_memory()
        return host

    def upload_rebuild(self, host: dict, dev: dict, chunks: int = 4, scratch=None, copy_stream=None,
                       trace=None, index: bool = True, outdeg_is_indeg: bool = False) -> int:
        """Copy the compact topology from pinned host memory (host["vsrc"],
        its bit-packed form host["vsrc_bits"] or its delta-coded form
        host["lane_stream"/"lane_widths"/"lane_blocks"], host["voff"], optional
        host["vw8"] / host["vw"]) into this graph's device arrays (dev[...]
        views of them; dev["vsrc_bits"] receives the packed words) and rebuild
        vsrc (unpacked chunk by chunk), vec_dst, the edge index and the
        out-degrees, with the index built chunk by chunk so each chunk's sort
        overlaps the copy of the next (wg_unpack_lanes, wg_index_chunk /
        wg_index_finish).  With host["outdeg"] (the out-degrees, the
        `degrees` input of the reference call) the index is placed instead:
        offsets from the degrees, every chunk's lanes take their slots as the
        chunk arrives (wg_index_place_*; the same lists with the order inside
        each list unspecified, no sort), verified at the end, with the
        sort-based builder as the fallback.  index=False rebuilds only
        vsrc and vec_dst (PageRank reads no index; host["outdeg"] then just
        lands in the out-degrees).  The compact degree form (host_format:
        "indeg8"/"indeg_big" instead of voff, "outdeg8"/"outdeg_big" or
        outdeg_is_indeg for a symmetric graph) is widened on the device
        (wg_widen_degrees, wg_vector_offsets).  Returns the index length (0
        without).  trace: an optional list that receives (label, event)
        pairs (profiling)."""
        torch = _torch()
        L = _lib.load()
        cs = copy_stream or torch.cuda.Stream()
        main = torch.cuda.current_stream()
        W = self.width
        packed = "vsrc_bits" in host
        coded = "lane_stream" in host
        compact = "indeg8" in host
        has_deg = "outdeg" in host or "outdeg8" in host or (compact and outdeg_is_indeg)
        placed = has_deg and index
        if compact and getattr(self, "_indeg", None) is None:
            self._indeg = torch.empty(self.n + 1, dtype=torch.int32, device=self.vsrc.device)
            self._voff = torch.empty(self.n + 1, dtype=torch.int32, device=self.vsrc.device)
        for k in ("indeg8", "indeg_big", "outdeg8", "outdeg_big"):
            if k in host and k not in dev:
                dev[k] = torch.empty(max(host[k].numel(), 1), dtype=host[k].dtype,
                                     device=self.vsrc.device)[: host[k].numel()].view(host[k].shape)
        bits = self.lane_bits() if packed else 32
        # packed chunks start on a word: lane offsets multiples of 32; coded
        # chunks are runs of whole blocks
        align = max(1, 32 // W) if packed else (_lib.WG_CODED_BLOCK_VECTORS if coded else 1)
        cuts = [min(self.nvec, (self.nvec * c // chunks) // align * align) for c in range(chunks)] + [self.nvec]
        if coded:
            base = host["lane_blocks"].numpy()
        max_lanes = max(max(cuts[c + 1] - cuts[c] for c in range(chunks)) * W, 1)
        need = max(int(L.wg_index_chunked_scratch_bytes(self.nvec * W, max_lanes, self.n)),
                   int(L.wg_index_scratch_bytes(self.nvec * W, self.n)), int(L.wg_expand_scratch_bytes(self.nvec)),
                   int(L.wg_index_placed_scratch_bytes(self.n)), int(L.wg_vector_offsets_scratch_bytes(self.n)))
        if scratch is None or scratch.numel() < need:
            scratch = torch.empty(need, dtype=torch.uint8, device=self.vsrc.device)
        words = int(host["vsrc_bits"].numel()) if packed else 0
        cs.wait_stream(main)  # the previous use of the buffers is done
        evs = []
        with torch.cuda.stream(cs):
            for k in ("voff", "indeg8", "indeg_big", "outdeg8", "outdeg_big"):
                if k in host and host[k].numel():
                    dev[k].copy_(host[k], non_blocking=True)
            if "outdeg" in host:
                self.outdeg[: self.n].copy_(host["outdeg"], non_blocking=True)
            if coded:
                dev["lane_blocks"].copy_(host["lane_blocks"], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
            evs.append(e)
            for c in range(chunks):
                a, b = cuts[c] * W, cuts[c + 1] * W
                if packed:
                    wa, wb = a * bits // 32, (words if c == chunks - 1 else b * bits // 32)
                    dev["vsrc_bits"][wa:wb].copy_(host["vsrc_bits"][wa:wb], non_blocking=True)
                elif coded:
                    ba, bb = cuts[c] // align, -(-cuts[c + 1] // align)
                    wa, wb = int(base[ba]) // 32, int(base[bb]) // 32
                    dev["lane_stream"][wa:wb].copy_(host["lane_stream"][wa:wb], non_blocking=True)
                    dev["lane_widths"][ba * WIDTH_WORDS: bb * WIDTH_WORDS].copy_(
                        host["lane_widths"][ba * WIDTH_WORDS: bb * WIDTH_WORDS], non_blocking=True)
                else:
                    dev["vsrc"][a:b].copy_(host["vsrc"][a:b], non_blocking=True)
                e = torch.cuda.Event(enable_timing=trace is not None)
                e.record(cs)
                evs.append(e)
                if trace is not None:
                    trace.append((f"copied {c}", e))
            for k in ("vw8", "vw"):
                if k in host:
                    dev[k].copy_(host[k], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
            evs.append(e)
        st = _lib.stream_ptr()
        main.wait_event(evs[0])
        voff = dev.get("voff")
        if compact:  # in-degrees -> voff; out-degrees
            check(L.wg_widen_degrees(self.n, _ptr(dev["indeg8"]), _ptr(dev["indeg_big"]), host["indeg_big"].shape[0],
                                     _ptr(self._indeg), st))
            check(L.wg_vector_offsets(self.n, _ptr(self._indeg), W, _ptr(self._voff), _ptr(scratch), scratch.numel(),
                                      st))
            voff = self._voff
            if "outdeg8" in host:
                check(L.wg_widen_degrees(self.n, _ptr(dev["outdeg8"]), _ptr(dev["outdeg_big"]),
                                         host["outdeg_big"].shape[0], _ptr(self.outdeg), st))
            elif outdeg_is_indeg:
                self.outdeg[: self.n].copy_(self._indeg[: self.n])
        check(L.wg_expand_destinations(self.n, _ptr(voff), self.nvec, _ptr(self.vdst), _ptr(scratch),
                                       scratch.numel(), st))
        gs = ctypes.byref(self.struct())
        if placed:
            check(L.wg_index_place_begin(gs, _ptr(self.idx_off), _ptr(scratch), scratch.numel(), st))
        for c in range(chunks):
            main.wait_event(evs[1 + c])
            if packed:
                check(L.wg_unpack_lanes(_ptr(dev["vsrc_bits"]), bits, cuts[c] * W, cuts[c + 1] * W,
                                        _ptr(self.vsrc), st))
            if trace is not None:
                trace.append((f"decoded {c}", torch.cuda.Event(enable_timing=True)))
                trace[-1][1].record(main)
            if not index:  # lanes only
                if coded:
                    check(L.wg_decode_lanes(self.nvec, W, _ptr(self.vdst), _ptr(dev["lane_stream"]),
                                            _ptr(dev["lane_widths"]), _ptr(dev["lane_blocks"]), cuts[c] // align,
                                            -(-cuts[c + 1] // align), _ptr(self.vsrc), st))
            elif placed and coded:  # decode fused with the placement
                check(L.wg_index_place_coded(gs, _ptr(dev["lane_stream"]), _ptr(dev["lane_widths"]),
                                             _ptr(dev["lane_blocks"]), cuts[c] // align, -(-cuts[c + 1] // align),
                                             _ptr(self.idx_off), _ptr(self.idx_pos), _ptr(scratch), scratch.numel(),
                                             st))
            elif placed:
                check(L.wg_index_place_chunk(gs, cuts[c], cuts[c + 1], _ptr(self.idx_off), _ptr(self.idx_pos),
                                             _ptr(scratch), scratch.numel(), st))
            elif coded:  # decode fused into the chunk's pair generation
                check(L.wg_index_chunk_coded(gs, _ptr(dev["lane_stream"]), _ptr(dev["lane_widths"]),
                                             _ptr(dev["lane_blocks"]), cuts[c] // align, -(-cuts[c + 1] // align), c,
                                             max_lanes, _ptr(scratch), scratch.numel(), st))
            else:
                check(L.wg_index_chunk(gs, cuts[c], cuts[c + 1], c, max_lanes, _ptr(scratch), scratch.numel(), st))
            if trace is not None:
                trace.append((f"indexed {c}", torch.cuda.Event(enable_timing=True)))
                trace[-1][1].record(main)
        ent = ctypes.c_uint64(0)
        if not index:
            pass
        elif placed:
            ok = ctypes.c_int(0)
            check(L.wg_index_place_end(gs, _ptr(scratch), scratch.numel(), ctypes.byref(ok), st))
            if ok.value:
                ent.value = self.edges
            else:  # parallel edges or degrees that do not match the lanes
                check(L.wg_build_index(gs, _ptr(self.idx_off), _ptr(self.idx_pos), _ptr(self.outdeg), _ptr(scratch),
                                       scratch.numel(), ctypes.byref(ent), st))
        else:
            check(L.wg_index_finish(gs, max_lanes, _ptr(self.idx_off), _ptr(self.idx_pos), _ptr(self.outdeg),
                                    _ptr(scratch), scratch.numel(), ctypes.byref(ent), st))
        if trace is not None:
            trace.append(("finished", torch.cuda.Event(enable_timing=True)))
            trace[-1][1].record(main)
        main.wait_event(evs[-1])
        if "vw8" in host and self.vw is not None:
            check(L.wg_widen_weights(self.nvec * W, _ptr(dev["vw8"]), _ptr(self.vw), st))
        self._upload_scratch = scratch
        return int(ent.value)

    def rebuild_derived(self, voff, scratch=None, stream=None) -> int:
        """Recompute vdst, the edge index and the out-degrees in place from
        vsrc and voff (the arrays keep their addresses, so captured loop
        graphs stay valid).  Returns the index length."""
        torch = _torch()
        L = _lib.load()
        need = max(int(L.wg_index_scratch_bytes(self.nvec * self.width, self.n)),
                   int(L.wg_expand_scratch_bytes(self.nvec)))
        if scratch is None or scratch.numel() < need:
            scratch = torch.empty(need, dtype=torch.uint8, device=self.vsrc.device)
        check(L.wg_expand_destinations(self.n, _ptr(voff), self.nvec, _ptr(self.vdst), _ptr(scratch), scratch.numel(),
                                       _lib.stream_ptr(stream)))
        ent = ctypes.c_uint64(0)
        check(L.wg_build_index(ctypes.byref(self.struct()), _ptr(self.idx_off), _ptr(self.idx_pos),
                               _ptr(self.outdeg), _ptr(scratch), scratch.numel(), ctypes.byref(ent),
                               _lib.stream_ptr(stream)))
        entries = int(ent.value)
        if entries != self.entries:
            self.entries = entries
            self.idx_pos = self.idx_pos[: max(entries, 1)] if self.idx_pos.numel() >= entries else self.idx_pos
            self.lens_are_degrees = entries == self.edges
            self._struct = None
        return entries

    def struct(self) -> WgGraph:
        if self._struct is None:
            self._struct = WgGraph(self.n, self.width, self.nvec, self.edges, self.entries,
                                   _ptr(self.vsrc), _ptr(self.vdst), _ptr(self.vw), _ptr(self.idx_off),
                                   _ptr(self.idx_pos), _ptr(self.outdeg),
                                   _lib.WG_GRAPH_LENS_ARE_DEGREES if self.lens_are_degrees else 0,
                                   _ptr(self.vw8), _ptr(self.voff), _ptr(self.vfirst))
        return self._struct

    def all_vertex_counts(self):
        """Counts of the frontier holding every vertex (cached): members with
        index entries, their entries, members without, out-degree sum."""
        c = getattr(self, "_all_counts", None)
        if c is None:
            torch = _torch()
            deg = self.outdeg[: self.n].to(torch.int64) & U32_INF
            lens = deg if self.lens_are_degrees else (self.idx_off[1: self.n + 1] - self.idx_off[: self.n])
            nz = int((lens > 0).sum().item())
            c = (nz, int(lens.sum().item()), self.n - nz, int(deg.sum().item()))
            self._all_counts = c
        return c

    def ensure_voff(self, stream=None, refresh: bool = False):
        """Per-destination vector offsets (wg_vector_offsets_from_dst), kept
        resident for the destination-major dense pulls (WG_DST_MAJOR=0
        disables them)."""
        if os.environ.get("WG_DST_MAJOR", "1") == "0":
            if self.voff is not None:
                self.voff = self.vfirst = None
                self._struct = None
            return None
        if self.voff is not None and not refresh:
            return self.voff
        torch = _torch()
        if self.voff is None or self.voff.numel() != self.n + 1:
            self.voff = torch.empty(self.n + 1, dtype=torch.int32, device=self.vdst.device)
            self.vfirst = torch.empty(max(self.n, 1), dtype=torch.int32, device=self.vdst.device)
        self._struct = None
        L = _lib.load()
        vf = self.vfirst
        self.vfirst = None  # the struct handed to the builders carries voff only
        check(L.wg_vector_offsets_from_dst(ctypes.byref(self.struct()), _ptr(self.voff), _lib.stream_ptr(stream)))
        check(L.wg_first_lanes(ctypes.byref(self.struct()), _ptr(self.voff), _ptr(vf), _lib.stream_ptr(stream)))
        self.vfirst = vf
        self._struct = None
        return self.voff

    def signature(self) -> bytes:
        """Every field of the C struct: a loop graph captured for one
        signature must not be replayed after any of them changed."""
        st = self.struct()
        return ctypes.string_at(ctypes.addressof(st), ctypes.sizeof(st))

    def weighted(self) -> bool:
        return self.vw is not None

    # -- host views in the reference layout (int64) -------------------------
    def vec_dst_np(self) -> np.ndarray:
        return u32_to_np64(self.vdst[: self.nvec]) if self.nvec else np.empty(0, np.int64)

    def lanes_np(self):
        """(lane_src, lane_weight, lane_count) with the reference's zero padding."""
        W = self.width
        if self.nvec == 0:
            e = np.empty((0, W), np.int64)
            return e, (e.copy() if self.weighted() else None), np.empty(0, np.int64)
        vs = self.vsrc[: self.nvec * W].cpu().numpy().view(np.uint32).reshape(self.nvec, W)
        valid = vs != NO_LANE
        lane_src = np.where(valid, vs.astype(np.int64), 0)
        lane_w = None
        if self.weighted():
            lw = self.vw[: self.nvec * W].cpu().numpy().view(np.uint32).reshape(self.nvec, W)
            lane_w = np.where(valid, lw.astype(np.int64), 0)
        return lane_src, lane_w, valid.sum(axis=1).astype(np.int64)

    def offsets_np(self) -> np.ndarray:
        return self.idx_off.cpu().numpy().astype(np.int64)

    def positions_np(self) -> np.ndarray:
        return u32_to_np64(self.idx_pos[: self.entries]) if self.entries else np.empty(0, np.int64)

    def outdeg_np(self) -> np.ndarray:
        return u32_to_np64(self.outdeg[: self.n]) if self.n else np.empty(0, np.int64)

    def memory_bytes(self) -> int:
        t = [self.vsrc, self.vdst, self.vw, self.vw8, self.idx_off, self.idx_pos, self.outdeg]
        return sum(x.numel() * x.element_size() for x in t if x is not None)


# ---------------------------------------------------------------------------
# Per-call kernels: the reference backend protocol (kernels.py:55-125)
# ---------------------------------------------------------------------------
def _minplus(kern, sentinel) -> WgMinPlus:
    return WgMinPlus(int(bool(kern.filter_unvisited)), int(bool(kern.use_weight)),
                     int(kern.apply_increment), int(sentinel))


def _workspace(g: DeviceGraph, shift: int):
    torch = _torch()
    nbytes = int(_lib.load().wg_kernel_workspace_bytes(ctypes.byref(g.struct()), shift))
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")


def _words_dev(words_u64: np.ndarray, nbits: int):
    """uint64 LE words (reference Bitmask) -> device uint32 words (same bytes)."""
    torch = _torch()
    w = np.ascontiguousarray(words_u64, dtype=np.uint64).view(np.int32)
    need = (nbits + 31) >> 5
    out = torch.zeros(max(need, w.size, 1), dtype=torch.int32, device="cuda")
    if w.size:
        out[: w.size].copy_(torch.from_numpy(w.copy()))
    return out


def _words_back(dev_words, out_u64: np.ndarray) -> None:
    host = dev_words.cpu().numpy().view(np.uint32)
    view = out_u64.view(np.uint32)
    view[:] = host[: view.size]


def pull_call(g: DeviceGraph, prev: np.ndarray, nxt: np.ndarray, out_words: np.ndarray, kern,
              sentinel: int, wedge_words: Optional[np.ndarray] = None, shift: int = 0) -> int:
    """Run wg_pull_full / wg_pull_wedge on host int64 buffers (reference
    semantics, WG_VAL_I64) and write nxt / out_words back in place."""
    torch = _torch()
    L = _lib.load()
    if g.nvec == 0:
        return 0
    dprev = torch.from_numpy(np.ascontiguousarray(prev, dtype=np.int64)).cuda()
    dnxt = torch.from_numpy(np.ascontiguousarray(nxt, dtype=np.int64)).cuda()
    dout = _words_dev(out_words, g.n)
    ws = _workspace(g, shift)
    k = _minplus(kern, sentinel)
    touched = ctypes.c_uint64(0)
    st = _lib.stream_ptr()
    if wedge_words is None:
        check(L.wg_pull_full(ctypes.byref(g.struct()), WG_VAL_I64, _ptr(dprev), _ptr(dnxt), _ptr(dout),
                             ctypes.byref(k), _ptr(ws), ws.numel(), ctypes.byref(touched), st))
    else:
        groups = (g.nvec + (1 << shift) - 1) >> shift
        dw = _words_dev(wedge_words, groups)
        check(L.wg_pull_wedge(ctypes.byref(g.struct()), _ptr(dw), shift, WG_VAL_I64, _ptr(dprev),
                              _ptr(dnxt), _ptr(dout), ctypes.byref(k), _ptr(ws), ws.numel(),
                              ctypes.byref(touched), st))
    nxt[...] = dnxt.cpu().numpy()
    _words_back(dout, out_words)
    return int(touched.value)


def transform_call(g: DeviceGraph, frontier_words: np.ndarray, shift: int,
                   wedge_words: np.ndarray) -> int:
    """wg_transform on host buffers: OR group bits into wedge_words; returns
    index entries visited (frontier.py:174-209)."""
    L = _lib.load()
    groups = (g.nvec + (1 << shift) - 1) >> shift
    df = _words_dev(frontier_words, g.n)
    dw = _words_dev(wedge_words, groups)
    ws = _workspace(g, shift)
    visited = ctypes.c_uint64(0)
    check(L.wg_transform(ctypes.byref(g.struct()), _ptr(df), shift, _ptr(dw), _ptr(ws), ws.numel(),
                         ctypes.byref(visited), _lib.stream_ptr()))
    _words_back(dw, wedge_words)
    return int(visited.value)


def covered_groups(words_u64: np.ndarray, group_count: int) -> np.ndarray:
    """Ascending set group ids (device compaction, K4)."""
    torch = _torch()
    L = _lib.load()
    if group_count == 0:
        return np.empty(0, np.int64)
    dw = _words_dev(words_u64, group_count)
    out = torch.empty(group_count, dtype=torch.int32, device="cuda")
    ws = torch.empty(4096 + 16 * ((group_count >> 15) + 2) + 1024, dtype=torch.uint8, device="cuda")
    cnt = ctypes.c_uint64(0)
    check(L.wg_covered_groups(_ptr(dw), group_count, _ptr(out), _ptr(ws), ws.numel(),
                              ctypes.byref(cnt), _lib.stream_ptr()))
    return u32_to_np64(out[: cnt.value]) if cnt.value else np.empty(0, np.int64)


# ---------------------------------------------------------------------------
# Device-resident convergence loop (engine.py:330-388)
# ---------------------------------------------------------------------------
MODE_NAMES = {1: "FullScan", 2: "Wedge"}


HEAD_RECORDS = 64  # records read back with the control words (drive_graph)


@dataclass
class IterRecord:
    iteration: int
    mode: str
    active_edges: int
    vectors_touched: int
    frontier_out_size: int
    covered_vectors: int
    transform_entries: int
    lanes_read: int = 0   # destination-major dense pulls: lanes read ...
    gathers: int = 0      # ... and gathers / bit tests made (their algorithmic bytes)


@dataclass
class LoopResult:
    values: object            # device tensor (int32 bits of uint32, or int64)
    val_type: int
    records: list = field(default_factory=list)
    converged: bool = False

    def values_int64(self) -> np.ndarray:
        """Final values in the reference encoding (int64, UNREACHED sentinel)."""
        return values_to_int64(self.values, self.val_type)


def values_to_int64(t, val_type: int) -> np.ndarray:
    """Device values -> host int64 with the reference sentinel (engine.py:43),
    widened on the device and read into pinned host memory."""
    torch = _torch()
    if val_type == WG_VAL_I64:
        v = t
    else:
        v = t.to(torch.int64) & U32_INF
        v.masked_fill_(v == U32_INF, UNREACHED)
    out = torch.empty(v.shape, dtype=torch.int64, pin_memory=True)
    out.copy_(v)
    return out.numpy()


def wedge_limit(threshold: Fraction, edges: int) -> int:
    """Smallest edge sum that is NOT below the threshold share:
    sum*den < num*E  <=>  sum < ceil(num*E/den) (frontier.py:163-171)."""
    num, den = threshold.numerator, threshold.denominator
    return -((-num * edges) // den)


FUSED_MAX_LEN = 256  # pull.cuh FUSED_MAX_LEN


def fused_transform_pays(g: DeviceGraph) -> bool:
    """Fuse the Wedge transform into the persistent loop's pull when no
    vertex has more than FUSED_MAX_LEN out-edges (measured: grid SSSP 635 ->
    505 ms; RMAT s26 BFS 11.2 -> 11.8 ms, so power-law graphs keep two phases).
    WG_FUSED_LOOP=0/1 forces it."""
    import os
    env = os.environ.get("WG_FUSED_LOOP")
    if env:
        return env != "0"
    if g.n == 0:
        return False
    return int(g.outdeg[: g.n].max().item()) <= FUSED_MAX_LEN


class DeviceLoop:
    """Buffers and host driver of the device loop for one graph / precision.

    The host enqueues batches of iterations (wg_run_enqueue); every kernel
    re-derives the gate and convergence from the previous iteration's device
    record, so the host only reads the records after each batch.
    """

    def __init__(self, g: DeviceGraph, shift: int, val_type: int = WG_VAL_U32, ring: int = 1024,
                 fused: Optional[bool] = None):
        torch = _torch()
        self.g, self.shift, self.val_type, self.ring = g, int(shift), int(val_type), int(ring)
        L = _lib.load()
        sizes = (ctypes.c_uint64 * 5)()
        check(L.wg_run_buffer_sizes(ctypes.byref(g.struct()), self.shift, sizes))
        fwords, groups, gwords, nbc, ntst = (int(x) for x in sizes)
        n = max(g.n, 1)
        dt = torch.int32 if self.val_type == WG_VAL_U32 else torch.int64
        dev = "cuda"
        self.vals = [torch.empty(n, dtype=dt, device=dev) for _ in range(2)]
        self.fbits = [torch.zeros(max(fwords, 1), dtype=torch.int32, device=dev) for _ in range(2)]
        self.fvert = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
        self.fpref = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
        self.tstart = [torch.zeros(max(ntst, 1), dtype=torch.int32, device=dev) for _ in range(2)]
        self.gbits = torch.zeros(max(gwords, 1), dtype=torch.int32, device=dev)
        self.glist = torch.empty(max(groups, 1), dtype=torch.int32, device=dev)
        # second group buffers: the persistent sparse loop fuses the next
        # iteration's transform into the pull (wg_run_bufs.gbits_alt) on
        # graphs without long index lists (meshes, road-like graphs); with
        # hubs the separate load-balanced transform phase is faster
        self.fused = fused_transform_pays(g) if fused is None else bool(fused)
        self.gbits_alt = torch.zeros(max(gwords, 1), dtype=torch.int32, device=dev) if self.fused else None
        self.glist_alt = torch.empty(max(groups, 1), dtype=torch.int32, device=dev) if self.fused else None
        self.bcount = torch.empty(max(nbc, 1), dtype=torch.int64, device=dev)
        g.ensure_voff()
        self.work = torch.zeros(n + 64, dtype=torch.int32, device=dev)  # >= 8 words per 8192-vertex chunk
        # control words and the record ring in one allocation (ctrl first): a
        # short run's state comes back in ONE small D2H copy (drive_graph)
        self.state = torch.zeros(4 + self.ring * REC_U64, dtype=torch.int64, device=dev)
        self.ctrl, self.recs = self.state[:4], self.state[4:]
        self.host_state = torch.zeros(4 + self.ring * REC_U64, dtype=torch.int64).pin_memory()
        self.ctrl_host, self.host_recs = self.host_state[:4], self.host_state[4:]
        self._host_np = self.host_state.numpy().view(np.uint64)
        b = WgRunBufs()
        for i in range(2):
            b.vals[i] = _ptr(self.vals[i])
            b.fbits[i] = _ptr(self.fbits[i])
            b.fvert[i] = _ptr(self.fvert[i])
            b.fpref[i] = _ptr(self.fpref[i])
            b.tstart[i] = _ptr(self.tstart[i])
        b.gbits, b.glist, b.bcount = _ptr(self.gbits), _ptr(self.glist), _ptr(self.bcount)
        b.gbits_alt, b.glist_alt = _ptr(self.gbits_alt), _ptr(self.glist_alt)
        b.recs, b.ctrl, b.ring = _ptr(self.recs), _ptr(self.ctrl), self.ring
        b.work = _ptr(self.work)
        self.bufs = b
        self.graph_cache = {}
        self._level_base = 0

    def params(self, kern, threshold: Fraction, first_hit: bool = False,
               identity_init: bool = False, extra_flags: int = 0) -> WgRunParams:
        ck = (kern, threshold, first_hit, identity_init, extra_flags, self._level_base if first_hit else 0,
              os.environ.get("WG_FLOOR_SKIP", "1"), self.g.edges, self.g.entries)
        hit = getattr(self, "_params_cache", None)
        if hit is not None and hit[0] == ck:
            return WgRunParams.from_buffer_copy(hit[1])  # a fresh copy: callers may set timer / flags
        p = self._make_params(kern, threshold, first_hit, identity_init, extra_flags)
        self._params_cache = (ck, WgRunParams.from_buffer_copy(p))
        return p

    def _make_params(self, kern, threshold: Fraction, first_hit: bool = False,
                     identity_init: bool = False, extra_flags: int = 0) -> WgRunParams:
        p = WgRunParams()
        p.val_type = self.val_type
        p.shift = self.shift
        p.kern = _minplus(kern, UNREACHED)
        # WG_RUN_LOCAL_GATE (shards): the gate compares the shard's own index entries
        total = self.g.entries if extra_flags & _lib.WG_RUN_LOCAL_GATE else self.g.edges
        p.wedge_limit = wedge_limit(threshold, total) if total > 0 else 0
        p.flags = (_lib.WG_RUN_FIRST_HIT if first_hit else 0) | (_lib.WG_RUN_IDENTITY_INIT if identity_init else 0)
        p.flags |= int(extra_flags)
        if identity_init and os.environ.get("WG_FLOOR_SKIP", "1") != "0":
            p.flags |= _lib.WG_RUN_FLOOR_SKIP  # CC-like runs: label 0 spreads over the giant component
        p.level_base = int(self._level_base) if first_hit else 0
        return p

    def seed(self, init_values, init_words, kern, threshold, stream=None, first_hit: bool = False,
             level_base: int = 0, identity_init: bool = False, extra_flags: int = 0,
             defer: bool = False) -> WgRunParams:
        """Write both value buffers and build iteration 0 from the frontier bitmap.
        first_hit: the caller checked first_hit_ok (level-synchronous values);
        level_base: then the common value of the initial frontier (first_hit_level).
        defer: leave the seed to the next drive(), which runs it as the first
        nodes of the loop graph (one launch per run; wg_run_loop_graph_create_seeded)."""
        if init_values.numel() < self.g.n or init_values.dtype != self.vals[0].dtype:
            raise ValueError("initial values do not match the loop's value buffers")
        self._level_base = int(level_base)
        p = self.params(kern, threshold, first_hit, identity_init, extra_flags)
        counts = None
        if getattr(init_words, "_wg_all", False) and not (p.flags & _lib.WG_RUN_KEEP_LISTS):
            c4 = self.g.all_vertex_counts()
            if not (self.g.edges > 0 and c4[3] < p.wedge_limit):  # iteration 1 is dense
                counts = tuple(int(x) for x in c4)
        self._pending = (init_values, init_words, counts)
        if not defer:
            self._run_pending_seed(p, stream)
        return p

    def _run_pending_seed(self, p, stream=None):
        init_values, init_words, counts = self._pending
        self._pending = None
        c = (ctypes.c_uint64 * 4)(*counts) if counts is not None else None
        check(_lib.load().wg_run_seed(ctypes.byref(self.g.struct()), ctypes.byref(self.bufs), ctypes.byref(p),
                                      _ptr(init_values), _ptr(init_words), c, _lib.stream_ptr(stream)))

    def enqueue(self, p: WgRunParams, it_begin: int, count: int, stream=None) -> None:
        if getattr(self, "_pending", None) is not None:
            self._run_pending_seed(p, stream)
        check(_lib.load().wg_run_enqueue(ctypes.byref(self.g.struct()), ctypes.byref(self.bufs),
                                         ctypes.byref(p), it_begin, count, _lib.stream_ptr(stream)))

    def _read(self, it_begin: int, count: int, stream=None):
        torch = _torch()
        s = stream or torch.cuda.current_stream()
        lo = it_begin % self.ring
        hi = lo + count
        if hi <= self.ring:
            self.host_recs[lo * REC_U64: hi * REC_U64].copy_(self.recs[lo * REC_U64: hi * REC_U64],
                                                             non_blocking=True)
        else:
            self.host_recs.copy_(self.recs, non_blocking=True)
        s.synchronize()
        arr = self.host_recs.numpy().view(np.uint64).reshape(self.ring, REC_U64)
        return [arr[(it_begin + j) % self.ring] for j in range(count)]

    def launch(self, p: WgRunParams, limit: int, stream=None) -> None:
        """Run the loop graph up to iteration `limit` without reading anything
        back (one launch instead of one per kernel; the caller synchronises)."""
        if getattr(self, "_pending", None) is not None:
            self._run_pending_seed(p, stream)
        check(_lib.load().wg_run_loop_launch(self._graph_for(p, stream), ctypes.byref(self.bufs), int(limit),
                                             _lib.stream_ptr(stream)))

    def _seed_buffers(self, words_numel: int):
        """The seeded graph's own initial-state buffers."""
        torch = _torch()
        if getattr(self, "seed_vals", None) is None:
            self.seed_vals = torch.empty_like(self.vals[0])
        if getattr(self, "seed_words", None) is None or self.seed_words.numel() < words_numel:
            self.seed_words = torch.empty(words_numel, dtype=torch.int32, device=self.vals[0].device)
        return self.seed_vals, self.seed_words

    def _graph_for(self, p: WgRunParams, stream=None, seeded=None):
        """seeded: (counts or None) -- the graph with the seed prologue."""
        q0 = WgRunParams.from_buffer_copy(p)
        q0.timer = None  # the graphs never carry a timer
        key = (ctypes.string_at(ctypes.addressof(q0), ctypes.sizeof(q0)), self.g.signature(), seeded)
        exe = self.graph_cache.get(key)
        if exe is None:
            q = WgRunParams()
            ctypes.pointer(q)[0] = p
            q.timer = None
            L = _lib.load()
            if seeded is not None:
                sv, sw = self._seed_buffers(max((self.g.n + 31) >> 5, 1))
                c = (ctypes.c_uint64 * 4)(*seeded[1]) if seeded[1] is not None else None
                exe = L.wg_run_loop_graph_create_seeded(ctypes.byref(self.g.struct()), ctypes.byref(self.bufs),
                                                        ctypes.byref(q), _ptr(sv), _ptr(sw), c,
                                                        _lib.stream_ptr(stream))
            else:
                exe = L.wg_run_loop_graph_create(ctypes.byref(self.g.struct()), ctypes.byref(self.bufs),
                                                 ctypes.byref(q), _lib.stream_ptr(stream))
            if not exe:
                raise _lib.WedgeError(_lib.WG_ECUDA, L.wg_last_error().decode())
            if len(self.graph_cache) >= 8:  # keep a few (the stream is ordered: no replay in flight reads it)
                old = self.graph_cache.pop(next(iter(self.graph_cache)))
                _torch().cuda.current_stream().synchronize()
                L.wg_run_graph_destroy(old)
            self.graph_cache[key] = exe
        return exe

    def __del__(self):
        try:
            L = _lib.load()
            for exe in self.graph_cache.values():
                L.wg_run_graph_destroy(exe)
        except Exception:
            pass

    def _parse(self, rows, it0, records, trace):
        """Append records of iterations it0.. until one did not run or converged.
        rows: per-iteration records as lists of Python ints (ndarray.tolist())."""
        for j, r in enumerate(rows):
            mode = r[0]
            if mode == 0:
                return True, None
            if r[10]:
                raise _lib.OverflowError32(_lib.WG_EOVERFLOW, "uint32 value overflow in device loop")
            wedge = mode == 2
            records.append(IterRecord(it0 + j, MODE_NAMES[mode], r[1], r[2], r[3], r[7] if wedge else 0,
                                      r[8] if wedge else 0, r[16], r[17]))
            if trace is not None:
                trace(self, it0 + j)
            if r[4] == 0:
                return True, it0 + j
        return False, None

    def drive_graph(self, p: WgRunParams, max_iterations: int, stream=None):
        """Whole loop as one conditional CUDA graph per launch (no host round
        trip between iterations); at most ring-2 iterations per launch."""
        torch = _torch()
        s = stream or torch.cuda.current_stream()
        L = _lib.load()
        sp = _lib.stream_ptr(stream)
        pending = getattr(self, "_pending", None)
        self._pending = None
        exe = self._graph_for(p, stream)
        records: list[IterRecord] = []
        it, converged, last = 1, False, 0
        ctrl_host = self.ctrl_host
        while it <= max_iterations and not converged:
            limit = min(max_iterations, it - 1 + self.ring - 2)
            if pending is not None:  # the run's seed is the first launch's prologue
                init_values, init_words, counts = pending
                pending = None
                exe0 = self._graph_for(p, stream, seeded=("all" if counts is not None else "words", counts))
                sv, sw = self._seed_buffers(init_words.numel())
                check(L.wg_run_loop_launch_seeded(exe0, ctypes.byref(self.bufs), limit, _ptr(init_values), _ptr(sv),
                                                  self.g.n * init_values.element_size(), _ptr(init_words), _ptr(sw),
                                                  min(init_words.numel(), sw.numel()) * 4, sp))
            else:
                check(L.wg_run_loop_launch(exe, ctypes.byref(self.bufs), limit, sp))
            # the control words and the head of the record ring in one small copy;
            # the whole ring only when the launch ran past the head (a launch runs
            # at most ring - 2 iterations, so its records are all in the ring)
            head = 4 + HEAD_RECORDS * REC_U64
            self.host_state[:head].copy_(self.state[:head], non_blocking=True)
            s.synchronize()
            hs = self._host_np
            done = min(int(hs[0]), limit)
            lo = it % self.ring
            if done >= it and (lo + (done - it) >= HEAD_RECORDS):
                self.host_state.copy_(self.state, non_blocking=True)
                s.synchronize()
            arr = hs[4:].reshape(self.ring, REC_U64)
            if done < it:
                rows = []
            elif lo + (done - it) < self.ring:
                rows = arr[lo: lo + done - it + 1].tolist()
            else:
                rows = [arr[(it + j) % self.ring].tolist() for j in range(done - it + 1)]
            conv, at = self._parse(rows, it, records, None)
            if records:
                last = records[-1].iteration
            if conv:
                converged = True
            it = done + 1
        return records, converged, last

    def drive(self, p: WgRunParams, max_iterations: int, trace=None, stream=None, graph=None):
        """Run to convergence or the cap; returns (records, converged, last_it).
        Default: one conditional-graph launch per ring of iterations; trace
        mode (frontier/value logs) steps one iteration at a time."""
        import os
        if graph is None:
            graph = os.environ.get("WG_GRAPH", "1") != "0"
        if trace is None and graph and p.timer is None:
            return self.drive_graph(p, max_iterations, stream)
        if getattr(self, "_pending", None) is not None:  # a deferred seed: run it now
            self._run_pending_seed(p, stream)
        records: list[IterRecord] = []
        converged = False
        it, batch, last = 1, 2, 0
        if trace is not None:  # frontier_members reads every produced list
            p.flags |= _lib.WG_RUN_KEEP_LISTS
        cap_batch = min(256, self.ring - 2)
        while it <= max_iterations and not converged:
            cnt = 1 if trace is not None else min(batch, max_iterations - it + 1)
            self.enqueue(p, it, cnt, stream)
            rows = self._read(it, cnt, stream)
            for j, r in enumerate(rows):
                mode = int(r[0])
                if mode == 0:
                    converged = True
                    break
                if int(r[10]):
                    raise _lib.OverflowError32(_lib.WG_EOVERFLOW, "uint32 value overflow in device loop")
                records.append(IterRecord(it + j, MODE_NAMES[mode], int(r[1]), int(r[2]), int(r[3]),
                                          int(r[7]) if mode == 2 else 0, int(r[8]) if mode == 2 else 0,
                                          int(r[16]), int(r[17])))
                last = it + j
                if trace is not None:
                    trace(self, last)
                if int(r[4]) == 0:
                    converged = True
                    break
            it += cnt
            batch = min(batch * 2, cap_batch)
        return records, converged, last

    def frontier_members(self, it: int) -> np.ndarray:
        """Sorted members of the frontier produced by iteration it (trace mode)."""
        arr = self.host_recs.numpy().view(np.uint64).reshape(self.ring, REC_U64)[it % self.ring]
        nz, z = int(arr[5]) >> 32, int(arr[6])
        lst = self.fvert[it & 1]
        parts = []
        if nz:
            parts.append(u32_to_np64(lst[:nz]))
        if z:
            parts.append(u32_to_np64(lst[self.g.n - z:]))
        return np.sort(np.concatenate(parts)) if parts else np.empty(0, np.int64)

    def values_after(self, it: int):
        return self.vals[it & 1]


def first_hit_ok(kern, init_values: np.ndarray, members: Optional[np.ndarray]) -> bool:
    """True when the run is level-synchronous (WG_RUN_FIRST_HIT): a filtered,
    unweighted kernel whose initially finite values are all equal and all in
    the initial frontier (members None = every vertex).  By induction every
    finite in-neighbour of a destination still unvisited at iteration k then
    holds the same value, so any one of them gives the minimum."""
    if not kern.filter_unvisited or kern.use_weight:
        return False
    v = np.asarray(init_values, dtype=np.int64)
    fin = v != UNREACHED
    if not fin.any():
        return True
    vals = v[fin]
    if np.any(vals != vals[0]):
        return False
    if members is None:
        return True
    mem = np.zeros(v.shape[0], dtype=bool)
    m = np.asarray(members, dtype=np.int64)
    mem[m[(m >= 0) & (m < v.shape[0])]] = True
    return bool(mem[fin].all())


def identity_values(init_values: np.ndarray) -> bool:
    """True when the initial values are the vertex ids (WG_RUN_IDENTITY_INIT)."""
    v = np.asarray(init_values, dtype=np.int64)
    return bool(np.array_equal(v, np.arange(v.shape[0], dtype=np.int64)))


def first_hit_level(init_values: np.ndarray) -> int:
    """The common finite initial value of a first_hit_ok run (0 if none)."""
    v = np.asarray(init_values, dtype=np.int64)
    fin = v[v != UNREACHED]
    return int(fin[0]) if fin.size else 0


def initial_words(n: int, members: np.ndarray):
    """Device uint32 bitmap of the initial frontier."""
    torch = _torch()
    words = np.zeros(max((n + 31) >> 5, 1), np.uint32)
    m = np.unique(np.asarray(members, dtype=np.int64))
    if m.size:
        if m.min() < 0 or m.max() >= n:
            raise IndexError("bit position out of range")
        np.bitwise_or.at(words, m >> 5, (np.uint32(1) << (m & 31).astype(np.uint32)))
    return torch.from_numpy(words.view(np.int32)).cuda()


def all_words(n: int):
    torch = _torch()
    words = torch.full((max((n + 31) >> 5, 1),), -1, dtype=torch.int32, device="cuda")
    words._wg_all = True
    return words


def encode_values(values: np.ndarray, val_type: int):
    """Reference int64 values -> device buffer of `val_type` (UNREACHED <-> 0xFFFFFFFF)."""
    torch = _torch()
    v = np.asarray(values, dtype=np.int64)
    if val_type == WG_VAL_I64:
        return torch.from_numpy(np.ascontiguousarray(v)).cuda()
    u = np.where(v == UNREACHED, U32_INF, v)
    if u.size and (u.min() < 0 or u.max() > U32_INF):
        raise ValueError("values do not fit the uint32 encoding")
    if u.size and np.any((u == U32_INF) & (v != UNREACHED)):
        raise ValueError("value 0xFFFFFFFF collides with the uint32 sentinel")
    return torch.from_numpy(u.astype(np.uint32).view(np.int32)).cuda()


@dataclass
class InitialValues:
    """Initial values on the device plus the facts the loop specialises on,
    derived by one device pass (wg_values_scan) instead of host scans."""
    i64: object            # device int64 copy (the WG_VAL_I64 seed)
    u32: object            # device uint32 encoding (valid when fits_u32)
    fits_u32: bool
    identity: bool         # init[v] == v (WG_RUN_IDENTITY_INIT)
    first_hit: bool        # level-synchronous run (WG_RUN_FIRST_HIT, see first_hit_ok)
    level_base: int

    def seed(self, val_type: int):
        return self.u32 if val_type == WG_VAL_U32 else self.i64


def prepare_initial_values(init: np.ndarray, kern, members: Optional[np.ndarray], stream=None) -> InitialValues:
    """Upload int64 initial values (engine.py:90-116) and scan them on the
    device: the same decisions as fits_u32 / identity_values / first_hit_ok /
    first_hit_level, one 32-byte read back."""
    torch = _torch()
    v = np.ascontiguousarray(init, dtype=np.int64)
    n = int(v.shape[0])
    d64 = torch.from_numpy(v).to("cuda", non_blocking=False)
    enc = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    stats = torch.empty(4, dtype=torch.int64, device="cuda")
    check(_lib.load().wg_values_scan(n, _ptr(d64), UNREACHED, _ptr(enc), _ptr(stats), _lib.stream_ptr(stream)))
    flags, cnt, lo, hi = (int(x) for x in stats.cpu().tolist())
    fits = not flags & _lib.WG_VALUES_NOT_U32
    identity = n > 0 and not flags & _lib.WG_VALUES_NOT_IDENTITY
    fh = bool(kern.filter_unvisited) and not kern.use_weight
    if fh and cnt:
        fh = lo == hi
        if fh and members is not None:
            m = np.asarray(members, dtype=np.int64)
            m = m[(m >= 0) & (m < n)]
            fh = int(np.count_nonzero(v[m] != UNREACHED)) == cnt  # members are unique
    return InitialValues(d64, enc[:n], fits, bool(identity), bool(fh), lo if (fh and cnt) else 0)


def fits_u32(values: np.ndarray, kern, g: DeviceGraph) -> bool:
    """Conservative check that the uint32 encoding cannot lose information
    before the device overflow flag would catch it."""
    v = np.asarray(values, dtype=np.int64)
    fin = v[v != UNREACHED]
    return not fin.size or (fin.min() >= 0 and fin.max() < U32_INF)


# ---------------------------------------------------------------------------
# PageRank (K8)
# ---------------------------------------------------------------------------
class PageRankLayout:
    """Hot-source layout of one graph for PageRank (wg_pagerank_hot_layout):
    contribution slots in descending out-degree order, a copy of the lanes
    holding slots, the slot -> vertex map and the slots' out-degrees."""

    def __init__(self, g: DeviceGraph, stream=None):
        torch = _torch()
        L = _lib.load()
        n = max(g.n, 1)
        lanes = g.nvec * g.width
        self.vsrc_hot = torch.empty(lanes + 16 * g.width, dtype=torch.int32, device="cuda")  # slack like vsrc
        self.vsrc_hot[lanes:].fill_(-1)
        self.order = torch.empty(n, dtype=torch.int32, device="cuda")
        self.od_hot = torch.empty(n, dtype=torch.int32, device="cuda")
        ws = torch.empty(int(L.wg_pagerank_hot_ws_bytes(ctypes.byref(g.struct()))), dtype=torch.uint8, device="cuda")
        nsrc = ctypes.c_uint64(0)
        check(L.wg_pagerank_hot_layout(ctypes.byref(g.struct()), _ptr(self.vsrc_hot), _ptr(self.order),
                                       _ptr(self.od_hot), ctypes.byref(nsrc), _ptr(ws), ws.numel(),
                                       _lib.stream_ptr(stream)))
        self.nsrc = int(nsrc.value)


def pagerank(g: DeviceGraph, iterations: int = 20, damping: float = 0.85, stream=None, bufs=None,
             hot: Optional[bool] = None):
    """hot (default on; WG_PR_HOT=0 turns it off): gather contributions through
    the hot-source layout, built on first use and kept with the graph."""
    torch = _torch()
    n = max(g.n, 1)
    if bufs is None:
        bufs = (torch.empty(n, dtype=torch.float32, device="cuda"),
                torch.empty(n, dtype=torch.float32, device="cuda"),
                torch.empty(n, dtype=torch.float32, device="cuda"),
                torch.zeros(4, dtype=torch.float64, device="cuda"))
    rank, acc, contrib, scal = bufs[:4]
    L = _lib.load()
    need = int(L.wg_pagerank_ws_bytes(ctypes.byref(g.struct())))
    ws = getattr(g, "_pr_ws", None)
    if ws is None or ws.numel() < need:
        ws = g._pr_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    if hot is None:
        hot = os.environ.get("WG_PR_HOT", "1") != "0"
    if hot and g.nvec:
        lay = getattr(g, "_pr_hot", None)
        if lay is None:
            lay = g._pr_hot = PageRankLayout(g, stream)
        check(L.wg_pagerank_hot(ctypes.byref(g.struct()), _ptr(lay.vsrc_hot), _ptr(lay.order), _ptr(lay.od_hot),
                                lay.nsrc, int(iterations), float(damping), _ptr(rank), _ptr(acc), _ptr(contrib),
                                _ptr(scal), _ptr(ws), ws.numel(), _lib.stream_ptr(stream)))
        return rank
    check(L.wg_pagerank(ctypes.byref(g.struct()), int(iterations), float(damping), _ptr(rank), _ptr(acc),
                        _ptr(contrib), _ptr(scal), _ptr(ws), ws.numel(), _lib.stream_ptr(stream)))
    return rank


# ---------------------------------------------------------------------------
# Generators (graph_io.py:87-221, K9)
# ---------------------------------------------------------------------------
RMAT_PROBS = (0.57, 0.19, 0.19, 0.05)


def rmat_edges(scale: int, edge_factor: int, seed: int = 1, probs=RMAT_PROBS, stream=None):
    """Bit-identical to graph_io._generate_rmat: numpy PCG64(seed) stream,
    draws (m, scale) row-major, quadrant thresholds a, a+b, a+b+c."""
    torch = _torch()
    n = 1 << scale
    m = edge_factor * n
    st = np.random.PCG64(seed).state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    a, b, c, _ = probs
    th = (ctypes.c_double * 3)(a, a + b, a + b + c)
    src = torch.empty(m, dtype=torch.int32, device="cuda")
    dst = torch.empty(m, dtype=torch.int32, device="cuda")
    M = (1 << 64) - 1
    check(_lib.load().wg_rmat_edges(scale, m, state >> 64, state & M, inc >> 64, inc & M, th,
                                    _ptr(src), _ptr(dst), _lib.stream_ptr(stream)))
    return n, src, dst


def rmat_edges_rows(scale: int, row_lo: int, row_hi: int, seed: int = 1, probs=RMAT_PROBS, stream=None):
    """Rows [row_lo, row_hi) of rmat_edges' stream: the PCG64 state jumped
    ahead by row_lo * scale draws (PCG64.advance), so shards of the edge list
    are generated independently and concatenate to the full one."""
    torch = _torch()
    bg = np.random.PCG64(seed)
    bg.advance(int(row_lo) * int(scale))
    st = bg.state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    a, b, c, _ = probs
    th = (ctypes.c_double * 3)(a, a + b, a + b + c)
    m = int(row_hi) - int(row_lo)
    src = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    dst = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    M = (1 << 64) - 1
    if m:
        check(_lib.load().wg_rmat_edges(scale, m, state >> 64, state & M, inc >> 64, inc & M, th,
                                        _ptr(src), _ptr(dst), _lib.stream_ptr(stream)))
    return src[:m], dst[:m]


def canonical_edges(src, dst, drop_loops: bool, symmetrize: bool, stream=None):
    """Sorted (src, dst)-unique edge list; optional self-loop removal and
    symmetrisation (graph_io.py:87-112 with dedup)."""
    torch = _torch()
    L = _lib.load()
    m = int(src.numel())
    cap = 2 * m if symmetrize else m
    s = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
    d = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
    s[:m].copy_(src)
    d[:m].copy_(dst)
    scratch = torch.empty(int(L.wg_canonical_scratch_bytes(m)), dtype=torch.uint8, device="cuda")
    out = ctypes.c_uint64(0)
    check(L.wg_canonical_edges(m, _ptr(s), _ptr(d), int(drop_loops), int(symmetrize), _ptr(scratch),
                               scratch.numel(), ctypes.byref(out), _lib.stream_ptr(stream)))
    k = int(out.value)
    return s[:k].clone(), d[:k].clone()


def weights_hash(src, dst, max_weight: int, stream=None):
    torch = _torch()
    m = int(src.numel())
    w = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    check(_lib.load().wg_weights_hash(m, _ptr(src), _ptr(dst), int(max_weight), _ptr(w),
                                      _lib.stream_ptr(stream)))
    return w[:m]


def grid_edges(rows: int, cols: int, seed: int, keep: float = 0.9, max_weight: int = 1000, stream=None):
    """4-neighbour grid, each undirected edge kept with probability `keep`,
    symmetric weight uniform in [1, max_weight] (BASELINE config 3; the
    reference has no such generator, so the stream is defined here and
    restated in oracle.grid_edges)."""
    torch = _torch()
    und = rows * (cols - 1) + (rows - 1) * cols
    cap = max(2 * und, 1)
    s = torch.empty(cap, dtype=torch.int32, device="cuda")
    d = torch.empty(cap, dtype=torch.int32, device="cuda")
    w = torch.empty(cap, dtype=torch.int32, device="cuda")
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = ctypes.c_uint64(0)
    check(_lib.load().wg_grid_edges(rows, cols, int(seed), int(round(keep * 1_000_000)), int(max_weight),
                                    _ptr(s), _ptr(d), _ptr(w), _ptr(ctr), ctypes.byref(out),
                                    _lib.stream_ptr(stream)))
    k = int(out.value)
    return rows * cols, s[:k], d[:k], w[:k]
