"""The B200 kernel backend behind the reference's plugin seam.

The reference resolves backends with ``get_backend(name_or_obj)`` and passes
backend objects straight through (kernels.py:137-151); every hot-path entry
point takes ``backend=`` (frontier.py:180, engine.py:257, 289, 336).
``B200Backend`` implements that protocol exactly -- ``pull_full``,
``pull_wedge``, ``transform`` with the reference's signatures, int64 numpy
values and uint64 bitmap words (kernels.py:55-125) -- so an instance can be
handed to the UNMODIFIED reference engine.  Each call
runs the sm_100a kernels through the C ABI (wg_pull_full / wg_pull_wedge /
wg_transform) on device copies of the arguments and writes the results back
in place: bit-identical to the reference, slow by design (PCIe per call).

The whole-loop fast path is ``run_until_convergence`` on this object: the
engine delegates to it when present (engine.py of this package), keeping the
loop resident on the device.

There is no CPU fallback: without the CUDA library or a GPU every method
raises.
"""

from __future__ import annotations

import os
import weakref

import numpy as np

from . import device as _dev


class _UploadCache:
    """Device copies of reference-layout host structures, keyed by object
    identity and dropped when the host object dies (objects without weak
    references -- the reference's __slots__ classes -- are held strongly,
    so the cache keeps at most `capacity` entries, oldest evicted first)."""

    def __init__(self, capacity: int = 16):
        self._items = {}
        self.capacity = capacity

    def clear(self):
        self._items.clear()

    def get(self, key_objs, make):
        key = tuple(id(o) for o in key_objs)
        hit = self._items.get(key)
        if hit is not None and all(r() is o for r, o in zip(hit[0], key_objs)):
            return hit[1]
        while len(self._items) >= self.capacity:
            self._items.pop(next(iter(self._items)))
        val = make()
        refs = []
        for o in key_objs:
            try:
                refs.append(weakref.ref(o, lambda _r, k=key: self._items.pop(k, None)))
            except TypeError:
                refs.append(lambda o=o: o)
        self._items[key] = (refs, val)
        return val


class B200Backend:
    name = "b200"
    # run_until_convergence: time each iteration's kernels with CUDA events
    # (one iteration per launch) instead of one whole-loop graph launch
    per_iteration_timing = False

    def __init__(self, reupload: bool = False):
        """reupload: re-read the caller's host arrays on every call (into the
        cached device buffers) instead of trusting an upload made earlier for
        the same objects -- for callers that mutate arrays in place, and the
        end-to-end measurement of the plugin call (bench.py e2e)."""
        self._cache = _UploadCache()
        self.reupload = bool(reupload)

    # -- device graph resolution -------------------------------------------
    def device_graph(self, topology, index=None, degrees=None) -> _dev.DeviceGraph:
        g = getattr(topology, "device", None)
        if isinstance(g, _dev.DeviceGraph):
            return g
        # a reference-layout topology: upload its lanes; the index / degrees
        # are only needed by the loop and the transform
        def make():
            if index is not None:
                g = _dev.DeviceGraph.from_reference(topology, index, degrees)
                g._fresh = True  # uploaded by this very call
                return g
            return _dev.DeviceGraph.from_reference(topology, _EmptyIndex(topology.vertex_count),
                                                   np.zeros(topology.vertex_count, np.int64))
        keys = [topology] + ([index] if index is not None else [])
        g = self._cache.get(keys, make)
        if self.reupload and getattr(g, "_fresh", False) is False and index is not None:
            g = _dev.DeviceGraph.from_reference(topology, index, degrees, into=g)
        g._fresh = False
        return g

    def _index_graph(self, offsets, positions, vertex_count, groups, shift) -> _dev.DeviceGraph:
        g = getattr(offsets, "device", None)
        if isinstance(g, _dev.DeviceGraph):
            return g

        def make():
            import torch
            off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).cuda()
            pos = np.asarray(positions, dtype=np.int64)
            dpos = _dev.to_dev_u32(pos if pos.size else np.zeros(1, np.int64))
            deg = torch.zeros(max(vertex_count, 1), dtype=torch.int32, device="cuda")
            dummy = torch.zeros(1, dtype=torch.int32, device="cuda")
            return off, dpos, int(pos.size), deg, dummy

        off, dpos, entries, deg, dummy = self._cache.get([offsets, positions], make)
        # the transform reads only the index; the vector count sizes the group space
        return _dev.DeviceGraph(vertex_count, 1, 0, groups << shift, entries, dummy, dummy, None, off,
                                dpos, deg)

    # -- reference backend protocol (kernels.py:55-125) ----------------------
    def pull_full(self, topology, prev, nxt, out_words, kern, sentinel, workers=1):
        g = self.device_graph(topology)
        return _dev.pull_call(g, prev, nxt, out_words, kern, sentinel)

    def pull_wedge(self, topology, wedge_words, shift, group_count, prev, nxt, out_words, kern,
                   sentinel, workers=1):
        g = self.device_graph(topology)
        if g.nvec == 0:
            return 0
        return _dev.pull_call(g, prev, nxt, out_words, kern, sentinel, wedge_words=wedge_words,
                              shift=int(shift))

    def transform(self, frontier_words, vertex_count, offsets, positions, shift, wedge_words,
                  slice_size=4096, workers=1):
        groups = int(np.asarray(wedge_words).size) * 64
        g = self._index_graph(offsets, positions, int(vertex_count), groups, int(shift))
        if g.entries == 0 or int(vertex_count) == 0:
            return 0
        return _dev.transform_call(g, frontier_words, int(shift), wedge_words)

    # -- whole-loop fast path --------------------------------------------------
    def run_until_convergence(self, topology, index, program, degrees, config, frontier_log=None,
                              value_log=None):
        from .engine import device_run
        return device_run(self, topology, index, program, degrees, config, frontier_log, value_log)


class _EmptyIndex:
    def __init__(self, n):
        self.offsets = np.zeros(n + 1, np.int64)
        self.positions = np.empty(0, np.int64)


_BACKENDS = {"b200": B200Backend()}


def available_backends() -> tuple[str, ...]:
    return tuple(sorted(_BACKENDS))


def get_backend(name=None):
    """kernels.py:137-151: None/"auto" -> the default; objects pass through."""
    if name is None or name == "auto":
        return DEFAULT
    if not isinstance(name, str):
        return name
    try:
        return _BACKENDS[name]
    except KeyError:
        raise RuntimeError(
            f"backend {name!r} is not available (have: {', '.join(available_backends())})") from None


def _select_default():
    forced = os.environ.get("WEDGE_BACKEND", "auto")
    if forced in ("auto", "b200"):
        return _BACKENDS["b200"]
    raise RuntimeError(f"WEDGE_BACKEND={forced!r} is not available in paper_1903_07754_b200")


DEFAULT = _select_default()
