"""Seeded input generation on the device (reference graph_io.py:115-221).

``generate(GenSpec("rmat", ...))`` reproduces the reference's RMAT stream
bit for bit (numpy PCG64 stepped on the GPU with jump-ahead, graph_io.py:
188-202); ``symmetrize(..., dedup=True)`` and directed de-duplication are a
device radix sort + unique; ``synthesize_weights`` is the reference's
multiplicative hash (graph_io.py:205-221).  ``grid_edges`` builds BASELINE
config 3's road-like grid, for which the reference has no generator.
Edge-list ingest: the reference's text format (parse_edge_list /
serialize_edge_list, graph_io.py:34-84) for the CLI, and a binary ``.npz``
form (src, dst[, weight], vertex_count) that loads without parsing
(SURVEY §8(f) row 4).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device as dv
from .graph import EdgeList

RMAT_DEFAULT_PROBS = dv.RMAT_PROBS
HASH_MULTIPLIER = 0x9E3779B97F4A7C15


@dataclass(frozen=True)
class GenSpec:
    """path(n), grid(rows, cols) or rmat(scale, edge_factor) (graph_io.py:115-157)."""

    kind: str
    n: int = 0
    rows: int = 0
    cols: int = 0
    scale: int = 0
    edge_factor: int = 0
    probs: tuple = RMAT_DEFAULT_PROBS
    seed: int = 1

    def __post_init__(self):
        if self.kind == "path":
            ok = self.n >= 1
        elif self.kind == "grid":
            ok = self.rows >= 1 and self.cols >= 1
        elif self.kind == "rmat":
            ok = self.scale >= 1 and self.edge_factor >= 1
            if ok and (any(p < 0 for p in self.probs) or abs(sum(self.probs) - 1.0) > 1e-9):
                raise ValueError("rmat probabilities must be non-negative and sum to 1")
        else:
            raise ValueError(f"unknown generator kind {self.kind!r}")
        if not ok:
            raise ValueError(f"bad {self.kind} generator parameters")

    @classmethod
    def parse(cls, text: str, seed: int = 1) -> "GenSpec":
        kind, *args = text.split(":")
        try:
            if kind == "path" and len(args) == 1:
                return cls("path", n=int(args[0]), seed=seed)
            if kind == "grid" and len(args) == 2:
                return cls("grid", rows=int(args[0]), cols=int(args[1]), seed=seed)
            if kind == "rmat" and len(args) in (2, 6):
                probs = tuple(float(p) for p in args[2:]) if len(args) == 6 else RMAT_DEFAULT_PROBS
                return cls("rmat", scale=int(args[0]), edge_factor=int(args[1]), probs=probs, seed=seed)
        except ValueError as exc:
            raise ValueError(f"bad generator spec {text!r}: {exc}") from None
        raise ValueError(f"malformed generator spec {text!r}")


def generate(spec: GenSpec) -> EdgeList:
    if spec.kind == "path":
        s = np.arange(spec.n - 1, dtype=np.int64)
        return EdgeList(spec.n, s, s + 1)
    if spec.kind == "grid":
        r, c = spec.rows, spec.cols
        v = np.arange(r * c, dtype=np.int64).reshape(r, c)
        # per vertex in row-major order: right link then down link, each both ways
        right = np.stack([v[:, :-1], v[:, 1:]], -1).reshape(r, c - 1, 2)
        down = np.stack([v[:-1, :], v[1:, :]], -1).reshape(r - 1, c, 2)
        pairs = []
        for i in range(r):
            for j in range(c):
                if j + 1 < c:
                    pairs.append(right[i, j])
                if i + 1 < r:
                    pairs.append(down[i, j])
        if not pairs:
            return EdgeList(r * c, [], [])
        p = np.array(pairs, dtype=np.int64)
        src = np.stack([p[:, 0], p[:, 1]], 1).ravel()
        dst = np.stack([p[:, 1], p[:, 0]], 1).ravel()
        return EdgeList(r * c, src, dst)
    n, s, d = dv.rmat_edges(spec.scale, spec.edge_factor, spec.seed, spec.probs)
    return EdgeList.from_device(n, s, d)


def symmetrize(edges: EdgeList, dedup: bool = False) -> EdgeList:
    """graph_io.py:87-112: add reverses (self-loops once); with dedup the
    result is canonical (sorted by (src, dst), unique, minimum weight)."""
    if edges.is_weighted() or not dedup:
        # weighted / non-dedup forms are host-side input preparation
        loops = edges.src == edges.dst
        src = np.concatenate([edges.src, edges.dst[~loops]])
        dst = np.concatenate([edges.dst, edges.src[~loops]])
        w = None if edges.weight is None else np.concatenate([edges.weight, edges.weight[~loops]])
        if not dedup:
            return EdgeList(edges.vertex_count, src, dst, w)
        order = np.lexsort((w, dst, src))
        src, dst, w = src[order], dst[order], w[order]
        keep = np.ones(len(src), bool)
        keep[1:] = (src[1:] != src[:-1]) | (dst[1:] != dst[:-1])
        return EdgeList(edges.vertex_count, src[keep], dst[keep], w[keep])
    s, d, _ = edges.device_arrays()
    s2, d2 = dv.canonical_edges(s, d, drop_loops=False, symmetrize=True)
    return EdgeList.from_device(edges.vertex_count, s2, d2)


def drop_self_loops_dedup(edges: EdgeList, symmetric: bool) -> EdgeList:
    """BASELINE preparation: self-loops removed, duplicates
    removed, optionally symmetrised; canonical (src, dst) order."""
    s, d, _ = edges.device_arrays()
    s2, d2 = dv.canonical_edges(s, d, drop_loops=True, symmetrize=symmetric)
    return EdgeList.from_device(edges.vertex_count, s2, d2)


def synthesize_weights(edges: EdgeList, max_weight: int) -> EdgeList:
    """graph_io.py:205-221: w = 1 + ((((s*K) ^ d) * K) >> 48) % max_weight."""
    if edges.is_weighted():
        raise ValueError("edge list already carries weights")
    if max_weight < 1:
        raise ValueError("max_weight must be >= 1")
    s, d, _ = edges.device_arrays()
    w = dv.weights_hash(s, d, max_weight)
    return EdgeList.from_device(edges.vertex_count, s, d, w)


def grid_graph(rows: int, cols: int, seed: int, keep: float = 0.9, max_weight: int = 1000) -> EdgeList:
    n, s, d, w = dv.grid_edges(rows, cols, seed, keep, max_weight)
    return EdgeList.from_device(n, s, d, w)


# ---------------------------------------------------------------------------
# Ingest (graph_io.py:34-84) and the binary form
# ---------------------------------------------------------------------------
class ParseError(ValueError):
    """Malformed edge-list input, with the offending line number in the message."""


def parse_edge_list(text: str) -> EdgeList:
    """graph_io.py:34-73: ``src dst [weight]`` per line; ``#``/``%`` comments;
    the first ``# vertices N`` header sets the vertex count (else 1 + max id);
    mixed weighted/unweighted lines, negative ids, non-integer tokens and
    weights < 1 are rejected with the line number."""
    srcs, dsts, wts = [], [], []
    weighted = None
    header_n = None
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line:
            continue
        if line[0] in "#%":
            tok = line[1:].split()
            if header_n is None and len(tok) == 2 and tok[0] == "vertices" and tok[1].isdigit():
                header_n = int(tok[1])
            continue
        tok = line.split()
        if len(tok) not in (2, 3):
            raise ParseError(f"line {lineno}: expected 2 or 3 fields, got {len(tok)}")
        try:
            f = [int(t) for t in tok]
        except ValueError:
            raise ParseError(f"line {lineno}: non-integer token") from None
        if f[0] < 0 or f[1] < 0:
            raise ParseError(f"line {lineno}: negative vertex id")
        has_w = len(f) == 3
        if weighted is None:
            weighted = has_w
        elif weighted != has_w:
            raise ParseError(f"line {lineno}: mixed weighted and unweighted edges")
        if has_w and f[2] < 1:
            raise ParseError(f"line {lineno}: weight must be positive")
        srcs.append(f[0])
        dsts.append(f[1])
        if has_w:
            wts.append(f[2])
    implied = 1 + max(max(srcs, default=-1), max(dsts, default=-1))
    n = header_n if header_n is not None else implied
    return EdgeList(n, srcs, dsts, wts if weighted else None)


def serialize_edge_list(edges: EdgeList) -> str:
    """graph_io.py:76-84: inverse of parse_edge_list; a vertex header only
    when the count is not implied by the ids."""
    src, dst = np.asarray(edges.src, np.int64), np.asarray(edges.dst, np.int64)
    lines = []
    implied = 1 + int(max(src.max(initial=-1), dst.max(initial=-1)))
    if edges.vertex_count != implied:
        lines.append(f"# vertices {edges.vertex_count}")
    cols = [src, dst] + ([np.asarray(edges.weight, np.int64)] if edges.weight is not None else [])
    body = np.stack(cols, 1) if src.size else np.empty((0, len(cols)), np.int64)
    lines.extend(" ".join(map(str, row)) for row in body.tolist())
    return "".join(line + "\n" for line in lines)


def save_edge_list_binary(edges: EdgeList, path) -> None:
    """Binary edge list (.npz: vertex_count, src, dst[, weight] as uint32)."""
    arrs = {"vertex_count": np.array([edges.vertex_count], np.int64),
            "src": np.asarray(edges.src, np.int64).astype(np.uint32),
            "dst": np.asarray(edges.dst, np.int64).astype(np.uint32)}
    if edges.weight is not None:
        arrs["weight"] = np.asarray(edges.weight, np.int64).astype(np.uint32)
    with open(path, "wb") as fh:
        np.savez(fh, **arrs)


def load_edge_list(path) -> EdgeList:
    """Edge list from a file: ``.npz`` binary form (no parsing), else the
    reference text format."""
    path = str(path)
    if path.endswith(".npz"):
        with np.load(path) as z:
            n = int(z["vertex_count"][0])
            w = z["weight"].astype(np.int64) if "weight" in z.files else None
            return EdgeList(n, z["src"].astype(np.int64), z["dst"].astype(np.int64), w)
    with open(path, "r", encoding="utf-8") as fh:
        return parse_edge_list(fh.read())
