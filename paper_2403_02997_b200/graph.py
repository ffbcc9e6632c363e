"""Graph types and the device-side CSR build (drop-in for tricount.graph).

Mirrors the reference's ``EdgeList``/``Graph``/``normalize``
(graph.py:37-125, 177-194): same fields, dtypes (int64 offsets, int32 ids,
lexicographic u<v edge arrays), frozen arrays and ValueError behaviour.  The
difference is where the work happens: ``normalize`` uploads the pairs and
builds the CSR on the GPU (``tcb_csr_build``: one radix sort of 64-bit
(src, dst) keys + ordered compactions), and the resulting ``Graph`` keeps its
device copy (``DeviceGraph``) so the counting entry points do not re-upload.
"""
from __future__ import annotations

import io
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = [
    "EdgeList",
    "Graph",
    "DeviceGraph",
    "ParseError",
    "parse_edge_list",
    "load_edge_list",
    "normalize",
    "normalize_device",
    "to_edge_list",
    "device_graph",
]


class ParseError(ValueError):
    """Raised for malformed edge-list input (graph.py:33-34)."""


@dataclass
class EdgeList:
    """Raw edge pairs with dense 0-based ids (graph.py:37-54); may hold
    duplicates and self-loops, which :func:`normalize` removes."""

    n: int
    edges: np.ndarray  # (k, 2) int64
    original_ids: np.ndarray | None = None

    def __post_init__(self):
        self.edges = np.asarray(self.edges, dtype=np.int64).reshape(-1, 2)
        if self.edges.size and (self.edges.min() < 0 or self.edges.max() >= self.n):
            raise ValueError("edge endpoint out of range [0, n)")


def _freeze(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


@dataclass(frozen=True)
class Graph:
    """Immutable undirected CSR graph (graph.py:57-92).

    ``neighbors[row_offsets[v]:row_offsets[v+1]]`` is v's strictly increasing
    neighbour list; ``edge_u``/``edge_v`` list each edge once with u<v,
    lexicographically.  ``_device`` caches the GPU copy.
    """

    n: int
    m: int
    row_offsets: np.ndarray
    neighbors: np.ndarray
    edge_u: np.ndarray = field(repr=False)
    edge_v: np.ndarray = field(repr=False)
    _device: object = field(default=None, repr=False, compare=False)

    def degree(self, v: int) -> int:
        return int(self.row_offsets[v + 1] - self.row_offsets[v])

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    @property
    def max_degree(self) -> int:
        return int(self.degrees.max()) if self.n else 0

    def adjacency(self, v: int) -> np.ndarray:
        return self.neighbors[self.row_offsets[v]:self.row_offsets[v + 1]]

    def has_edge(self, u: int, v: int) -> bool:
        nb = self.adjacency(u)
        i = np.searchsorted(nb, v)
        return bool(i < len(nb) and nb[i] == v)


@dataclass
class DeviceGraph:
    """The same CSR resident in HBM (torch tensors on one CUDA device):
    int64 row offsets, int32 neighbours, and ``src`` — the int32 row id of
    every entry (COO rows).  ``src`` has the footprint of the reference's
    edge_u/edge_v pair, whose entries are exactly the src < neighbour ones in
    order; those arrays are derived on demand (``edge_arrays``)."""

    n: int
    m: int
    row_offsets: "object"   # torch.int64 [n+1]
    neighbors: "object"     # torch.int32 [2m]
    src: "object"           # torch.int32 [2m]

    @property
    def device(self):
        return self.row_offsets.device

    def edge_arrays(self):
        """Graph.edge_u/edge_v (u<v, lexicographic) as int32 device tensors."""
        import torch
        ctx = _lib.context(self.device.index)
        eu = torch.empty(max(self.m, 1), dtype=torch.int32, device=self.device)
        ev = torch.empty(max(self.m, 1), dtype=torch.int32, device=self.device)
        ctx.check(ctx.lib.tcb_csr_edges(ctx.h, _lib.ptr(self.row_offsets),
                                        _lib.ptr(self.neighbors), self.n, self.m,
                                        _lib.ptr(eu), _lib.ptr(ev)))
        return eu[: self.m], ev[: self.m]

    def to_host(self) -> Graph:
        eu, ev = self.edge_arrays()
        g = Graph(
            n=self.n,
            m=self.m,
            row_offsets=_freeze(self.row_offsets.cpu().numpy()),
            neighbors=_freeze(self.neighbors.cpu().numpy()),
            edge_u=_freeze(eu.cpu().numpy()),
            edge_v=_freeze(ev.cpu().numpy()),
        )
        object.__setattr__(g, "_device", self)
        return g

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size()
                   for t in (self.row_offsets, self.neighbors, self.src))


def _check_vertex_count(n: int):
    if n < 0:
        raise ValueError("n must be >= 0")
    if n >= 2**31:
        raise ValueError("this build stores vertex ids as int32 (n < 2^31)")


def normalize_device(n: int, pairs) -> DeviceGraph:
    """graph.py:177-194 on the GPU: pairs (torch int64 [k,2] on a CUDA
    device, or anything numpy accepts) -> DeviceGraph."""
    import torch
    _check_vertex_count(n)
    if not isinstance(pairs, torch.Tensor) or not pairs.is_cuda:
        ctx = _lib.context()  # raises without a CUDA device: no CPU fallback
        arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
        pairs = torch.from_numpy(arr).to(torch.device("cuda", ctx.device))
    pairs = pairs.reshape(-1, 2).contiguous()
    if pairs.dtype != torch.int64:
        pairs = pairs.to(torch.int64)
    dev = pairs.device
    ctx = _lib.context(dev.index)
    k = pairs.shape[0]
    row = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nb = torch.empty(max(2 * k, 1), dtype=torch.int32, device=dev)
    src = torch.empty(max(2 * k, 1), dtype=torch.int32, device=dev)
    m = _lib.ctypes.c_int64(0)
    ctx.check(ctx.lib.tcb_csr_build(ctx.h, _lib.ptr(pairs), k, n, _lib.ptr(row),
                                    _lib.ptr(nb), _lib.ptr(src), None, None,
                                    _lib.ctypes.byref(m)))
    m = int(m.value)
    return DeviceGraph(n=n, m=m, row_offsets=row, neighbors=nb[: 2 * m], src=src[: 2 * m])


def degree_order_device(dg: DeviceGraph) -> DeviceGraph:
    """graph.py:203-213 on the GPU (tcb_degree_order): relabel by
    non-increasing degree, ties by ascending old id."""
    import torch
    ctx = _lib.context(dg.device.index)
    row = torch.empty(dg.n + 1, dtype=torch.int64, device=dg.device)
    nb = torch.empty(max(2 * dg.m, 1), dtype=torch.int32, device=dg.device)
    src = torch.empty(max(2 * dg.m, 1), dtype=torch.int32, device=dg.device)
    ctx.check(ctx.lib.tcb_degree_order(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                       _lib.ptr(dg.src), dg.n, dg.m, _lib.ptr(row),
                                       _lib.ptr(nb), _lib.ptr(src)))
    return DeviceGraph(n=dg.n, m=dg.m, row_offsets=row, neighbors=nb[: 2 * dg.m],
                       src=src[: 2 * dg.m])


def degree_order(g: Graph) -> Graph:
    """Relabel vertices by non-increasing degree, ties by ascending old id
    (graph.py:203-213).  The result is isomorphic to ``g``; vertex 0 has
    maximal degree."""
    return degree_order_device(device_graph(g)).to_host()


def normalize(el: EdgeList) -> Graph:
    """Canonicalize an EdgeList into a Graph (graph.py:177-194): self-loops
    dropped, duplicates collapsed, both directions stored, rows sorted."""
    return normalize_device(el.n, el.edges).to_host()


def device_graph(g, device=None) -> DeviceGraph:
    """The DeviceGraph behind a Graph (uploads the CSR once, expands the row
    ids on the device, caches the result on the Graph)."""
    import torch
    if isinstance(g, DeviceGraph):
        return g
    # any object with the reference Graph's fields works (the reference's own
    # tricount.Graph included); the device copy is cached when it can be
    dg = getattr(g, "_device", None)
    if dg is not None and (device is None or dg.device == torch.device(device)):
        return dg
    ctx = _lib.context(torch.device(device).index if device is not None else None)
    dev = torch.device("cuda", ctx.device)
    _check_vertex_count(g.n)
    # the frozen (pageable) numpy arrays go up through the library's pinned
    # staging ring (tcb_copy_to_device): host copies overlap the DMA
    row_h = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
    nb_h = np.ascontiguousarray(g.neighbors, dtype=np.int32)
    row = torch.empty(g.n + 1, dtype=torch.int64, device=dev)
    nb = torch.empty(max(len(nb_h), 1), dtype=torch.int32, device=dev)[: len(nb_h)]
    ctx.check(ctx.lib.tcb_copy_to_device(ctx.h, _lib.ptr(row), row_h.ctypes.data, row_h.nbytes))
    if nb_h.nbytes:
        ctx.check(ctx.lib.tcb_copy_to_device(ctx.h, _lib.ptr(nb), nb_h.ctypes.data, nb_h.nbytes))
    src = torch.empty(max(2 * g.m, 1), dtype=torch.int32, device=dev)
    ctx.check(ctx.lib.tcb_csr_rows(ctx.h, _lib.ptr(row), g.n, _lib.ptr(src)))
    dg = DeviceGraph(n=g.n, m=g.m, row_offsets=row, neighbors=nb, src=src[: 2 * g.m])
    try:
        object.__setattr__(g, "_device", dg)
    except (AttributeError, TypeError):  # __slots__ without the field
        pass
    return dg


def to_edge_list(g: Graph) -> EdgeList:
    """One (u, v) pair per undirected edge, u < v (graph.py:197-200)."""
    edges = np.stack([g.edge_u, g.edge_v], axis=1).astype(np.int64)
    return EdgeList(n=g.n, edges=edges)


# ---------------------------------------------------------------------------
# edge-list text input (graph.py:128-174) — host-side ingest, off the timed path


def _lines(data):
    if isinstance(data, (bytes, bytearray)):
        data = bytes(data).decode("ascii", errors="replace")
    src = io.StringIO(data) if isinstance(data, str) else data
    for no, raw in enumerate(src, start=1):
        yield no, (raw.decode("ascii", errors="replace") if isinstance(raw, bytes) else raw)


def _token_int(tok: str, no: int) -> int:
    try:
        x = int(tok)
    except ValueError:
        raise ParseError(f"line {no}: non-integer token") from None
    if x < 0:
        raise ParseError(f"line {no}: negative vertex id")
    return x


def parse_edge_list(data) -> EdgeList:
    """Text pairs -> EdgeList with the reference's rules (graph.py:128-169):
    '#'/'%' comment lines and blank lines skipped, exactly two non-negative
    integers per line, external ids relabeled 0.. in first-appearance order
    (kept in ``original_ids``), ParseError naming the offending line."""
    dense: dict[int, int] = {}
    flat: list[int] = []
    for no, line in _lines(data):
        body = line.strip()
        if not body or body[0] in "#%":
            continue
        tok = body.split()
        if len(tok) != 2:
            raise ParseError(f"line {no}: expected 2 tokens, got {len(tok)}")
        a, b = _token_int(tok[0], no), _token_int(tok[1], no)
        flat.append(dense.setdefault(a, len(dense)))
        flat.append(dense.setdefault(b, len(dense)))
    edges = np.asarray(flat, dtype=np.int64).reshape(-1, 2)
    original = np.asarray(list(dense), dtype=np.int64)
    return EdgeList(n=len(dense), edges=edges, original_ids=original)


def load_edge_list(path) -> EdgeList:
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        return parse_edge_list(fh)
