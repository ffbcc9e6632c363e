"""CETC-Seq entry point and registry (drop-in for tricount.sequential's
cover-edge path).

Every CETC id of the reference's ``cetc-family`` group (bench.py:42-43) keeps
the reference contract (sequential.py:164-238): a normalized read-only Graph
in, the exact triangle count out as ``int``, with the BFS preprocessing
charged to the call.

* ``CETC-Seq``: the fused GPU path (``tcb_cetc``).
* ``CETC-Seq-D``: the same after ``degree_order`` on the GPU.
* ``CETC-Seq-FE``: covering ratio below ``COVER_RATIO_THRESHOLD`` -> cover-edge
  counting, else the forward count (``tcb_cetc_fe``).
* ``CETC-Seq-S`` / ``-SD`` / ``-SR``: the split hybrid as the reference
  runs it (sequential.py:186-238): BFS levels, G0 = the horizontal edges as
  a CSR of its own (``tcb_split_by_level``), the forward count of G0
  (``tcb_forward_count``) plus the cross count (``tcb_split_cross_count``:
  split_cross_count_k, triangles with one G0 edge and two level-spanning
  ones); -SD after degree relabeling, -SR re-splitting G0 while it holds
  more than the threshold of the edges and shrinks.
"""
from __future__ import annotations

from . import ops as _ops
from .graph import Graph, degree_order_device, device_graph

__all__ = ["COVER_RATIO_THRESHOLD", "SEQUENTIAL_IDS", "tc_cetc", "tc_cetc_degree",
           "tc_cetc_fe", "tc_cetc_split", "tc_cetc_split_degree", "tc_cetc_split_recursive",
           "tc_forward_gpu", "count_sequential"]

# sequential.py:53-56: the covering-ratio switch point of the hybrids
COVER_RATIO_THRESHOLD = 0.7


def tc_cetc(g: Graph) -> int:
    """Cover-edge counting: BFS levels, then one intersection per horizontal
    edge with the off-level-or-greater-apex uniqueness test."""
    return int(_ops.cetc(device_graph(g)).triangles)


def tc_cetc_degree(g: Graph) -> int:
    """Cover-edge counting after degree relabeling (sequential.py:171-173)."""
    return int(_ops.cetc(degree_order_device(device_graph(g))).triangles)


def tc_cetc_fe(g: Graph, threshold: float = COVER_RATIO_THRESHOLD) -> int:
    """Forward-exchanging hybrid (sequential.py:176-183): cover-edge counting
    when the covering ratio is below ``threshold``, else forward."""
    r, _ = _ops.cetc_fe(device_graph(g), threshold)
    return int(r.triangles)


# sequential.py:62: the split recursion bottoms out below this many edges
SPLIT_RECURSION_FLOOR = 1024


def _split_count(dg) -> int:
    """One split (sequential.py:197-209) on the GPU: levels, G0 = the
    horizontal subgraph, T = forward count of G0 + the cross count."""
    level, _, _ = _ops.bfs_levels(dg)
    g0 = _ops.split_by_level(dg, level)
    return _ops.forward_count(g0) + _ops.split_cross_count(dg, level)


def tc_cetc_split(g: Graph) -> int:
    """Split hybrid (sequential.py:197-209): BFS levels, G0 = the horizontal
    edges and G1 = the level-spanning ones (tcb_split_by_level), the forward
    count of G0 (tcb_forward_count; the reference forward-hashes G0) plus the
    triangles with one G0 edge and two G1 edges (tcb_split_cross_count,
    split_cross_count_k)."""
    return _split_count(device_graph(g))


def tc_cetc_split_degree(g: Graph) -> int:
    """Split hybrid after degree relabeling (sequential.py:212-213)."""
    return _split_count(degree_order_device(device_graph(g)))


def tc_cetc_split_recursive(g: Graph, threshold: float = COVER_RATIO_THRESHOLD) -> int:
    """Recursive split (sequential.py:216-238): while the horizontal
    subgraph still holds more than `threshold` of the edges, shrinks, and has
    at least SPLIT_RECURSION_FLOOR edges, split it again (a new BFS on G0)
    instead of counting it forward."""
    return _split_recursive(device_graph(g), threshold, 1.0)


def _split_recursive(dg, threshold: float, prev_ratio: float) -> int:
    if dg.m == 0:
        return 0
    level, _, _ = _ops.bfs_levels(dg)
    g0 = _ops.split_by_level(dg, level)
    cross = _ops.split_cross_count(dg, level)
    ratio = g0.m / dg.m
    if ratio > threshold and ratio < prev_ratio and g0.m >= SPLIT_RECURSION_FLOOR:
        inner = _split_recursive(g0, threshold, ratio)
    else:
        inner = _ops.forward_count(g0)
    return inner + cross


def tc_forward_gpu(g: Graph) -> int:
    """The forward count on the GPU (the FE fallback; tcb_forward_count)."""
    return _ops.forward_count(device_graph(g))


SEQUENTIAL_IDS = {
    "CETC-Seq": tc_cetc,
    "CETC-Seq-D": tc_cetc_degree,
    "CETC-Seq-FE": tc_cetc_fe,
    "CETC-Seq-S": tc_cetc_split,
    "CETC-Seq-SD": tc_cetc_split_degree,
    "CETC-Seq-SR": tc_cetc_split_recursive,
}


def count_sequential(alg: str, g: Graph) -> int:
    """Dispatch by algorithm id (sequential.py:270-275)."""
    try:
        fn = SEQUENTIAL_IDS[alg]
    except KeyError:
        raise ValueError(f"unknown sequential algorithm id {alg!r}") from None
    return fn(g)
