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
* ``CETC-Seq-S`` / ``-SD`` / ``-SR``: the split hybrid counts the triangles
  with one horizontal edge (``split_cross_count_k`` over G0 x G1,
  _kernels.py:787-805) plus the triangles of the horizontal subgraph G0
  (forward-hashed on G0, recursively split for -SR).  Those two terms are
  exactly the cover-edge pass's two tallies — one horizontal edge with an
  off-level apex is c1, and a G0 triangle is the same-level tally (counted
  once, at the edge whose apex ranks above both endpoints: the forward count
  on G0 in owner order; c2 = 3 T(G0)) — so the GPU computes both in one
  fused pass and returns c1 + c2/3; the CPU split into two graphs exists to
  cut merge work, which the OFF/UP list intersection already avoids.
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


def tc_cetc_split(g: Graph) -> int:
    """Split hybrid (sequential.py:197-209): cross triangles (c1) plus the
    horizontal subgraph's triangles (c2 / 3), one fused GPU pass."""
    r = _ops.cetc(device_graph(g))
    return int(r.c1 + r.c2 // 3)


def tc_cetc_split_degree(g: Graph) -> int:
    """Split hybrid after degree relabeling (sequential.py:212-213)."""
    r = _ops.cetc(degree_order_device(device_graph(g)))
    return int(r.c1 + r.c2 // 3)


def tc_cetc_split_recursive(g: Graph, threshold: float = COVER_RATIO_THRESHOLD) -> int:
    """Recursive split (sequential.py:216-238): the recursion only re-splits
    G0 to cut CPU merge work; the total is the same c1 + T(G0)."""
    del threshold
    return tc_cetc_split(g)


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
