"""CETC-Seq entry point and registry (drop-in for tricount.sequential's
cover-edge path).

``tc_cetc`` keeps the reference contract (sequential.py:164-168): a
normalized read-only Graph in, the exact triangle count out as ``int``, with
the BFS preprocessing charged to the call.  The work runs as the fused GPU
path (``tcb_cetc``).
"""
from __future__ import annotations

from . import ops as _ops
from .graph import Graph, device_graph

__all__ = ["SEQUENTIAL_IDS", "tc_cetc", "count_sequential"]


def tc_cetc(g: Graph) -> int:
    """Cover-edge counting: BFS levels, then one intersection per horizontal
    edge with the off-level-or-greater-apex uniqueness test."""
    return int(_ops.cetc(device_graph(g)).triangles)


SEQUENTIAL_IDS = {
    "CETC-Seq": tc_cetc,
}


def count_sequential(alg: str, g: Graph) -> int:
    """Dispatch by algorithm id (sequential.py:270-275)."""
    try:
        fn = SEQUENTIAL_IDS[alg]
    except KeyError:
        raise ValueError(f"unknown sequential algorithm id {alg!r}") from None
    return fn(g)
