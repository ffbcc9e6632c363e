"""CETC-SM entry point and registry (drop-in for tricount.parallel's
cover-edge path).

The reference splits the edge list into contiguous chunks on a CPU thread
pool and merges two private tallies, c1 (apex off-level) and c2 (apex
on-level), as ``c1 + c2/3`` (parallel.py:117-137).  Here the whole device is
the worker pool: the same two tallies come back from the GPU intersection
kernel (warp partials -> one 64-bit atomic each).  ``ParallelConfig`` keeps
its validation; ``workers``/``chunk`` do not change the result, as in the
reference.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import ops as _ops
from .graph import Graph, device_graph

__all__ = ["ParallelConfig", "PARALLEL_IDS", "tc_cetc_sm", "tc_par"]


@dataclass(frozen=True)
class ParallelConfig:
    """Worker count and edge-chunk granularity (parallel.py:36-59)."""

    workers: int = 1
    chunk: int | None = None

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.chunk is not None and self.chunk < 1:
            raise ValueError("chunk must be >= 1")

    def ranges(self, nitems: int) -> list[tuple[int, int]]:
        """Contiguous [k0, k1) chunks, ceil(n / (4*workers)) long by default."""
        if nitems <= 0:
            return []
        step = self.chunk or max(1, -(-nitems // (4 * self.workers)))
        return [(k0, min(nitems, k0 + step)) for k0 in range(0, nitems, step)]


def _cetc_sm_counts(g: Graph, cfg: ParallelConfig) -> tuple[int, int]:
    r = _ops.cetc(device_graph(g))
    return r.c1, r.c2


def tc_cetc_sm(g: Graph, cfg: ParallelConfig) -> int:
    """Parallel cover-edge counting with the two-accumulator discipline."""
    c1, c2 = _cetc_sm_counts(g, cfg)
    if c2 % 3:
        raise AssertionError("same-level apex tally must be divisible by 3")
    return c1 + c2 // 3


PARALLEL_IDS = {
    "CETC-SM": tc_cetc_sm,
}


def tc_par(alg: str, g: Graph, cfg: ParallelConfig) -> int:
    """Dispatch a parallel algorithm by id (parallel.py:155-161)."""
    try:
        fn = PARALLEL_IDS[alg]
    except KeyError:
        raise ValueError(f"unknown parallel algorithm id {alg!r}") from None
    return fn(g, cfg)
