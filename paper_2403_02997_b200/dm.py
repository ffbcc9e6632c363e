"""CETC-DM, the paper's distributed-memory cover-edge count (dmsim.py), on
GPUs.

Vertices are split into p contiguous ranges of about 2m/p adjacency
endpoints (partition_graph, dmsim.py:96-113).  Processor i owns the cover
edges whose lower endpoint falls in its range and counts, for every cover
edge it sees, only the apexes in its own range (cetc_count_restricted_k,
_kernels.py:759-783) — so it needs the adjacency restricted to its id range,
a column block of 2m/p entries, not the whole graph.  It first counts its own
edges, then in rounds j = 1 .. p-1 the edge set of processor i XOR j (a
perfect pairing when p is a power of two, dmsim.py:147-152); the tallies sum
to the triangle count (every apex lies in exactly one range).

* `simulate_cetc_dm(g, p)` runs the p logical processors on one GPU (the
  reference's simulator, dmsim.py:144-200): same count, same per-processor
  edge counts, same shipment log.
* `cetc_dm_distributed(dg, group)` runs one processor per rank of a
  torch.distributed group: cover sets are all-gathered (the XOR rounds'
  union), each rank counts its apex range on its GPU, one all-reduce sums
  the tallies.  With NCCL the exchange runs over NVLink; the CPU tests run
  the same host logic over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Partition",
    "Shipment",
    "DmSimResult",
    "partition_graph",
    "partition_bounds",
    "owned_cover",
    "xor_schedule",
    "simulate_cetc_dm",
    "cetc_dm_distributed",
    "exchange_cover",
    "reduce_tally",
]


@dataclass(frozen=True)
class Partition:
    p: int
    bounds: np.ndarray          # length p+1; bounds[i]..bounds[i+1] owned by i
    owner: np.ndarray           # per-vertex processor id
    endpoint_loads: np.ndarray  # sum of degrees per processor

    def vertex_range(self, i: int) -> tuple[int, int]:
        return int(self.bounds[i]), int(self.bounds[i + 1])


def partition_bounds(degrees: np.ndarray, p: int) -> np.ndarray:
    """dmsim.py:96-109: p contiguous ranges of about 2m/p endpoints each."""
    n = len(degrees)
    if p < 1:
        raise ValueError("p must be >= 1")
    if p > n:
        raise ValueError(f"p={p} exceeds vertex count n={n}")
    cum = np.cumsum(np.asarray(degrees, dtype=np.int64))
    total = int(cum[-1]) if n else 0
    bounds = np.zeros(p + 1, dtype=np.int64)
    for i in range(1, p):
        bounds[i] = np.searchsorted(cum, i * total / p, side="right")
    bounds[p] = n
    np.maximum.accumulate(bounds, out=bounds)
    return bounds


def partition_graph(g, p: int) -> Partition:
    """dmsim.py:96-113 partition_graph on a Graph (host arrays)."""
    deg = np.diff(np.asarray(g.row_offsets, dtype=np.int64))
    bounds = partition_bounds(deg, p)
    cum = np.cumsum(deg)
    owner = np.searchsorted(bounds, np.arange(g.n), side="right").astype(np.int32) - 1
    loads = np.array([int(cum[b - 1]) if b else 0 for b in bounds[1:]], dtype=np.int64)
    loads[1:] -= loads[:-1].copy()
    return Partition(p=p, bounds=bounds, owner=owner, endpoint_loads=loads)


@dataclass(frozen=True)
class Shipment:
    """One cover-edge set transfer: sender -> receiver in a given round."""

    round: int
    sender: int
    receiver: int
    edges: int


@dataclass(frozen=True)
class DmSimResult:
    count: int
    p: int
    local_edges: tuple[int, ...]  # |S_i| consumed at home by each processor
    shipments: tuple[Shipment, ...] = field(repr=False)

    @property
    def total_shipped(self) -> int:
        return sum(s.edges for s in self.shipments)


def xor_schedule(p: int):
    """dmsim.py:187-196: round j = 1 .. p-1, receiver i gets i ^ j's set."""
    if p < 1 or (p & (p - 1)) != 0:
        raise ValueError("p must be a power of two")
    return [[(i ^ j, i) for i in range(p)] for j in range(1, p)]


def owned_cover(cover_u, bounds):
    """Processor of each cover edge: the range holding its lower endpoint
    (dmsim.py:164-167).  Works on numpy arrays or torch tensors."""
    try:
        import torch
        if isinstance(cover_u, torch.Tensor):
            b = torch.as_tensor(bounds, dtype=torch.int64, device=cover_u.device)
            return torch.searchsorted(b, cover_u.to(torch.int64), right=True) - 1
    except ImportError:  # pragma: no cover
        pass
    return np.searchsorted(bounds, cover_u, side="right") - 1


def simulate_cetc_dm(g, p: int) -> DmSimResult:
    """dmsim.py:144-200 simulate_cetc_dm with every processor's counting on
    the GPU (tcb_cetc_count_restricted): count, per-processor local edge
    counts and the XOR shipment log."""
    from . import ops
    from .graph import device_graph
    schedule = xor_schedule(p)
    part = partition_graph(g, p)
    dg = device_graph(g)
    level, _, _ = ops.bfs_levels(dg)
    cu, cv = ops.cover_select(dg, level)
    own = owned_cover(cu, part.bounds)
    sets = [(cu[own == i], cv[own == i]) for i in range(p)]

    def count_for(i: int, edges) -> int:
        lo, hi = part.vertex_range(i)
        return ops.cetc_count_restricted(dg, level, edges[0], edges[1], lo, hi)[0]

    tallies = [count_for(i, sets[i]) for i in range(p)]
    shipments = []
    for j, pairs in enumerate(schedule, start=1):
        for sender, receiver in pairs:
            shipments.append(Shipment(round=j, sender=sender, receiver=receiver,
                                      edges=int(sets[sender][0].numel())))
            tallies[receiver] += count_for(receiver, sets[sender])
    return DmSimResult(count=int(sum(tallies)), p=p,
                       local_edges=tuple(int(s[0].numel()) for s in sets),
                       shipments=tuple(shipments))


def cetc_dm_distributed(dg, group=None) -> int:
    """One CETC-DM processor per rank.  Each rank labels its replica, keeps
    the cover edges its vertex range owns, all-gathers the cover sets (the
    union the XOR rounds deliver), counts the apexes of its range for all of
    them on its GPU, and one all-reduce sums the tallies."""
    import torch
    import torch.distributed as dist

    from . import ops
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    deg = (dg.row_offsets[1:] - dg.row_offsets[:-1]).cpu().numpy()
    bounds = partition_bounds(deg, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    level, _, _ = ops.bfs_levels(dg)
    cu, cv = ops.cover_select(dg, level)
    mine = owned_cover(cu, bounds) == rank
    dev = dg.device
    if world > 1 and dist.get_backend(group) != "nccl":
        dev = torch.device("cpu")
    us, vs = exchange_cover(cu[mine].to(dev), cv[mine].to(dev), group)
    t, _, _ = ops.cetc_count_restricted(dg, level, us.to(dg.device), vs.to(dg.device), lo, hi)
    return reduce_tally(t, group, dev)


def exchange_cover(my_u, my_v, group=None):
    """The XOR rounds' net effect: every rank ends with every rank's cover
    set (dmsim.py:187-196).  Two all-gathers (sizes, then the padded
    (u, v) pairs) on the tensors' device.  Returns (us, vs) in rank order."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return my_u, my_v
    world = dist.get_world_size(group)
    dev = my_u.device
    size = torch.tensor([my_u.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(x.item()) for x in sizes]
    cap = max(max(sizes), 1)
    pairs = torch.zeros(2, cap, dtype=torch.int32, device=dev)
    pairs[0, : my_u.numel()] = my_u.to(torch.int32)
    pairs[1, : my_v.numel()] = my_v.to(torch.int32)
    got = [torch.empty_like(pairs) for _ in range(world)]
    dist.all_gather(got, pairs, group=group)
    us = torch.cat([got[r][0, : sizes[r]] for r in range(world)])
    vs = torch.cat([got[r][1, : sizes[r]] for r in range(world)])
    return us, vs


def reduce_tally(t: int, group=None, device=None) -> int:
    """The final integer reduction (dmsim.py:198): one all-reduce."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return int(t)
    buf = torch.tensor([int(t)], dtype=torch.int64, device=device)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return int(buf.item())
