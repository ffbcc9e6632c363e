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
* The communication-volume model (dmsim.py:203-336): `comm_volume_*`,
  `projected_comm_volume`, `fit_scaling`, `comm_report`, `reports_to_csv`,
  `format_volume` — host arithmetic over the GPU labeling and count.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "CommReport",
    "ScalingFit",
    "ceil_log2",
    "format_volume",
    "wedge_count",
    "comm_volume_previous",
    "comm_volume_cetc_dm",
    "comm_volume_breakdown",
    "projected_comm_volume",
    "fit_scaling",
    "comm_report",
    "reports_to_csv",
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

    def local_adjacency(self, g, i: int) -> tuple[np.ndarray, np.ndarray]:
        """dmsim.py:88-93: the CSR slice of processor i's owned vertices,
        offsets rebased to 0."""
        lo, hi = self.vertex_range(i)
        row = np.asarray(g.row_offsets)
        start = row[lo]
        return row[lo:hi + 1] - start, np.asarray(g.neighbors)[start:row[hi]]


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


def simulate_cetc_dm(g, p: int, workers: int = 1) -> DmSimResult:
    """dmsim.py:144-200 simulate_cetc_dm with every processor's counting on
    the GPU (tcb_cetc_count_restricted): count, per-processor local edge
    counts and the XOR shipment log.  ``workers`` is accepted for the
    reference's signature; as there (dmsim.py:149-151) the result and the
    exchange log do not depend on it — the GPU is the worker pool."""
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


# ---------------------------------------------------------------------------
# The communication-volume model (dmsim.py:203-336). Pure host arithmetic over
# graph statistics; the labeling it prices (levels, |S|, depth) and the
# triangle count come from the GPU path.

_BYTE_SCALES = tuple((u, 1 << (10 * k)) for k, u in
                     ((6, "EB"), (5, "PB"), (4, "TB"), (3, "GB"), (2, "MB"), (1, "KB")))


def ceil_log2(x: int) -> int:
    """dmsim.py:61-65: the least b with 2**b >= x (x >= 1)."""
    x = int(x)
    if x < 1:
        raise ValueError("ceil_log2 requires x >= 1")
    return (x - 1).bit_length()


def format_volume(bits: float) -> str:
    """dmsim.py:68-73: a bit count rendered in binary byte units, 3 sig. digits."""
    nbytes = bits / 8
    unit, scale = next(((u, sc) for u, sc in _BYTE_SCALES if nbytes >= sc), ("B", 1))
    return f"{nbytes / scale:.3g}{unit}"


def wedge_count(g) -> int:
    """graph.py:216-219: 2-paths, the sum over vertices of C(d(v), 2)."""
    deg = np.diff(np.asarray(g.row_offsets, dtype=np.int64))
    return int(np.sum(deg * (deg - 1)) // 2)


def comm_volume_previous(g, p: int = 1) -> int:
    """dmsim.py:203-212: the wedge-query baseline, 2 ids per wedge; p is
    accepted for symmetry and does not enter."""
    return 0 if g.n == 0 else 2 * ceil_log2(g.n) * wedge_count(g)


def comm_volume_breakdown(g, lab, p: int) -> tuple[int, int, int]:
    """dmsim.py:225-238: bits for (BFS construction, cover-edge exchange,
    final reduction) in exact integers: m(log D + 3 log n), |S| p log n,
    (p - 1) log n with log = ceil_log2 of max(., 1)."""
    ln = ceil_log2(max(g.n, 1))
    ld = ceil_log2(max(lab.max_level, 1))
    return (g.m * (ld + 3 * ln), lab.horizontal_count * p * ln, (p - 1) * ln)


def comm_volume_cetc_dm(g, lab, p: int) -> int:
    """dmsim.py:215-222: total model bits for distributed cover-edge counting."""
    if len(lab.level) != g.n:
        raise ValueError("labeling does not match graph")
    return 0 if g.n == 0 else sum(comm_volume_breakdown(g, lab, p))


def projected_comm_volume(n: int, m: int, k: float, p: int, log_d: int) -> float:
    """dmsim.py:241-250: the model for a graph too large to build, with a
    covering-ratio estimate k and a fixed depth width log_d (float bits)."""
    ln = ceil_log2(n)
    return m * log_d + m * (k * p + 3) * ln + (p - 1) * ln


@dataclass(frozen=True)
class ScalingFit:
    """dmsim.py:253-263: y = a exp(b x) ("exponential") or y = a x^b ("power")."""

    kind: str
    a: float
    b: float
    r_squared: float

    def predict(self, x: float) -> float:
        if self.kind == "exponential":
            return self.a * math.exp(self.b * x)
        return self.a * x**self.b


_FIT_AXES = {"exponential": lambda x: x, "power": np.log}


def fit_scaling(xs, ys, kind: str = "exponential") -> ScalingFit:
    """dmsim.py:266-290: degree-1 least squares of ln y against x (or ln x);
    r^2 computed in log space, 1.0 for an exact constant fit."""
    if kind not in _FIT_AXES:
        raise ValueError(f"unknown fit kind {kind!r}")
    x = np.asarray(xs, dtype=np.float64)
    y = np.asarray(ys, dtype=np.float64)
    if len(x) != len(y) or len(x) < 3:
        raise ValueError("need at least 3 (x, y) points")
    if (y <= 0).any():
        raise ValueError("y values must be positive for a log-space fit")
    if kind == "power" and (x <= 0).any():
        raise ValueError("x values must be positive for a power-law fit")
    t, ly = _FIT_AXES[kind](x), np.log(y)
    slope, icpt = np.polyfit(t, ly, 1)
    ss_res = float(((ly - (icpt + slope * t)) ** 2).sum())
    ss_tot = float(((ly - ly.mean()) ** 2).sum())
    r2 = (1.0 - ss_res / ss_tot) if ss_tot != 0.0 else float(ss_res < 1e-12)
    return ScalingFit(kind, float(np.exp(icpt)), float(slope), r2)


@dataclass(frozen=True)
class CommReport:
    """dmsim.py:293-305: one baseline-vs-cover-edge comparison row."""

    graph: str
    n: int
    m: int
    triangles: int
    wedges: int
    k: float
    p: int
    bits_previous: int
    bits_cetc_dm: int
    reduction: float
    log_n: int
    log_d: int


def comm_report(g, p: int, name: str = "") -> CommReport:
    """dmsim.py:308-326; labeling and triangle count computed on the GPU
    (one bfs_label plus the cover-edge count)."""
    from .bfs import bfs_label
    from .sequential import tc_cetc
    lab = bfs_label(g)
    tri = tc_cetc(g)
    before = comm_volume_previous(g, p)
    after = comm_volume_cetc_dm(g, lab, p)
    return CommReport(
        graph=name, n=g.n, m=g.m, triangles=tri, wedges=wedge_count(g),
        k=(lab.horizontal_count / g.m) if g.m else 0.0, p=p,
        bits_previous=before, bits_cetc_dm=after,
        reduction=(before / after) if after else float("inf"),
        log_n=ceil_log2(max(g.n, 1)), log_d=ceil_log2(max(lab.max_level, 1)))


_CSV_HEADER = "graph,n,m,triangles,wedges,c,p,bits_previous,bits_cetc_dm,reduction"


def reports_to_csv(reports) -> str:
    """dmsim.py:329-336: CSV rows, covering ratio to 6 places, reduction to 4."""
    rows = [_CSV_HEADER]
    rows += [",".join((r.graph, str(r.n), str(r.m), str(r.triangles), str(r.wedges),
                       f"{r.k:.6f}", str(r.p), str(r.bits_previous), str(r.bits_cetc_dm),
                       f"{r.reduction:.4f}")) for r in reports]
    return "\n".join(rows) + "\n"
