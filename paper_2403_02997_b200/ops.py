"""Device-level operations of the CETC path over a DeviceGraph.

Thin wrappers over the C ABI (include/tricount_b200.h); each cites the
reference function it replaces.  Everything runs on the current torch stream
of the graph's device.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import DeviceGraph

__all__ = [
    "CetcResult",
    "bfs_levels",
    "cover_select",
    "cetc_count",
    "cetc_count_restricted",
    "cetc",
    "cetc_shard",
    "cetc_host",
]


@dataclass(frozen=True)
class CetcResult:
    triangles: int
    c1: int
    c2: int
    ncover: int
    components: int
    max_level: int
    level: object = None      # torch int32 [n] on device (when requested)
    cover_u: object = None    # torch int32 [ncover]
    cover_v: object = None


def bfs_levels(dg: DeviceGraph):
    """_kernels.py:129-157 bfs_levels_k (levels, components, max_level).
    Returns (level int32 tensor [n], components, max_level)."""
    import torch
    ctx = _lib.context(dg.device.index)
    level = torch.empty(max(dg.n, 1), dtype=torch.int32, device=dg.device)
    comps = ctypes.c_int64(0)
    ml = ctypes.c_int64(0)
    ctx.check(ctx.lib.tcb_bfs_levels(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                     _lib.ptr(dg.src), dg.n, dg.m, _lib.ptr(level),
                                     ctypes.byref(comps), ctypes.byref(ml)))
    return level[: dg.n], int(comps.value), int(ml.value)


def bfs_parent(dg: DeviceGraph, level, max_level: int):
    """The FIFO parents of bfs_levels_k (_kernels.py:143-156): int32 tensor
    [n], -1 at component roots (tcb_bfs_parent)."""
    import torch
    ctx = _lib.context(dg.device.index)
    level = level.to(device=dg.device, dtype=torch.int32).contiguous()
    parent = torch.empty(max(dg.n, 1), dtype=torch.int32, device=dg.device)
    ctx.check(ctx.lib.tcb_bfs_parent(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                     dg.n, _lib.ptr(level), int(max_level), _lib.ptr(parent)))
    return parent[: dg.n]


def edge_classes(dg: DeviceGraph, level, parent):
    """bfs.py:83-87: int8 EdgeClass per canonical edge (tcb_edge_classes)."""
    import torch
    ctx = _lib.context(dg.device.index)
    level = level.to(device=dg.device, dtype=torch.int32).contiguous()
    parent = parent.to(device=dg.device, dtype=torch.int32).contiguous()
    out = torch.empty(max(dg.m, 1), dtype=torch.int8, device=dg.device)
    ctx.check(ctx.lib.tcb_edge_classes(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                       _lib.ptr(dg.src), dg.n, dg.m, _lib.ptr(level),
                                       _lib.ptr(parent), _lib.ptr(out)))
    return out[: dg.m]


def cover_select(dg: DeviceGraph, level):
    """bfs.py:97-106 cover_edges: horizontal u<v edges, lexicographic.
    Returns (cover_u, cover_v) int32 tensors."""
    import torch
    ctx = _lib.context(dg.device.index)
    level = level.to(device=dg.device, dtype=torch.int32).contiguous()
    cu = torch.empty(max(dg.m, 1), dtype=torch.int32, device=dg.device)
    cv = torch.empty(max(dg.m, 1), dtype=torch.int32, device=dg.device)
    k = ctypes.c_int64(0)
    ctx.check(ctx.lib.tcb_cover_select(ctx.h, _lib.ptr(level), _lib.ptr(dg.src),
                                       _lib.ptr(dg.neighbors), dg.m, _lib.ptr(cu), _lib.ptr(cv),
                                       ctypes.byref(k)))
    k = int(k.value)
    return cu[:k], cv[:k]


def cetc_count(dg: DeviceGraph, level, cover_u, cover_v, k0: int = 0, k1: int | None = None):
    """_kernels.py:729-755 cetc_sm_range_k over cover edges [k0, k1).
    Returns (t, c1, c2); over the full set t == c1 + c2 // 3."""
    import torch
    ctx = _lib.context(dg.device.index)
    k = int(cover_u.numel())
    if int(cover_v.numel()) != k:
        raise ValueError("cover_u and cover_v differ in length")
    if k1 is None:
        k1 = k
    if not 0 <= k0 <= k1 <= k:
        raise ValueError(f"need 0 <= k0 <= k1 <= {k}, got k0={k0}, k1={k1}")
    out = (ctypes.c_int64 * 3)()
    level = level.to(device=dg.device, dtype=torch.int32).contiguous()
    cu = cover_u.to(device=dg.device, dtype=torch.int32).contiguous()
    cv = cover_v.to(device=dg.device, dtype=torch.int32).contiguous()
    ctx.check(ctx.lib.tcb_cetc_count(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                     _lib.ptr(level), dg.n, _lib.ptr(cu),
                                     _lib.ptr(cv), k0, k1,
                                     ctypes.cast(out, ctypes.POINTER(ctypes.c_int64))))
    return int(out[0]), int(out[1]), int(out[2])


def cetc_count_restricted(dg: DeviceGraph, level, cover_u, cover_v, lo: int, hi: int):
    """_kernels.py:759-783 cetc_count_restricted_k: the cover edges'
    apexes with lo <= w < hi only (one CETC-DM processor's share).  Returns
    (t, c1, c2) of those apexes; t is the reference's count."""
    import torch
    ctx = _lib.context(dg.device.index)
    k = int(cover_u.numel())
    out = (ctypes.c_int64 * 3)()
    level = level.to(device=dg.device, dtype=torch.int32).contiguous()
    cu = cover_u.to(device=dg.device, dtype=torch.int32).contiguous()
    cv = cover_v.to(device=dg.device, dtype=torch.int32).contiguous()
    ctx.check(ctx.lib.tcb_cetc_count_restricted(
        ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors), _lib.ptr(level), dg.n,
        _lib.ptr(cu), _lib.ptr(cv), k, int(lo), int(hi),
        ctypes.cast(out, ctypes.POINTER(ctypes.c_int64))))
    return int(out[0]), int(out[1]), int(out[2])


def cetc(dg: DeviceGraph, keep_level: bool = False, keep_cover: bool = False) -> CetcResult:
    """sequential.py:164-168 tc_cetc, fused on the device: CC roots -> BFS
    levels -> cover selection -> intersection -> exact 64-bit count."""
    import torch
    ctx = _lib.context(dg.device.index)
    level = cu = cv = None
    if keep_level:
        level = torch.empty(max(dg.n, 1), dtype=torch.int32, device=dg.device)
    if keep_cover:
        cu = torch.empty(max(dg.m, 1), dtype=torch.int32, device=dg.device)
        cv = torch.empty(max(dg.m, 1), dtype=torch.int32, device=dg.device)
    r = _lib.TcbResult()
    ctx.check(ctx.lib.tcb_cetc(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                               _lib.ptr(dg.src), dg.n, dg.m, _lib.ptr(level), _lib.ptr(cu),
                               _lib.ptr(cv), ctypes.byref(r)))
    d = r.as_dict()
    return CetcResult(
        level=level[: dg.n] if level is not None else None,
        cover_u=cu[: d["ncover"]] if cu is not None else None,
        cover_v=cv[: d["ncover"]] if cv is not None else None,
        **d)


def split_by_level(dg: DeviceGraph, level) -> DeviceGraph:
    """_split_by_level (sequential.py:186-193): the horizontal subgraph G0
    (edges with equal levels) as a DeviceGraph of its own (tcb_split_by_level)."""
    import torch
    ctx = _lib.context(dg.device.index)
    level = level.to(device=dg.device, dtype=torch.int32).contiguous()
    row0 = torch.empty(dg.n + 1, dtype=torch.int64, device=dg.device)
    nb0 = torch.empty(max(2 * dg.m, 1), dtype=torch.int32, device=dg.device)
    src0 = torch.empty(max(2 * dg.m, 1), dtype=torch.int32, device=dg.device)
    m0 = ctypes.c_int64(0)
    ctx.check(ctx.lib.tcb_split_by_level(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                         _lib.ptr(dg.src), dg.n, dg.m, _lib.ptr(level),
                                         _lib.ptr(row0), _lib.ptr(nb0), _lib.ptr(src0),
                                         ctypes.byref(m0)))
    m0 = int(m0.value)
    return DeviceGraph(n=dg.n, m=m0, row_offsets=row0, neighbors=nb0[: 2 * m0],
                       src=src0[: 2 * m0])


def split_cross_count(dg: DeviceGraph, level) -> int:
    """split_cross_count_k (_kernels.py:786-805) for the split of `dg` by
    `level`: triangles with one horizontal edge and two level-spanning ones
    (tcb_split_cross_count: the owner-staged intersection of the OFF lists)."""
    import torch
    ctx = _lib.context(dg.device.index)
    level = level.to(device=dg.device, dtype=torch.int32).contiguous()
    t = ctypes.c_int64(0)
    ctx.check(ctx.lib.tcb_split_cross_count(ctx.h, _lib.ptr(dg.row_offsets),
                                            _lib.ptr(dg.neighbors), _lib.ptr(dg.src), dg.n,
                                            dg.m, _lib.ptr(level), ctypes.byref(t)))
    return int(t.value)


def forward_count(dg: DeviceGraph) -> int:
    """Forward triangle count on the GPU (tcb_forward_count; the forward
    branch of tc_cetc_fe, sequential.py:176-183)."""
    ctx = _lib.context(dg.device.index)
    t = ctypes.c_int64(0)
    ctx.check(ctx.lib.tcb_forward_count(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                        _lib.ptr(dg.src), dg.n, dg.m, ctypes.byref(t)))
    return int(t.value)


def cetc_fe(dg: DeviceGraph, threshold: float = 0.7):
    """tc_cetc_fe (sequential.py:176-183) fused on the GPU (tcb_cetc_fe).
    Returns (CetcResult, used_forward); c1/c2 are -1 on the forward branch."""
    ctx = _lib.context(dg.device.index)
    r = _lib.TcbResult()
    fwd = ctypes.c_int32(0)
    ctx.check(ctx.lib.tcb_cetc_fe(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                  _lib.ptr(dg.src), dg.n, dg.m, float(threshold),
                                  ctypes.byref(r), ctypes.byref(fwd)))
    return CetcResult(**r.as_dict()), bool(fwd.value)


def cetc_shard(dg: DeviceGraph, shard: int, nshards: int) -> CetcResult:
    """One rank's share of the fused path: replicated
    labeling/selection, intersection over slice `shard` of `nshards`.
    c1/c2 are partials (sum them across shards, then T = c1 + c2/3 —
    dist.reduce_counts); triangles is -1 when nshards > 1."""
    ctx = _lib.context(dg.device.index)
    r = _lib.TcbResult()
    ctx.check(ctx.lib.tcb_cetc_shard(ctx.h, _lib.ptr(dg.row_offsets), _lib.ptr(dg.neighbors),
                                     _lib.ptr(dg.src), dg.n, dg.m, shard, nshards,
                                     ctypes.byref(r)))
    return CetcResult(**r.as_dict())


def cetc_host(row_offsets: np.ndarray, neighbors: np.ndarray, n: int,
              want_level: bool = False, device: int | None = None):
    """The host-buffer entry (tcb_cetc_host): numpy CSR in, result (and int64
    levels, BfsLabeling.level's dtype) out; uploads and downloads are inside."""
    ctx = _lib.context(device)
    row = np.ascontiguousarray(row_offsets, dtype=np.int64)
    nb = np.ascontiguousarray(neighbors, dtype=np.int32)
    if len(row) != n + 1:
        raise ValueError("row_offsets must have n+1 entries")
    level = np.empty(max(n, 1), dtype=np.int64) if want_level else None
    r = _lib.TcbResult()
    ctx.check(ctx.lib.tcb_cetc_host(
        ctx.h, row.ctypes.data_as(ctypes.c_void_p),
        nb.ctypes.data_as(ctypes.c_void_p) if len(nb) else ctypes.c_void_p(0), n,
        level.ctypes.data_as(ctypes.c_void_p) if level is not None else ctypes.c_void_p(0),
        ctypes.byref(r)))
    d = r.as_dict()
    if level is not None:
        d["level"] = level[:n]
    return d


def cetc_host_shard(row_offsets: np.ndarray, neighbors: np.ndarray, n: int, shard: int,
                    nshards: int, device: int | None = None) -> dict:
    """One rank's host-buffer entry (tcb_cetc_host_shard): numpy CSR in,
    c1/c2 partials out (sum them across ranks: dist.reduce_counts)."""
    ctx = _lib.context(device)
    row = np.ascontiguousarray(row_offsets, dtype=np.int64)
    nb = np.ascontiguousarray(neighbors, dtype=np.int32)
    if len(row) != n + 1:
        raise ValueError("row_offsets must have n+1 entries")
    r = _lib.TcbResult()
    ctx.check(ctx.lib.tcb_cetc_host_shard(
        ctx.h, row.ctypes.data_as(ctypes.c_void_p),
        nb.ctypes.data_as(ctypes.c_void_p) if len(nb) else ctypes.c_void_p(0), n,
        int(shard), int(nshards), ctypes.byref(r)))
    return r.as_dict()
