"""Multi-rank path on CPU (gloo, world size 2) and on one GPU (shards run one
after another, no rank waits on another).

The CPU test restates the sharded intersection with numpy on the oracle's
levels: each rank counts the cover edges whose owner maps to it, and
reduce_counts sums the partials with a real all-reduce.  It pins the owner /
shard rule (every cover edge counted by exactly one rank) and the reduction.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import SMALL_CASES
from paper_2403_02997_b200 import dist as tdist

CASES = [c for c in SMALL_CASES if c.name in ("karate", "rmat10_42", "k8", "er60_915", "rmat7_9")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partials(case, rank, world):
    level, _, _, _ = oracle.bfs_levels(case.row, case.nb, case.n)
    deg = np.diff(case.row)
    cov = oracle.cover_select(level, case.eu, case.ev)
    c1 = c2 = t = 0
    if len(cov):
        u, v = cov[:, 0], cov[:, 1]
        own = tdist.owner_of(u, v, deg[u], deg[v])
        partner = np.where(own == u, v, u)
        # rank of each edge among its owner's cover edges, by partner id
        order = np.lexsort((partner, own))
        prank = np.empty(len(own), dtype=np.int64)
        so = own[order]
        starts = np.searchsorted(so, so, side="left")
        prank[order] = np.arange(len(so)) - starts
        mine = tdist.shard_of(own, prank, deg[own], world) == rank
        for a, b, x in zip(cov[mine][:, 0], cov[mine][:, 1], own[mine]):
            common = np.intersect1d(case.nb[case.row[a]:case.row[a + 1]],
                                    case.nb[case.row[b]:case.row[b + 1]])
            for w in common:
                if level[w] != level[a]:
                    c1 += 1
                    t += 1
                elif tdist.ranks_above(w, tdist.degree_bucket(deg[w]), x,
                                       tdist.degree_bucket(deg[x])):
                    # a same-level triangle is kept at the edge whose apex
                    # ranks above both endpoints (intersect.cu); the device
                    # tallies c2 in the reference's units (3 per triangle)
                    c2 += 3
                    t += 1
    return t, c1, c2


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for case in CASES:
            part = _partials(case, rank, world)
            res[case.name] = (part, tdist.reduce_counts(part[1], part[2]))
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_sum_to_reference():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for case in CASES:
        parts = [out[r][case.name][0] for r in range(world)]
        reduced = [out[r][case.name][1] for r in range(world)]
        assert reduced[0] == reduced[1] == (case.T, case.c1, case.c2), case.name
        assert sum(p[0] for p in parts) == case.T


def test_owner_rule():
    # degree bucket floor(log2 d) first, ties (same bucket) to the lower id:
    # (6, 8) with degrees 5 and 7 share bucket 2, so 6 owns it
    u = np.array([1, 5, 3, 6]); v = np.array([2, 4, 9, 8])
    du = np.array([3, 7, 2, 5]); dv = np.array([3, 1, 5, 7])
    assert tdist.owner_of(u, v, du, dv).tolist() == [1, 5, 9, 6]
    # tiny owners shard by id; warp-tier blocks of 64 and CTA-tier blocks of
    # 1024 partners rotate over the ranks
    own = np.array([4, 5, 7, 7, 7, 9, 9])
    prank = np.array([0, 3, 0, 63, 64, 1023, 1024])
    deg = np.array([8, 10, 100, 100, 100, 4000, 4000])
    assert tdist.shard_of(own, prank, deg, 2).tolist() == [0, 1, 1, 1, 0, 1, 0]


def test_reduce_counts_single_process_passthrough():
    assert tdist.reduce_counts(4, 9) == (7, 4, 9)
    with pytest.raises(AssertionError):
        tdist.reduce_counts(4, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_gpu_shards_sum_to_total(world):
    import paper_2403_02997_b200 as tb
    for case in CASES:
        g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
        dg = tb.device_graph(g)
        parts = [tb.ops.cetc_shard(dg, r, world) for r in range(world)]
        assert all(p.triangles == -1 for p in parts)  # T is formed after the sum
        assert sum(p.c1 for p in parts) + sum(p.c2 for p in parts) // 3 == case.T, case.name
        assert sum(p.c1 for p in parts) == case.c1
        assert sum(p.c2 for p in parts) == case.c2
        assert all(p.ncover == len(case.cover) for p in parts)
        # the device's item sharding is exactly dist.shard_of's rule
        for r, p in enumerate(parts):
            _, c1, c2 = _partials(case, r, world)
            assert (p.c1, p.c2) == (c1, c2), (case.name, r)
        # the host-buffer entry of each rank gives the same partials
        for r, p in enumerate(parts):
            h = tb.ops.cetc_host_shard(case.row, case.nb, case.n, r, world)
            assert (h["c1"], h["c2"], h["triangles"]) == (p.c1, p.c2, -1 if world > 1 else h["triangles"])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 5])
def test_gpu_shards_build_their_own_records(world):
    """Every shard's CTA-tier items read partner records that the same call's
    record pass wrote: the record array is poisoned before each call
    (TCB_TEST_POISON_RECORDS), the tiers are shrunk so hub-and-spoke RMAT
    graphs run the CTA tier with several partner blocks per owner, and the
    shards' tallies must add up to the single-GPU ones."""
    import numpy as np
    import paper_2403_02997_b200 as tb
    ctx = tb._lib.context()
    for seed in (1, 2):
        g = tb.normalize(tb.generate_rmat(tb.RmatParams(scale=13, edge_factor=24, seed=seed)))
        dg = tb.device_graph(g)
        whole = tb.cetc(dg)
        try:
            ctx.set_test_flags(16 | 8)  # poison the records; general path
            for tuning in ((4, 16), (16, 4096), (0, 0)):
                ctx.set_tuning(*tuning)
                parts = [tb.ops.cetc_shard(dg, r, world) for r in range(world)]
                assert sum(p.c1 for p in parts) == whole.c1, (seed, tuning)
                assert sum(p.c2 for p in parts) == whole.c2, (seed, tuning)
                one = tb.cetc(dg)
                assert (one.triangles, one.c1, one.c2) == (whole.triangles, whole.c1, whole.c2)
        finally:
            ctx.set_tuning(0, 0)
            ctx.set_test_flags(0)


def _nccl_worker(rank, world, port, out):
    """One rank per GPU over NCCL: the product's distributed entries, each
    rank on its own GPU with its own replica of the graph."""
    import torch
    import paper_2403_02997_b200 as tb
    from paper_2403_02997_b200 import dm as tdm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                           device_id=torch.device("cuda", rank))
    try:
        res = {}
        for case in CASES:
            g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
            dg = tb.device_graph(g, device=rank)
            res[case.name] = (tdist.tc_cetc_distributed(dg), tdm.cetc_dm_distributed(dg))
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_ranks_sum_to_reference():
    """SURVEY.md §8(e) on real GPUs: owner-block shards + one 16-byte NCCL
    all-reduce (tc_cetc_distributed), and the CETC-DM cover-set all-gather +
    all-reduce (cetc_dm_distributed).  Needs two visible GPUs; the round's
    GPU box has one, so this skips there."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (one rank per GPU)")
    world = min(torch.cuda.device_count(), 4)
    out = mp.Manager().dict()
    mp.start_processes(_nccl_worker, args=(world, _free_port(), out), nprocs=world,
                       join=True, start_method="spawn")
    for case in CASES:
        for r in range(world):
            assert out[r][case.name] == (case.T, case.T), (case.name, r)


def _gloo_gpu_worker(rank, world, port, out):
    """The product's distributed entries with a real process group: gloo
    collectives on CPU tensors, every rank's kernels on cuda:0 (the ranks'
    kernels never wait on each other; only the host-side all-reduce and
    all-gather join them)."""
    import torch
    import paper_2403_02997_b200 as tb
    from paper_2403_02997_b200 import dm as tdm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for case in CASES:
            g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
            dg = tb.device_graph(g, device=0)
            res[case.name] = (tdist.tc_cetc_distributed(dg), tdm.cetc_dm_distributed(dg))
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_product_distributed_entries_gloo_world2():
    """tc_cetc_distributed and cetc_dm_distributed (not a restatement) over a
    world-2 gloo group, both ranks on one GPU: every rank gets T."""
    out = mp.Manager().dict()
    mp.start_processes(_gloo_gpu_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    for case in CASES:
        assert out[0][case.name] == out[1][case.name] == (case.T, case.T), case.name
