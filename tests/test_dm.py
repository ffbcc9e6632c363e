"""CETC-DM (dmsim.py): the distributed-memory cover-edge count.

Pinned by tests/golden/dm_cases.json, produced by the reference's own
partition_graph / simulate_cetc_dm / cetc_count_restricted_k
(tests/golden/make_dm_golden.py).  CPU tests check the oracle and the host
logic (partition, XOR schedule, cover-set exchange over gloo world-2);
GPU tests check the device counts through the C ABI.
"""
from __future__ import annotations

import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import SMALL_CASES
from paper_2403_02997_b200 import dm

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "dm_cases.json").read_text())
CASES = {c.name: c for c in SMALL_CASES if c.name in GOLD}
PARAMS = [(name, p) for name in sorted(GOLD) for p in sorted(GOLD[name], key=int)]


@pytest.mark.parametrize("name,p", PARAMS)
def test_oracle_matches_reference(name, p):
    c, g = CASES[name], GOLD[name][p]
    count, local, ships, restricted, bounds = oracle.dm_simulate(c.row, c.nb, c.level, c.cover,
                                                                 int(p))
    assert bounds.tolist() == g["bounds"]
    assert count == g["count"] == c.T
    assert local == g["local_edges"]
    assert [list(s) for s in ships] == g["shipments"]
    assert restricted == g["restricted"]


@pytest.mark.parametrize("name,p", PARAMS)
def test_host_partition_and_schedule(name, p):
    c, g = CASES[name], GOLD[name][p]
    p = int(p)
    assert dm.partition_bounds(np.diff(c.row), p).tolist() == g["bounds"]
    sched = dm.xor_schedule(p)
    assert [[j + 1, s, r] for j, rnd in enumerate(sched) for s, r in rnd] == \
        [s[:3] for s in g["shipments"]]
    own = dm.owned_cover(np.asarray(c.cover, dtype=np.int64).reshape(-1, 2)[:, 0],
                         np.asarray(g["bounds"]))
    assert np.bincount(own, minlength=p).tolist() == g["local_edges"]


def test_partition_errors():
    with pytest.raises(ValueError):
        dm.partition_bounds(np.ones(4, dtype=np.int64), 0)
    with pytest.raises(ValueError):
        dm.partition_bounds(np.ones(4, dtype=np.int64), 5)
    with pytest.raises(ValueError):
        dm.xor_schedule(3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for name, c in CASES.items():
            if str(world) not in GOLD[name]:
                continue
            bounds = dm.partition_bounds(np.diff(c.row), world)
            cover = torch.as_tensor(np.asarray(c.cover, dtype=np.int64).reshape(-1, 2))
            mine = dm.owned_cover(cover[:, 0], bounds) == rank
            us, vs = dm.exchange_cover(cover[mine, 0].to(torch.int32),
                                       cover[mine, 1].to(torch.int32))
            t = oracle.cetc_count_restricted(c.row, c.nb, c.level, us.numpy(), vs.numpy(),
                                             int(bounds[rank]), int(bounds[rank + 1]))
            res[name] = (t, dm.reduce_tally(t, device=torch.device("cpu")), int(us.numel()))
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_and_reduce():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for name, c in CASES.items():
        if str(world) not in GOLD[name]:
            continue
        g = GOLD[name][str(world)]
        parts = [out[r][name] for r in range(world)]
        assert all(pt[1] == c.T for pt in parts), name  # the all-reduced total
        assert [pt[0] for pt in parts] == [sum(row) for row in g["restricted"]], name
        assert all(pt[2] == len(c.cover) for pt in parts)  # every rank saw every edge


@pytest.mark.gpu
@pytest.mark.parametrize("name,p", PARAMS)
def test_gpu_simulate_cetc_dm(name, p):
    import paper_2403_02997_b200 as tb
    c, g = CASES[name], GOLD[name][p]
    graph = tb.normalize(tb.EdgeList(n=c.n, edges=c.pairs))
    r = tb.simulate_cetc_dm(graph, int(p))
    assert r.count == g["count"] == c.T
    assert list(r.local_edges) == g["local_edges"]
    assert [[s.round, s.sender, s.receiver, s.edges] for s in r.shipments] == g["shipments"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD))
def test_gpu_restricted_counts(name):
    import paper_2403_02997_b200 as tb
    c = CASES[name]
    dg = tb.device_graph(tb.normalize(tb.EdgeList(n=c.n, edges=c.pairs)))
    level, _, _ = tb.ops.bfs_levels(dg)
    cu, cv = tb.ops.cover_select(dg, level)
    for p, g in GOLD[name].items():
        bounds = np.asarray(g["bounds"])
        own = dm.owned_cover(cu, bounds)
        for i in range(int(p)):
            for s in range(int(p)):
                t = tb.ops.cetc_count_restricted(dg, level, cu[own == s], cv[own == s],
                                                 int(bounds[i]), int(bounds[i + 1]))[0]
                assert t == g["restricted"][i][s], (name, p, i, s)
    assert dm.cetc_dm_distributed(dg) == c.T
