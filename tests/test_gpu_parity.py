"""GPU parity: the CUDA path (through the C ABI) against the reference's
outputs (golden fixtures) and the CPU oracle.  Bit-exact: integer work."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
import paper_2403_02997_b200 as tb
from conftest import SMALL_CASES, SMALL_IDS, config_goldens
from paper_2403_02997_b200 import configs as C

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module", autouse=True)
def _lib_loaded():
    tb._lib.load_library()


@pytest.mark.parametrize("case", SMALL_CASES, ids=SMALL_IDS)
def test_normalize_matches_reference(case):
    g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
    assert g.n == case.n and g.m == case.m
    assert g.row_offsets.dtype == np.int64 and g.neighbors.dtype == np.int32
    assert np.array_equal(g.row_offsets, case.row)
    assert np.array_equal(g.neighbors, case.nb)
    assert np.array_equal(g.edge_u, case.eu) and np.array_equal(g.edge_v, case.ev)
    with pytest.raises(ValueError):
        g.neighbors[:1] = 0  # frozen, as graph.py:99-101


@pytest.mark.parametrize("case", SMALL_CASES, ids=SMALL_IDS)
def test_labels_cover_counts_match_reference(case):
    g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
    lab = tb.bfs_label(g)
    assert lab.level.dtype == np.int64
    assert np.array_equal(lab.level, case.level)
    assert lab.parent.dtype == np.int64 and np.array_equal(lab.parent, case.parent)
    assert lab.edge_class.dtype == np.int8 and np.array_equal(lab.edge_class, case.edge_class)
    assert lab.components == case.components
    assert lab.max_level == case.max_level
    cov = tb.cover_edges(lab, g)
    assert cov.edges.dtype == np.int64 and cov.edges.shape == (len(case.cover), 2)
    assert np.array_equal(cov.edges, case.cover)
    assert cov.ratio == case.ratio
    assert lab.horizontal_count == len(case.cover)
    assert tb.tc_cetc(g) == case.T
    assert tb.SEQUENTIAL_IDS["CETC-Seq"](g) == case.T
    for w in (1, 2, 8):
        assert tb.tc_cetc_sm(g, tb.ParallelConfig(workers=w)) == case.T
    assert tb.parallel._cetc_sm_counts(g, tb.ParallelConfig(workers=2)) == (case.c1, case.c2)


@pytest.mark.parametrize("case", SMALL_CASES, ids=SMALL_IDS)
def test_cetc_family_and_forward(case):
    """Every CETC id of the cetc-family group (bench.py:42-43), the GPU forward
    count, the FE branch choice (sequential.py:176-183) and degree_order
    (graph.py:203-213) against the reference's outputs."""
    g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
    for alg, fn in tb.SEQUENTIAL_IDS.items():
        assert fn(g) == case.T, alg
    assert tb.count_sequential("CETC-Seq-FE", g) == case.T
    assert tb.tc_forward_gpu(g) == case.T
    r, used_forward = tb.ops.cetc_fe(tb.device_graph(g))
    assert used_forward == case.fe_forward
    assert r.triangles == case.T and r.ncover == len(case.cover)
    if not used_forward:
        assert (r.c1, r.c2) == (case.c1, case.c2)
    gd = tb.degree_order(g)
    assert gd.m == g.m
    assert np.array_equal(gd.row_offsets, case.deg_row)
    assert np.array_equal(gd.neighbors, case.deg_nb)


@pytest.mark.parametrize("case", SMALL_CASES, ids=SMALL_IDS)
def test_host_buffer_entry(case):
    r = tb.cetc_host(case.row, case.nb, case.n, want_level=True)
    assert (r["triangles"], r["c1"], r["c2"]) == (case.T, case.c1, case.c2)
    assert r["ncover"] == len(case.cover)
    assert r["components"] == case.components and r["max_level"] == case.max_level
    assert np.array_equal(r["level"], case.level)


def test_cetc_count_ranges_sum():
    case = next(c for c in SMALL_CASES if c.name == "rmat10_42")
    dg = tb.device_graph(tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs)))
    level, _, _ = tb.ops.bfs_levels(dg)
    cu, cv = tb.ops.cover_select(dg, level)
    k = cu.numel()
    parts = [tb.ops.cetc_count(dg, level, cu, cv, a, b)
             for a, b in tb.ParallelConfig(workers=3).ranges(k)]
    assert sum(p[1] for p in parts) == case.c1
    assert sum(p[2] for p in parts) == case.c2
    assert sum(p[0] for p in parts) == case.T


@pytest.mark.parametrize("scale,ef,seed", [(4, 8, 4), (10, 16, 42), (14, 16, 3), (16, 16, 1)])
def test_device_rmat_matches_oracle(scale, ef, seed):
    got = tb.generate_rmat(tb.RmatParams(scale=scale, edge_factor=ef, seed=seed)).edges
    assert np.array_equal(got, oracle.rmat_pairs(scale, ef, seed=seed))


def test_device_rmat_matches_reference_fixture():
    case = next(c for c in SMALL_CASES if c.name == "rmat10_42")
    got = tb.generate_rmat(tb.RmatParams(scale=10, edge_factor=16, seed=42)).edges
    assert np.array_equal(got, case.pairs)


def test_csr_with_loops_and_duplicates_random():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 100, 5000):
        pairs = rng.integers(0, n, size=(3 * n + 5, 2))
        g = tb.normalize(tb.EdgeList(n=n, edges=pairs))
        row, nb, eu, ev = oracle.normalize(n, pairs)
        assert np.array_equal(g.row_offsets, row) and np.array_equal(g.neighbors, nb)
        assert np.array_equal(g.edge_u, eu) and np.array_equal(g.edge_v, ev)


@pytest.mark.parametrize("n,p,seed", [(2, 0.5, 0), (30, 0.25, 3), (48, 0.18, 205),
                                       (4096, 16 / 4095, 1), (1000, 0.9, 7)])
def test_device_er_recipe_matches_numpy(n, p, seed):
    got = C.er_pairs_device(n, p, seed).cpu().numpy()
    assert np.array_equal(got, C.er_pairs(n, p, seed))


@pytest.mark.parametrize("side", [1, 2, 3, 17, 2048])
def test_device_lattice_matches_host(side):
    got = C.lattice_pairs_device(side).cpu().numpy()
    assert np.array_equal(got, C.lattice_pairs(side))


def _check_config(name):
    import torch
    gold = config_goldens()[name]
    dg = C.build_device_graph(name)
    assert dg.m == gold["m"]
    assert sha(dg.row_offsets.cpu().numpy()) == gold["row_offsets_sha"]
    assert sha(dg.neighbors.cpu().numpy()) == gold["neighbors_sha"]
    r = tb.cetc(dg, keep_level=True, keep_cover=True)
    assert (r.triangles, r.c1, r.c2) == (gold["T"], gold["c1"], gold["c2"])
    assert r.components == gold["components"] and r.max_level == gold["max_level"]
    assert r.ncover == gold["cover_count"]
    assert sha(r.level.cpu().numpy()) == gold["level_sha"]
    cover = torch.stack([r.cover_u, r.cover_v], dim=1).cpu().numpy()
    assert sha(cover) == gold["cover_sha"]
    hist = np.bincount(r.level.cpu().numpy(), minlength=len(gold["level_hist"]))
    assert hist.tolist() == gold["level_hist"]


@pytest.mark.parametrize("name", ["er4096", "rmat16", "lattice2048"])
def test_config_parity(name):
    _check_config(name)


@pytest.mark.parametrize("name", ["er4096", "lattice2048"])
def test_config_parity_general_path(name):
    """ER-4096 (small-graph kernel) and the lattice (low-degree count) again
    with TCB_TEST_GENERAL_PATH: the owner-order lists and tiers at config
    scale must give the same outputs."""
    ctx = tb._lib.context()
    ctx.set_test_flags(8)
    try:
        _check_config(name)
    finally:
        ctx.set_test_flags(0)


def _check_parent(name):
    """FIFO parents and edge classes at config scale against the reference's
    own bfs_label (sha256 digests in configs.json, tests/golden/make_golden.py
    parents) and the C oracle's FIFO BFS."""
    import torch
    dg = C.build_device_graph(name)
    level, _, max_level = tb.ops.bfs_levels(dg)
    parent = tb.ops.bfs_parent(dg, level, max_level)
    classes = tb.ops.edge_classes(dg, level, parent)
    gold = config_goldens().get(name, {})
    if "parent_sha" in gold:
        assert sha(parent.cpu().numpy().astype(np.int64)) == gold["parent_sha"]
        assert sha(classes.cpu().numpy().astype(np.int8)) == gold["edge_class_sha"]
    row, nb = dg.row_offsets.cpu().numpy(), dg.neighbors.cpu().numpy()
    o_level, o_parent, _, _ = oracle.bfs_levels(row, nb, dg.n)
    assert np.array_equal(level.cpu().numpy(), o_level)
    assert np.array_equal(parent.cpu().numpy().astype(np.int64), o_parent)
    eu, ev = (t.cpu().numpy() for t in dg.edge_arrays())
    assert np.array_equal(classes.cpu().numpy(), oracle.edge_classes(o_level, o_parent, eu, ev))
    del torch


def _check_variants(name):
    gold = config_goldens()[name]
    dg = C.build_device_graph(name)
    assert tb.ops.forward_count(dg) == gold["T"]
    # the split hybrids (sequential.py:197-238): G0's forward count + the cross count
    level, _, _ = tb.ops.bfs_levels(dg)
    g0 = tb.ops.split_by_level(dg, level)
    assert g0.m == gold["cover_count"]
    cross = tb.ops.split_cross_count(dg, level)
    assert cross == gold["c1"]  # one horizontal edge, two level-spanning: the c1 triangles
    assert tb.ops.forward_count(g0) == gold["c2"] // 3
    assert tb.sequential._split_count(dg) == gold["T"]
    assert tb.sequential._split_recursive(dg, tb.COVER_RATIO_THRESHOLD, 1.0) == gold["T"]
    r, used_forward = tb.ops.cetc_fe(dg)
    assert r.triangles == gold["T"]
    assert used_forward == (gold["cover_count"] / dg.m >= tb.COVER_RATIO_THRESHOLD)
    dd = tb.degree_order_device(dg)
    rd = tb.cetc(dd)
    assert rd.triangles == gold["T"] and dd.m == dg.m


@pytest.mark.parametrize("name", ["er4096", "rmat16", "lattice2048"])
def test_config_variants(name):
    _check_variants(name)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["rmat22", "rmat24"])
def test_config_variants_large(name):
    _check_variants(name)


@pytest.mark.parametrize("name", ["er4096", "rmat16", "lattice2048"])
def test_config_parent_classes(name):
    _check_parent(name)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["rmat22", "rmat24"])
def test_config_parent_classes_large(name):
    _check_parent(name)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["rmat22", "rmat24"])
def test_config_parity_large(name):
    if name not in config_goldens():
        pytest.skip(f"no golden for {name}")
    _check_config(name)


@pytest.mark.parametrize("tuning", [(4, 4), (4, 8), (16, 64), (1024, 16), (0, 0)])
def test_every_intersection_path_small(tuning):
    """Shrunk thresholds push small owners through the CTA tier, its range
    groups and the sub-chunk path; counts must not change."""
    ctx = tb._lib.context()
    ctx.set_tuning(*tuning)
    try:
        for case in SMALL_CASES:
            g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
            r = tb.cetc(tb.device_graph(g))
            assert (r.triangles, r.c1, r.c2) == (case.T, case.c1, case.c2), case.name
    finally:
        ctx.set_tuning(0, 0)


def _numpy_split(case):
    """_split_by_level + split_cross_count_k restated with numpy/sets on the
    reference's levels (small cases only)."""
    lev = case.level
    row, nb = case.row, case.nb
    src = np.repeat(np.arange(case.n), np.diff(row))
    keep = lev[src] == lev[nb]
    row0 = np.concatenate([[0], np.cumsum(np.bincount(src[keep], minlength=case.n))])
    nb0 = nb[keep]
    n1 = [set(map(int, nb[row[v]:row[v + 1]][lev[nb[row[v]:row[v + 1]]] != lev[v]]))
          for v in range(case.n)]
    cross = 0
    for u, v in zip(case.eu, case.ev):
        if lev[u] == lev[v]:
            cross += len(n1[u] & n1[v])
    return row0, nb0, cross


@pytest.mark.parametrize("case", SMALL_CASES, ids=SMALL_IDS)
def test_split_by_level_and_cross_count(case):
    """tcb_split_by_level and tcb_split_cross_count against a numpy
    restatement of _split_by_level (sequential.py:186-193) and
    split_cross_count_k (_kernels.py:786-805) on the reference's levels."""
    import torch
    g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
    dg = tb.device_graph(g)
    level = torch.from_numpy(case.level.astype(np.int32))
    g0 = tb.ops.split_by_level(dg, level)
    row0, nb0, cross = _numpy_split(case)
    assert np.array_equal(g0.row_offsets.cpu().numpy(), row0)
    assert np.array_equal(g0.neighbors.cpu().numpy(), nb0)
    assert g0.m == len(case.cover)
    assert tb.ops.split_cross_count(dg, level) == cross == case.c1
    for alg in ("CETC-Seq-S", "CETC-Seq-SD", "CETC-Seq-SR"):
        assert tb.SEQUENTIAL_IDS[alg](g) == case.T, alg
    assert tb.tc_cetc_split_recursive(g, threshold=0.0) == case.T


def test_general_path_on_small_cases():
    """The small cases normally take the one-launch small-graph kernel; with
    TCB_TEST_GENERAL_PATH they take the general path (owner-order lists,
    default tiers): both must reproduce the reference."""
    ctx = tb._lib.context()
    ctx.set_test_flags(8)  # TCB_TEST_GENERAL_PATH
    try:
        for case in SMALL_CASES:
            g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
            r = tb.cetc(tb.device_graph(g), keep_level=True)
            assert (r.triangles, r.c1, r.c2) == (case.T, case.c1, case.c2), case.name
            assert r.ncover == len(case.cover), case.name
            assert np.array_equal(r.level.cpu().numpy(), case.level), case.name
    finally:
        ctx.set_test_flags(0)


@pytest.mark.parametrize("tuning", [(64, 64), (16, 512)])
def test_every_intersection_path_rmat16(tuning):
    gold = config_goldens()["rmat16"]
    dg = C.build_device_graph("rmat16")
    ctx = tb._lib.context()
    ctx.set_tuning(*tuning)
    try:
        r = tb.cetc(dg)
    finally:
        ctx.set_tuning(0, 0)
    assert (r.triangles, r.c1, r.c2) == (gold["T"], gold["c1"], gold["c2"])


def test_hub_outside_dominant_component():
    """A long cycle holding vertex 0 (the first BFS's root) plus a star whose
    hub is not its component's minimum: the star is left for the remainder
    union-find, where the hub's row takes the warp-cooperative hooking path
    (k_rest_hook), and a triangle fan on the star exercises the second BFS
    and the count on a non-root component."""
    rng = np.random.default_rng(11)
    n_cyc, leaves = 200_000, 5000
    cyc = np.stack([np.arange(n_cyc), (np.arange(n_cyc) + 1) % n_cyc], axis=1)
    hub = n_cyc + leaves  # the star's largest id; its minimum is the first leaf
    star = np.stack([np.full(leaves, hub), n_cyc + np.arange(leaves)], axis=1)
    fan = np.stack([n_cyc + np.arange(0, leaves - 1, 2), n_cyc + np.arange(1, leaves, 2)], axis=1)
    pairs = np.concatenate([cyc, star, fan])
    pairs = pairs[rng.permutation(len(pairs))]
    n = hub + 1
    g = tb.normalize(tb.EdgeList(n=n, edges=pairs))
    row, nb, eu, ev = oracle.normalize(n, pairs)
    ref = oracle.run(n, row, nb, eu, ev, threads=2)
    lab = tb.bfs_label(g)
    assert np.array_equal(lab.level, ref["level"])
    assert (lab.components, lab.max_level) == (ref["components"], ref["max_level"])
    assert tb.tc_cetc(g) == ref["T"] == leaves // 2


@pytest.mark.parametrize("tuning", [(16, 64), (0, 0)])
def test_cta_bucket_fallback_path(tuning):
    """The bucket-table fallback of the CTA tier (taken when a cuckoo build
    fails) forced on every pass: counts must not change."""
    ctx = tb._lib.context()
    ctx.set_tuning(*tuning)
    ctx.set_test_flags(4)  # TCB_TEST_FORCE_FALLBACK
    try:
        for case in SMALL_CASES:
            g = tb.normalize(tb.EdgeList(n=case.n, edges=case.pairs))
            r = tb.cetc(tb.device_graph(g))
            assert (r.triangles, r.c1, r.c2) == (case.T, case.c1, case.c2), case.name
        gold = config_goldens()["rmat16"]
        r = tb.cetc(C.build_device_graph("rmat16"))
        assert (r.triangles, r.c1, r.c2) == (gold["T"], gold["c1"], gold["c2"])
    finally:
        ctx.set_test_flags(0)
        ctx.set_tuning(0, 0)


@pytest.mark.slow
def test_capacity_rmat25_matches_forward():
    """Beyond BASELINE.json's sizes (2m ≈ 1.05e9 entries): the cover-edge
    count equals the independent GPU forward count, c2 is a multiple of 3 and
    the level rule splits T = c1 + c2/3 (size-independent properties)."""
    import torch
    dg = C.build_device_graph("rmat25")
    r = tb.cetc(dg)
    assert dg.m == 523_604_945
    assert r.c2 % 3 == 0 and r.triangles == r.c1 + r.c2 // 3
    assert r.triangles == tb.ops.forward_count(dg) == 22_534_446_128
    del dg
    torch.cuda.empty_cache()


def test_host_entry_copy_rmat22():
    """tcb_cetc_host on RMAT-22 (the neighbour array copied on the copy
    stream under the entry->row map): identical counts, components and
    levels to the device-resident path."""
    import torch
    dg = C.build_device_graph("rmat22")
    dev = tb.cetc(dg, keep_level=True)
    row = dg.row_offsets.cpu().numpy()
    nb = dg.neighbors.cpu().numpy()
    assert len(nb) >= 1 << 26
    host = tb.ops.cetc_host(row, nb, dg.n, want_level=True)
    assert (host["triangles"], host["c1"], host["c2"], host["ncover"], host["components"],
            host["max_level"]) == (dev.triangles, dev.c1, dev.c2, dev.ncover, dev.components,
                                   dev.max_level)
    assert np.array_equal(host["level"], dev.level.cpu().numpy().astype(np.int64))
    del dg, dev
    torch.cuda.empty_cache()


def test_concurrent_calls_from_threads():
    """The reference kernels are nogil and safe for concurrent calls
    (_kernels.py:1-8); here every Python thread gets its own library context
    (workspace + copy stream), so concurrent tc_cetc / bfs_label / host-entry
    calls on shared Graphs give the single-threaded answers."""
    from concurrent.futures import ThreadPoolExecutor
    cases = SMALL_CASES[:12]
    graphs = [tb.normalize(tb.EdgeList(n=c.n, edges=c.pairs)) for c in cases]

    def work(i):
        c, g = cases[i % len(cases)], graphs[i % len(cases)]
        lab = tb.bfs_label(g)
        h = tb.ops.cetc_host(c.row, c.nb, c.n) if c.n else {"triangles": 0}
        return tb.tc_cetc(g), np.asarray(lab.level).tolist(), h["triangles"]

    with ThreadPoolExecutor(max_workers=6) as ex:
        out = list(ex.map(work, range(4 * len(cases))))
    for i, (t, level, th) in enumerate(out):
        c = cases[i % len(cases)]
        assert t == th == c.T, c.name
        assert level == c.level.tolist(), c.name


@pytest.mark.parametrize("nbytes", [0, 4, 1 << 20, (96 << 20) + 12])
def test_copy_to_device_pageable_and_pinned(nbytes):
    """tcb_copy_to_device: pinned sources are one DMA, pageable ones go through
    the 32 MB staging ring (96 MB + 12 bytes: three full chunks and a tail);
    both must land byte-exact (the drop-in upload of a reference Graph)."""
    import torch
    ctx = tb._lib.context()
    rng = np.random.default_rng(nbytes)
    host = rng.integers(0, 256, size=nbytes, dtype=np.uint8)
    for pinned in (False, True):
        src = host
        if pinned:
            t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            t.numpy()[:] = host
            src = t.numpy()
        dev = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        ctx.check(ctx.lib.tcb_copy_to_device(ctx.h, tb._lib.ptr(dev), src.ctypes.data, nbytes))
        assert np.array_equal(dev[:nbytes].cpu().numpy(), host), pinned
