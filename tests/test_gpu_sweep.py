"""Randomised parity sweep of the cover-edge count against the CPU oracle.

The intersection departs from the reference in how it deduplicates
same-level apexes: the reference keeps an apex w on the cover edge's level
iff w > max(u, v) (_kernels.py:687); the GPU's general path keeps it iff w
ranks above both endpoints in (degree bucket desc, id asc) order (intersect.cu
header).  Both select
one of the three edges of an all-horizontal triangle, so T and c2 agree —
this sweep hunts for the inputs where a rank-order bug would hide: heavy
equal-degree ties (regular and circulant graphs, disjoint equal cliques),
dense same-level cliques, hubs outside the dominant component, many small
components, and RMAT/ER mixes, n up to 1e5.  Every graph is checked through
the host-buffer C entry (levels, components, max_level, T, c1, c2) and
through the device path under the default and shrunk tier thresholds
(tcb_set_tuning), which push small owners through the warp and CTA tiers,
their id-range groups and sub-chunk passes, and the CTA tier's bucket-table
fallback (tcb_set_test_flags).  Seeds are fixed, so a failure reproduces.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2403_02997_b200 as tb

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------------------
# generators (edge pairs, possibly with duplicates/loops: normalize drops them)


def _permute(n, pairs, rng):
    perm = rng.permutation(n)
    return perm[pairs] if len(pairs) else pairs


def g_er(rng):
    n = int(rng.integers(2, 4000))
    deg = float(rng.uniform(0.5, 40))
    k = int(n * deg / 2)
    return n, rng.integers(0, n, size=(k, 2))


def g_rmat(rng):
    scale = int(rng.integers(6, 15))
    ef = int(rng.choice([4, 8, 16, 24]))
    seed = int(rng.integers(0, 2**31))
    n = 1 << scale
    pairs = oracle.rmat_pairs(scale, ef, seed=seed)
    return n, _permute(n, pairs, rng)


def g_circulant(rng):
    """C_n(1..k): every vertex has degree 2k (all ranks decided by id)."""
    n = int(rng.integers(8, 3000))
    k = int(rng.integers(1, min(12, (n - 1) // 2) + 1))
    v = np.arange(n)
    pairs = np.concatenate([np.stack([v, (v + s) % n], 1) for s in range(1, k + 1)])
    return n, (_permute(n, pairs, rng) if rng.random() < 0.5 else pairs)


def g_equal_cliques(rng):
    """Disjoint equal-size cliques (each root's neighbours form one
    same-level clique with equal degrees), ids permuted or not."""
    c = int(rng.integers(3, 40))
    cnt = int(rng.integers(1, max(2, 3000 // c)))
    iu = np.stack(np.triu_indices(c, 1), 1)
    pairs = np.concatenate([iu + i * c for i in range(cnt)])
    n = c * cnt
    return n, (_permute(n, pairs, rng) if rng.random() < 0.7 else pairs)


def g_rooted_dense(rng):
    """A root joined to k vertices that form a dense random graph (a wide
    same-level layer with many degree ties), plus a second layer."""
    k = int(rng.integers(4, 400))
    p = float(rng.uniform(0.3, 1.0))
    iu = np.stack(np.triu_indices(k, 1), 1)
    layer = iu[rng.random(len(iu)) < p] + 1
    root = np.stack([np.zeros(k, np.int64), np.arange(1, k + 1)], 1)
    m2 = int(rng.integers(0, 3 * k))
    second = np.stack([rng.integers(1, k + 1, m2), rng.integers(k + 1, 2 * k + 1, m2)], 1)
    n = 2 * k + 1
    pairs = np.concatenate([root, layer, second])
    return n, (_permute(n, pairs, rng) if rng.random() < 0.5 else pairs)


def g_regular_bipartite_plus(rng):
    """K_{a,a} with a perfect matching inside each side: all degrees equal."""
    a = int(rng.integers(2, 120))
    a += a % 2
    left, right = np.arange(a), np.arange(a, 2 * a)
    kab = np.stack(np.meshgrid(left, right, indexing="ij"), -1).reshape(-1, 2)
    match = np.concatenate([np.stack([left[0::2], left[1::2]], 1),
                            np.stack([right[0::2], right[1::2]], 1)])
    n = 2 * a
    return n, _permute(n, np.concatenate([kab, match]), rng)


def g_hub_forest(rng):
    """Many small components; some are stars/fans whose hub is not the
    component minimum, some are triangles, isolated vertices in between."""
    parts, base = [], 0
    for _ in range(int(rng.integers(5, 300))):
        kind = rng.integers(0, 4)
        if kind == 0:  # fan: hub = largest id of the component
            L = int(rng.integers(2, 200))
            hub = base + L
            leaves = base + np.arange(L)
            parts.append(np.stack([np.full(L, hub), leaves], 1))
            parts.append(np.stack([leaves[0:-1:2], leaves[1::2]], 1))
            base += L + 1
        elif kind == 1:  # triangle
            parts.append(np.array([[base, base + 1], [base + 1, base + 2], [base, base + 2]]))
            base += 3
        elif kind == 2:  # small random component
            k = int(rng.integers(2, 60))
            parts.append(base + rng.integers(0, k, size=(3 * k, 2)))
            base += k
        else:  # isolated vertices
            base += int(rng.integers(1, 20))
    n = base + int(rng.integers(0, 5))
    pairs = np.concatenate(parts) if parts else np.zeros((0, 2), np.int64)
    return n, (_permute(n, pairs, rng) if rng.random() < 0.5 else pairs)


def g_mixed(rng):
    """A disjoint union of the other generators, ids shuffled together."""
    parts, base = [], 0
    for _ in range(int(rng.integers(2, 6))):
        gen = GENS[int(rng.integers(0, len(GENS) - 1))]
        n_i, p_i = gen(rng)
        parts.append(p_i + base)
        base += n_i
    return base, _permute(base, np.concatenate(parts), rng)


def g_large(rng):
    """n up to 1e5: RMAT with hubs or a big ER/circulant mix."""
    if rng.random() < 0.5:
        scale = int(rng.integers(15, 17))
        pairs = oracle.rmat_pairs(scale, 16, seed=int(rng.integers(0, 2**31)))
        n = 1 << scale
        return n, _permute(n, pairs, rng)
    n = int(rng.integers(30_000, 100_000))
    return n, rng.integers(0, n, size=(n * int(rng.integers(2, 12)), 2))


GENS = [g_er, g_rmat, g_circulant, g_equal_cliques, g_rooted_dense,
        g_regular_bipartite_plus, g_hub_forest, g_mixed]


def _case(gen, seed):
    rng = np.random.default_rng(seed)
    n, pairs = gen(rng)
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    row, nb, eu, ev = oracle.normalize(n, pairs)
    ref = oracle.run(n, row, nb, eu, ev, threads=4)
    return n, pairs, row, nb, ref


GENERAL_PATH = 8  # tcb_set_test_flags: skip the small-graph kernel (bfs.cu k_small_cetc)


def _check_default(n, row, nb, ref, tag):
    """Through the host entry twice: as dispatched (graphs of <= 2^17
    vertices and edges take the one-launch small-graph kernel) and with the
    general path forced, so the owner-order dedup is checked on every graph."""
    ctx = tb._lib.context()
    for flags in (0, GENERAL_PATH):
        ctx.set_test_flags(flags)
        try:
            r = tb.cetc_host(row, nb, n, want_level=True)
        finally:
            ctx.set_test_flags(0)
        t = (tag, flags)
        assert np.array_equal(r["level"], ref["level"]), t
        assert (r["components"], r["max_level"]) == (ref["components"], ref["max_level"]), t
        assert r["ncover"] == len(ref["cover"]), t
        assert (r["triangles"], r["c1"], r["c2"]) == (ref["T"], ref["c1"], ref["c2"]), t


TUNINGS = [(4, 4), (16, 64), (64, 512), (1024, 16)]


def _check_tuned(n, pairs, ref, tag, flags=0):
    dg = tb.device_graph(tb.normalize(tb.EdgeList(n=n, edges=pairs)))
    ctx = tb._lib.context()
    try:
        ctx.set_test_flags(flags)
        for t in TUNINGS:
            ctx.set_tuning(*t)
            r = tb.cetc(dg)
            assert (r.triangles, r.c1, r.c2) == (ref["T"], ref["c1"], ref["c2"]), (tag, t)
    finally:
        ctx.set_tuning(0, 0)
        ctx.set_test_flags(0)


@pytest.fixture(scope="module", autouse=True)
def _lib_loaded():
    tb._lib.load_library()


@pytest.mark.parametrize("gen", GENS, ids=[g.__name__ for g in GENS])
def test_sweep_default(gen):
    """30 seeded graphs per generator (240 in all) through the host entry."""
    for s in range(30):
        n, _, row, nb, ref = _case(gen, 1000 * GENS.index(gen) + s)
        _check_default(n, row, nb, ref, f"{gen.__name__} seed {s}")


@pytest.mark.parametrize("gen", GENS, ids=[g.__name__ for g in GENS])
def test_sweep_shrunk_tiers(gen):
    """8 seeded graphs per generator under four shrunk tier settings."""
    for s in range(8):
        n, pairs, _, _, ref = _case(gen, 50_000 + 1000 * GENS.index(gen) + s)
        _check_tuned(n, pairs, ref, f"{gen.__name__} seed {s}")


@pytest.mark.parametrize("gen", [g_equal_cliques, g_rooted_dense, g_rmat],
                         ids=["equal_cliques", "rooted_dense", "rmat"])
def test_sweep_cta_fallback(gen):
    """The CTA tier's bucket-table fallback forced on every pass."""
    for s in range(6):
        n, pairs, _, _, ref = _case(gen, 90_000 + s)
        _check_tuned(n, pairs, ref, f"{gen.__name__} seed {s}", flags=4)


def test_sweep_large():
    """Eight graphs with n between 3e4 and 1.3e5 (RMAT hubs, sparse ER)."""
    for s in range(8):
        n, pairs, row, nb, ref = _case(g_large, 70_000 + s)
        _check_default(n, row, nb, ref, f"large seed {s}")
        if s < 3:
            _check_tuned(n, pairs, ref, f"large seed {s}")


def g_wide_layer(rng):
    """A root joined to k = 600..1500 vertices that form a dense random graph
    whose degrees exceed the warp tier's 256: the CTA tier runs with its
    DEFAULT thresholds — UP(x) in the rank bitmap, long same-level lists with
    many degree ties, short bucket runs streamed uncut — and a sparse second
    layer gives every owner OFF ids as well."""
    k = int(rng.integers(600, 1500))
    p = float(rng.uniform(0.35, 0.8))
    iu = np.stack(np.triu_indices(k, 1), 1)
    layer = iu[rng.random(len(iu)) < p] + 1
    root = np.stack([np.zeros(k, np.int64), np.arange(1, k + 1)], 1)
    m2 = int(rng.integers(k, 40 * k))
    second = np.stack([rng.integers(1, k + 1, m2), rng.integers(k + 1, 3 * k + 1, m2)], 1)
    n = 3 * k + 1
    pairs = np.concatenate([root, layer, second])
    return n, (_permute(n, pairs, rng) if rng.random() < 0.7 else pairs)


def test_sweep_cta_tier_default_thresholds():
    """Graphs whose owners exceed degree 256, so the CTA tier (rank bitmap,
    partner records, clamped probes) runs as shipped; also with the bitmap
    window shrunk to 64 / 512 words (rank windows) and the bucket fallback."""
    for s in range(4):
        n, pairs, row, nb, ref = _case(g_wide_layer, 120_000 + s)
        assert int(np.diff(row).max()) > 256
        dg = tb.device_graph(tb.normalize(tb.EdgeList(n=n, edges=pairs)))
        ctx = tb._lib.context()
        try:
            for flags in (GENERAL_PATH, GENERAL_PATH | 4):
                ctx.set_test_flags(flags)
                for t in ((0, 0), (256, 64), (256, 512), (64, 4096)):
                    ctx.set_tuning(*t)
                    r = tb.cetc(dg)
                    assert (r.triangles, r.c1, r.c2) == (ref["T"], ref["c1"], ref["c2"]), (s, flags, t)
        finally:
            ctx.set_tuning(0, 0)
            ctx.set_test_flags(0)

