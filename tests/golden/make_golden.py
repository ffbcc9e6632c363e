"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py small
    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py configs [names...]
    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py parents [names...]

``small``   -> tests/golden/small_cases.npz: inputs and every hot-path output
               (CSR, levels, parents, edge classes, components, max_level,
               cover set, T, c1, c2, the degree-ordered CSR, and which branch
               CETC-Seq-FE takes) of the reference's own test graphs (tests/conftest.py fixtures, karate,
               and the edge cases of test_sequential.py / test_bfs.py).
``configs`` -> tests/golden/configs.json: per BASELINE config, sha256 digests
               of the reference's CSR, levels and cover set plus T, c1, c2,
               components, max_level and work statistics.

The reference is imported read-only from /root/reference/pkg/src.  For
rmat24, where the reference's ``normalize`` takes ~15 min, the CSR comes from
the oracle's ``normalize`` (pinned equal to the reference's on every smaller
config by this same script: see the ``csr_from`` field) and the reference's
``Graph``/``bfs_label``/``tc_cetc_sm`` run on it — the recipe SURVEY.md §8(c)
describes.  Nothing on the GPU box reads /root/reference: only these committed
fixtures travel.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import tricount as tc  # noqa: E402  (the reference)
from tricount.parallel import _cetc_sm_counts  # noqa: E402

from paper_2403_02997_b200 import configs as C  # noqa: E402

GOLDEN = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# small cases: the reference's own fixtures (tests/conftest.py) and edge cases


def _small_inputs():
    def complete(n):
        return n, [(a, b) for a in range(n) for b in range(a + 1, n)]

    def path(n):
        return n, [(i, i + 1) for i in range(n - 1)]

    def cycle(n):
        return n, [(i, (i + 1) % n) for i in range(n)]

    def star(leaves, center=0):
        return leaves + 1, [(center, v) for v in range(leaves + 1) if v != center]

    def er(n, p, seed):
        return n, C.er_pairs(n, p, seed)

    def rmat(scale, ef, seed):
        el = tc.generate_rmat(tc.RmatParams(scale=scale, edge_factor=ef, seed=seed))
        return el.n, el.edges

    karate = tc.load_edge_list("/root/reference/pkg/data/karate.txt")
    cases = {
        "empty0": (0, []),
        "single1": (1, []),
        "two_edges5": (5, [(0, 1), (2, 3)]),       # test_sequential.py:27-31
        "dup_loop3": (3, [(0, 1), (1, 0), (2, 2)]),  # test_graph.py:63-68
        "path3": path(3),                           # test_bfs.py:18-24
        "k3": complete(3),
        "k4": complete(4),
        "k7": complete(7),
        "k8": complete(8),
        "path10": path(10),
        "cycle9": cycle(9),
        "star6": star(6),
        "star4": star(4),                           # test_bfs.py:75-79
        "star3c2": star(3, center=2),
        "strut5": (5, [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4), (1, 4)]),  # test_bfs.py:41-50
        "comps6": (6, [(0, 1), (2, 3), (3, 4)]),    # test_bfs.py:68-71
        "karate": (karate.n, karate.edges),         # pkg/data/karate.txt
        "er60_915": er(60, 0.15, 915),              # test_sequential.py:23-25
        "er40_11": er(40, 0.2, 11),                 # test_bfs.py:112-115
        "rmat10_42": rmat(10, 16, 42),              # test_rmat.py:49-57
        "rmat8_77": rmat(8, 16, 77),                # test_parallel.py:53-58
        "rmat7_9": rmat(7, 16, 9),                  # test_sequential.py:96-99
    }
    for i, (n, p) in enumerate([(20, 0.2), (40, 0.15), (60, 0.1), (80, 0.08)]):
        cases[f"er{n}"] = er(n, p, 100 + i)         # conftest.py:98-99
    for s in (4, 5, 6):
        cases[f"rmat{s}"] = rmat(s, 8, s)           # conftest.py:100-101
    for seed in range(8):
        cases[f"er48_{200 + seed}"] = er(48, 0.18, 200 + seed)  # test_sequential.py:68-73
    for seed in range(6):
        cases[f"er30_{seed}"] = er(30, 0.25, seed)  # test_sequential.py:38-42
    return cases


def make_small():
    out = {}
    names = []
    for name, (n, pairs) in _small_inputs().items():
        edges = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        g = tc.normalize(tc.EdgeList(n=n, edges=edges))
        lab = tc.bfs_label(g)
        cov = tc.cover_edges(lab, g)
        c1, c2 = _cetc_sm_counts(g, tc.ParallelConfig(workers=2))
        T = tc.tc_cetc(g)
        assert T == tc.tc_triples(g) == c1 + c2 // 3, name
        for alg, fn in tc.SEQUENTIAL_IDS.items():  # every CETC id agrees
            if alg.startswith("CETC"):
                assert fn(g) == T, (name, alg)
        gd = tc.degree_order(g)
        p = f"{name}/"
        out[p + "n"] = np.int64(n)
        out[p + "pairs"] = edges
        out[p + "row_offsets"] = g.row_offsets
        out[p + "neighbors"] = g.neighbors
        out[p + "edge_u"] = g.edge_u
        out[p + "edge_v"] = g.edge_v
        out[p + "level"] = lab.level
        out[p + "parent"] = lab.parent
        out[p + "edge_class"] = lab.edge_class
        out[p + "components"] = np.int64(lab.components)
        out[p + "max_level"] = np.int64(lab.max_level)
        out[p + "cover"] = cov.edges
        out[p + "ratio"] = np.float64(cov.ratio)
        out[p + "T"] = np.int64(T)
        out[p + "c1"] = np.int64(c1)
        out[p + "c2"] = np.int64(c2)
        out[p + "deg_row_offsets"] = gd.row_offsets
        out[p + "deg_neighbors"] = gd.neighbors
        ratio = lab.horizontal_count / g.m if g.m else 0.0  # sequential.py:179
        out[p + "fe_forward"] = np.bool_(not ratio < tc.sequential.COVER_RATIO_THRESHOLD)
        names.append(name)
        print(f"{name}: n={n} m={g.m} T={T} c1={c1} c2={c2} cover={len(cov)}")
    out["_names"] = np.array(names)
    np.savez_compressed(GOLDEN / "small_cases.npz", **out)


# ---------------------------------------------------------------------------
# config-scale digests


def _config_graph(cfg, csr_from: str):
    """Build the reference Graph for a config.  csr_from: 'reference' uses the
    reference normalize; 'oracle' builds the CSR with the oracle's normalize
    and wraps it in the reference Graph."""
    n = cfg.n
    if cfg.kind == "er":
        pairs = C.er_pairs(n, cfg.p, cfg.seed)
    elif cfg.kind == "lattice":
        pairs = C.lattice_pairs(cfg.side)
    else:
        perm = C.id_permutation(n, cfg.perm_seed)
        if csr_from == "reference":
            el = tc.generate_rmat(tc.RmatParams(scale=cfg.scale,
                                                edge_factor=cfg.edge_factor,
                                                seed=cfg.seed))
            pairs = perm[el.edges]
        else:
            import oracle
            pairs = oracle.rmat_pairs(cfg.scale, cfg.edge_factor, seed=cfg.seed,
                                      perm=perm)
    if csr_from == "reference":
        return tc.normalize(tc.EdgeList(n=n, edges=pairs))
    import oracle
    row, nb, eu, ev = oracle.normalize(n, pairs)
    for a in (row, nb, eu, ev):
        a.setflags(write=False)
    return tc.Graph(n=n, m=len(eu), row_offsets=row, neighbors=nb,
                    edge_u=eu, edge_v=ev)


def config_digest(name: str, csr_from: str, workers: int = 8) -> dict:
    cfg = C.CONFIGS[name]
    t0 = time.time()
    g = _config_graph(cfg, csr_from)
    t_build = time.time() - t0
    lab = tc.bfs_label(g)
    cov = tc.cover_edges(lab, g)
    t1 = time.time()
    c1, c2 = _cetc_sm_counts(g, tc.ParallelConfig(workers=workers))
    t_sm = time.time() - t1
    T = c1 + c2 // 3
    assert c2 % 3 == 0
    deg = np.diff(g.row_offsets)
    cu = cov.edges[:, 0]
    cv = cov.edges[:, 1]
    du = deg[cu]
    dv = deg[cv]
    hist = np.bincount(lab.level, minlength=lab.max_level + 1)
    rec = dict(
        name=name, csr_from=csr_from, n=g.n, m=int(g.m),
        dmax=int(deg.max()) if g.n else 0,
        row_offsets_sha=sha(g.row_offsets.astype(np.int64)),
        neighbors_sha=sha(g.neighbors.astype(np.int32)),
        level_sha=sha(lab.level.astype(np.int32)),
        level_hist=[int(x) for x in hist],
        components=int(lab.components), max_level=int(lab.max_level),
        cover_count=int(len(cov)), cover_sha=sha(cov.edges.astype(np.int32)),
        ratio=float(cov.ratio),
        T=int(T), c1=int(c1), c2=int(c2),
        W=int((du + dv).sum()), W_min=int(np.minimum(du, dv).sum()),
        seconds_build=round(t_build, 2), seconds_cetc_sm=round(t_sm, 2),
        workers=workers,
    )
    if name == "er4096":
        rec["level_int8"] = [int(x) for x in lab.level]
    return rec


def make_configs(names):
    path = GOLDEN / "configs.json"
    data = json.loads(path.read_text()) if path.exists() else {}
    for name in names:
        csr_from = "oracle" if name == "rmat24" else "reference"
        rec = config_digest(name, csr_from)
        if csr_from == "reference" and name != "er4096":
            # pin the oracle's normalize against the reference's at this scale
            import oracle
            cfg = C.CONFIGS[name]
            g2 = _config_graph(cfg, "oracle")
            rec["oracle_csr_matches"] = bool(
                sha(g2.row_offsets.astype(np.int64)) == rec["row_offsets_sha"]
                and sha(g2.neighbors.astype(np.int32)) == rec["neighbors_sha"])
            assert rec["oracle_csr_matches"], name
            del oracle
        rec.pop("level_int8", None) if name != "er4096" else None
        data[name] = rec
        print(json.dumps({k: v for k, v in rec.items() if k != "level_int8"}))
        path.write_text(json.dumps(data, indent=1, sort_keys=True))


def add_parent_digests(names):
    """Add the reference's FIFO parents and edge classes (bfs_label,
    bfs.py:76-94) to existing config records as sha256 digests.  The CSR is
    the oracle's (identical to the reference's normalize at every config where
    both ran: oracle_csr_matches), wrapped in the reference Graph; only the
    labeling runs, so RMAT-24 takes seconds, not the CETC-SM hours."""
    path = GOLDEN / "configs.json"
    data = json.loads(path.read_text())
    for name in names:
        cfg = C.CONFIGS[name]
        g = _config_graph(cfg, "oracle")
        assert sha(g.row_offsets.astype(np.int64)) == data[name]["row_offsets_sha"], name
        assert sha(g.neighbors.astype(np.int32)) == data[name]["neighbors_sha"], name
        t0 = time.time()
        lab = tc.bfs_label(g)
        assert sha(lab.level.astype(np.int32)) == data[name]["level_sha"], name
        data[name]["parent_sha"] = sha(lab.parent.astype(np.int64))
        data[name]["edge_class_sha"] = sha(lab.edge_class.astype(np.int8))
        print(name, "bfs_label", round(time.time() - t0, 1), "s", data[name]["parent_sha"][:12])
        path.write_text(json.dumps(data, indent=1, sort_keys=True))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        make_small()
    elif what == "configs":
        make_configs(sys.argv[2:] or ["er4096", "rmat16", "lattice2048"])
    elif what == "parents":
        add_parent_digests(sys.argv[2:] or ["er4096", "rmat16", "lattice2048", "rmat22",
                                            "rmat24"])
    else:
        raise SystemExit(f"unknown target {what}")
